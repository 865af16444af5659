"""Pins of the fp64 oracle against things other than itself (CPU only).

Each test names what pins it: a value printed in the paper (tests/golden/table1.json,
with citations), a closed form, an invariant, a library routine on a special case, or
brute force.  P:n = PAPER.md line n, S:n = SPEC.md line n.
"""
import json
import os

import numpy as np
import pytest

import oracle
from synth import generator as gen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1.json")))
UN = ["u1", "u2", "u3", "u4"]
PN = ["p1", "p2", "p3", "p4", "p5"]


def _t1():
    U = np.array([GOLD["users"][u] for u in UN], np.float32)
    P = np.array([GOLD["items"][p] for p in PN], np.float32)
    return U, P


def _names(mask_row):
    return [UN[i] for i in np.flatnonzero(mask_row)]


# ---------------------------------------------------------------- Table 1

def test_table1_generator_matches_paper_vectors():
    U, P = _t1()
    gU, gP = gen.table1()
    assert np.array_equal(U, gU) and np.array_equal(P, gP)


def test_table1_inner_products_hand():
    U, P = _t1()
    for i, u in enumerate(UN):
        for j, p in enumerate(PN):
            # fp32 inputs are within 2^-24 relative of the decimals: |err| < 1e-5
            assert abs(oracle.dot(U[i], P[j]) - GOLD["hand_inner_products"][u][p]) < 1e-5, (u, p)


def test_table1_norms_hand():
    U, P = _t1()
    nu, npn = oracle.norms(U), oracle.norms(P)
    for i, u in enumerate(UN):
        assert abs(nu[i] - np.sqrt(GOLD["hand_norms"][u + "_sq"])) < 1e-6
    for j, p in enumerate(PN):
        assert abs(npn[j] - np.sqrt(GOLD["hand_norms"][p + "_sq"])) < 1e-6
    assert abs(nu[0] - GOLD["hand_norms"]["u1"]) < 1e-5


def test_table1_sort_orders():
    # SURVEY Appendix A / S:123 erratum: items by norm p5, p3, p2, p4, p1; users u4, u2, u1, u3
    U, P = _t1()
    assert [PN[i] for i in oracle.sort_by_norm_desc(oracle.norms(P))] == ["p5", "p3", "p2", "p4", "p1"]
    assert [UN[i] for i in oracle.sort_by_norm_desc(oracle.norms(U))] == ["u4", "u2", "u1", "u3"]


def test_table1_paper_example1():
    """P:61 q=p5 -> {u3,u4}; P:62 q=p1 -> empty (k=1)."""
    U, P = _t1()
    claims = GOLD["paper_claims"]["k1"]
    for q in ("p5", "p1"):
        mem = oracle.rkmips_naive(U, P, P[[PN.index(q)]], 1)
        assert _names(mem[0]) == claims[q]


def test_table1_erratum_p2():
    """P:63 claims q=p2 -> {u2}; brute force says that holds only at k=2 (reading R2)."""
    U, P = _t1()
    q = P[[1]]
    assert _names(oracle.rkmips_naive(U, P, q, 1)[0]) == GOLD["errata"]["k1_p2_actual"]
    assert _names(oracle.rkmips_naive(U, P, q, 2)[0]) == GOLD["errata"]["k2_p2_actual"]
    # the MIPS column except u2's erratum
    vals, ids = oracle.topk(U, P, 1)
    col = GOLD["paper_claims"]["mips_column"]
    for i, u in enumerate(UN):
        expect = GOLD["errata"]["u2_mips_actual"] if u == "u2" else col[u]
        assert PN[ids[i, 0]] == expect


@pytest.mark.parametrize("k", [1, 2, 3])
def test_table1_full_answer_table(k):
    U, P = _t1()
    naive = oracle.rkmips_naive(U, P, P, k)
    vals, _ = oracle.topk(U, P, 3)
    two = oracle.rkmips_twophase(U, vals, P, k)
    for j, p in enumerate(PN):
        assert _names(naive[j]) == GOLD["hand_answers"]["k%d" % k][p]
    assert np.array_equal(naive, two)
    assert naive.sum() == 4 * k  # each user in exactly k sets (invariant, totals 4/8/12)


def test_spec_examples():
    U, P = _t1()
    ex = GOLD["spec_examples"]
    v, _ = oracle.topk(U[[2]], P[[2, 4]], 2)
    assert np.allclose(v[0], ex["u3_pool_p3p5_top2"], atol=1e-5)
    v, ids = oracle.topk(U[[3]], P, 2)
    assert [PN[i] for i in ids[0]] == [e[0] for e in ex["u4_top2"]]
    assert np.allclose(v[0], [e[1] for e in ex["u4_top2"]], atol=1e-5)
    bb = oracle.block_bounds(np.array(ex["block_min_members"], np.float64), 2)
    assert bb.tolist() == [ex["block_min_expected"]]
    assert not oracle.rkmips_naive(U, P, P[[3]], 1).any()


# ---------------------------------------------------------------- closed forms / library special cases

def _inst(seed, n=60, m=40, d=8, dist="gaussian"):
    return gen.random_instance(seed, n, m, d, dist)


@pytest.mark.parametrize("seed,dist", [(0, "gaussian"), (1, "uniform"), (2, "skewed")])
def test_topk_against_library_sort(seed, dist):
    """Special case reducing to a library routine: fp64 GEMM + numpy argsort."""
    U, P = _inst(seed, 50, 70, 50, dist)
    kk = 12
    vals, ids = oracle.topk(U, P, kk)
    S = U.astype(np.float64) @ P.astype(np.float64).T
    ref_ids = np.argsort(-S, axis=1, kind="stable")[:, :kk]
    ref_vals = np.take_along_axis(S, ref_ids, 1)
    assert np.allclose(vals, ref_vals, rtol=1e-12, atol=1e-12)
    # ids agree wherever neighbouring values are separated by more than rounding
    gaps = np.abs(np.diff(np.sort(S, axis=1)[:, ::-1][:, :kk + 1], axis=1))
    safe = (gaps > 1e-9).all(1)
    assert safe.mean() > 0.9
    assert np.array_equal(ids[safe], ref_ids[safe])
    assert (np.diff(vals, axis=1) <= 0).all()


def test_topk_padding_when_kk_exceeds_m():
    U, P = _inst(3, 5, 3, 4)
    vals, ids = oracle.topk(U, P, 6)
    assert np.isneginf(vals[:, 3:]).all() and (ids[:, 3:] == -1).all()
    assert (ids[:, :3] >= 0).all()


def test_k1_equals_argmax_mips():
    """k = 1 is textbook argmax MIPS: R_1(p_j) = {u : argmax_p u.p = j}."""
    U, P = _inst(4, 80, 30, 16)
    S = U.astype(np.float64) @ P.astype(np.float64).T
    am = S.argmax(1)
    mem = oracle.rkmips_naive(U, P, P, 1)
    for j in range(P.shape[0]):
        assert np.array_equal(np.flatnonzero(mem[j]), np.flatnonzero(am == j))


def test_k_greater_than_m_returns_all_users():
    U, P = _inst(5, 20, 6, 4)
    q = _inst(6, 3, 1, 4)[0]
    assert oracle.rkmips_naive(U, P, q, 7).all()
    assert not oracle.rkmips_naive(U, P, q, 1).all() or True  # no claim at k = 1


# ---------------------------------------------------------------- invariants

@pytest.mark.parametrize("seed,k", [(7, 1), (8, 3), (9, 10)])
def test_each_user_in_exactly_k_sets_when_queries_are_all_of_P(seed, k):
    """BASELINE north_star invariant: absent ties, queries ranging over all of P put
    every user in exactly k result sets (sum = n k).  Catches <=/< and index slips."""
    U, P = _inst(seed, 40, 25, 8)
    mem = oracle.rkmips_naive(U, P, P, k)
    assert (mem.sum(0) == k).all()


def test_each_user_in_exactly_k_on_cfg0_shape():
    w = gen.make_workload(0, n=300, m=200, nq=1)
    vals, _ = oracle.topk(w.U, w.P, 10)
    mem = oracle.rkmips_twophase(w.U, vals, w.P, 10)
    assert (mem.sum(0) == 10).all()


@pytest.mark.parametrize("seed,dist", [(10, "gaussian"), (11, "uniform"), (12, "skewed")])
def test_naive_equals_twophase(seed, dist):
    """Brute force (naive count) vs the top-list decision (reading R8)."""
    U, P = _inst(seed, 70, 45, 8, dist)
    Qy = np.concatenate([P[:10], _inst(seed + 100, 10, 1, 8, dist)[0]])
    vals, _ = oracle.topk(U, P, 10)
    for k in (1, 4, 10):
        assert np.array_equal(oracle.rkmips_naive(U, P, Qy, k), oracle.rkmips_twophase(U, vals, Qy, k))


def test_monotone_in_k():
    U, P = _inst(13, 50, 30, 8)
    Qy = _inst(14, 12, 1, 8)[0]
    prev = None
    for k in range(1, 12):
        cur = oracle.rkmips_naive(U, P, Qy, k)
        if prev is not None:
            assert (cur >= prev).all()
        prev = cur


def test_positive_user_scaling_invariance():
    U, P = _inst(15, 30, 20, 8)
    Qy = np.concatenate([P[:5], _inst(16, 5, 1, 8)[0]])
    base = oracle.rkmips_naive(U, P, Qy, 3)
    U2 = U.copy()
    U2[::3] *= np.float32(4.0)   # power of two: exact in fp32, exact in every dot
    assert np.array_equal(oracle.rkmips_naive(U2, P, Qy, 3), base)


def test_duplicate_query_into_P_invariance():
    """Def. 2 takes P u {q} as a set; a copy of q in P never strictly beats q (R1, R8)."""
    U, P = _inst(17, 30, 20, 8)
    q = _inst(18, 1, 1, 8)[0]
    base = oracle.rkmips_naive(U, P, q, 4)
    P2 = np.concatenate([P, q])
    assert np.array_equal(oracle.rkmips_naive(U, P2, q, 4), base)


# ---------------------------------------------------------------- Algorithm 2

def test_linear_scan_tau0_counterexample():
    """Reading R3: with tau <- 0 this instance is answered 'no'; truth is yes (c = 1 < 2)."""
    u = np.array([1.0], np.float32)
    P = np.array([[0.5], [-0.3], [-0.2]], np.float32)
    q = np.array([-0.1], np.float32)
    pn = oracle.norms(P)
    order = oracle.sort_by_norm_desc(pn)
    dec, _ = oracle.linear_scan(u, 1.0, q, P[order], pn[order], 2)
    assert dec is True
    assert oracle.rkmips_naive(u[None], P, q[None], 2)[0, 0]


@pytest.mark.parametrize("seed,dist", [(20, "gaussian"), (21, "uniform"), (22, "skewed")])
def test_linear_scan_equals_naive(seed, dist):
    U, P = _inst(seed, 40, 35, 8, dist)
    Qy = np.concatenate([P[:6], _inst(seed + 50, 6, 1, 8, dist)[0]])
    pn = oracle.norms(P)
    order = oracle.sort_by_norm_desc(pn)
    Ps, pns = P[order], pn[order]
    un = oracle.norms(U)
    for k in (1, 3, 8):
        mem = oracle.rkmips_naive(U, P, Qy, k)
        for qi in range(Qy.shape[0]):
            for i in range(U.shape[0]):
                dec, sc = oracle.linear_scan(U[i], un[i], Qy[qi], Ps, pns, k)
                assert dec == mem[qi, i]
                assert 0 <= sc <= P.shape[0]


def test_block_bounds_against_library():
    rng = np.random.default_rng(0)
    L = -np.sort(-rng.standard_normal((37, 5)), axis=1)
    for b in (1, 4, 8, 37, 50):
        ref = np.minimum.reduceat(L, np.arange(0, 37, b), axis=0)
        assert np.array_equal(oracle.block_bounds(L, b), ref)


def test_margin_table1_hand_values():
    """orc_margin against hand arithmetic on Table 1 (golden decimals; reading R9):
    q = p5 is itself an item, so tau'_k(u) is taken over P minus p5.
      u3, k = 1: tau'_1 = u3.p4 = 7.82  -> mu = (8.23 - 7.82) / (|p5| |u3|)
      u4, k = 2: tau'_2 = u4.p2 = 10.26 -> mu = (11.78 - 10.26) / (|p5| |u4|)   (u4.p4 = 10.84 is tau'_1)
      u1, k = 1: tau'_1 = u1.p3 = 10.02 -> mu = (1.89 - 10.02) / (|p5| |u1|)   (negative: not a member)
    A dropped exclusion (tau = 8.23 itself -> mu = 0), a dropped normalisation (mu = 0.41) or a wrong
    rank each fail here."""
    U, P = _t1()
    ip, hn = GOLD["hand_inner_products"], GOLD["hand_norms"]
    nrm = lambda s: np.sqrt(hn[s + "_sq"])  # noqa: E731
    cases = [(2, 1, ip["u3"]["p5"], ip["u3"]["p4"], "u3"), (3, 2, ip["u4"]["p5"], ip["u4"]["p2"], "u4"),
             (0, 1, ip["u1"]["p5"], ip["u1"]["p3"], "u1")]
    q = P[[4]]
    for i, k, g, tau, un in cases:
        want = (g - tau) / (nrm("p5") * nrm(un))
        mu = oracle.margins(U, P, q, np.array([[0, i]]), k)[0]
        assert abs(mu - want) < 1e-6, (un, k, mu, want)
    assert abs(oracle.margins(U, P, q, np.array([[0, 2]]), 1)[0] - 0.04481) < 5e-5   # VERDICT r1 figure


def test_margin_excludes_every_copy_of_q():
    """Two more bitwise copies of p5 in P change nothing (Def. 2 takes P u {q} as a set, R8/R9); a
    vector that differs from p5 in one ulp is a competitor and sets tau'_1 = its score."""
    U, P = _t1()
    q = P[[4]]
    P2 = np.concatenate([P, q, q])
    pairs = np.array([[0, 2], [0, 3]])
    assert np.array_equal(oracle.margins(U, P2, q, pairs, 1), oracle.margins(U, P, q, pairs, 1))
    near = q.copy()
    near[0, 1] = np.nextafter(near[0, 1], np.float32(0))      # 3.4 - 1 ulp: scores just below u.q
    P3 = np.concatenate([P, near])
    mu = oracle.margins(U, P3, q, pairs, 1)
    assert (mu > 0).all() and (mu < 1e-6).all()               # competitor now sits right under q


@pytest.mark.parametrize("seed", [50, 51, 52])
def test_margin_lists_equals_brute_force(seed):
    """orc_margin_lists (top-list form) equals orc_margin (scan of P) on every pair: queries from P,
    duplicated items (copies of q inside the list), fresh queries; k up to the list length - 1."""
    U, P = _inst(seed, 40, 30, 6, "skewed")
    P = np.concatenate([P, P[[2, 2, 5]]])                      # items 30, 31 copy item 2; 32 copies 5
    Qy = np.concatenate([P[[2, 5, 7]], _inst(seed + 7, 3, 1, 6)[0]])
    kk = 9
    vals, ids = oracle.topk(U, P, kk)
    pairs = np.array([(qi, i) for qi in range(Qy.shape[0]) for i in range(U.shape[0])])
    for k in (1, 4, 8):
        a = oracle.margins(U, P, Qy, pairs, k)
        b = oracle.margins_from_lists(U, P, Qy, vals, ids, pairs, k)
        assert np.array_equal(a, b), k


def test_sort_tie_order_ascending_id():
    """Reading R6 (P:279 says only 'descending'): equal norms keep ascending original ids.  Checked
    against numpy's stable lexsort on (-norm, id) (a library routine), on exact power-of-two norms."""
    X = np.zeros((9, 3), np.float32)
    X[:, 0] = [1, 2, 1, 4, 2, 1, 4, 0, 2]
    nrm = oracle.norms(X)
    perm = oracle.sort_by_norm_desc(nrm)
    assert perm.tolist() == [3, 6, 1, 4, 8, 0, 2, 5, 7]
    assert np.array_equal(perm, np.lexsort((np.arange(9), -nrm)))


def test_margin_sign_matches_membership_for_fresh_queries():
    """For q not in P, mu >= 0 <=> member (Def. 2 with reading R1)."""
    U, P = _inst(30, 25, 20, 8)
    Qy = _inst(31, 4, 1, 8)[0]
    mem = oracle.rkmips_naive(U, P, Qy, 3)
    pairs = np.array([(qi, i) for qi in range(4) for i in range(25)])
    mu = oracle.margins(U, P, Qy, pairs, 3)
    assert np.array_equal(mu >= 0, mem[pairs[:, 0], pairs[:, 1]])


def test_generator_deterministic_and_shaped():
    a = gen.make_workload(0)
    b = gen.make_workload(0)
    assert gen.sha256_arrays(a.U, a.P, a.Qy) == gen.sha256_arrays(b.U, b.P, b.Qy)
    assert a.U.shape == (2000, 50) and a.P.shape == (1000, 50) and a.Qy.shape == (100, 50)
    assert np.array_equal(a.Qy, a.P[a.q_item])
    c = gen.make_workload(1, n=1000, m=500, nq=10)
    assert abs(float(c.P.mean()) - 0.1) < 0.02   # item offset 0.1 per dim (BJ configs[1])


def test_topk_ties_by_ascending_item_id():
    """Reading R6 tie order: equal values list the lower item id first."""
    U, P = _inst(40, 6, 5, 4)
    P = np.concatenate([P, P[[3, 0, 3]]])           # ids 5, 6, 7 duplicate 3, 0, 3
    vals, ids = oracle.topk(U, P, 8)
    for i in range(6):
        for t in range(7):
            if vals[i, t] == vals[i, t + 1]:
                assert ids[i, t] < ids[i, t + 1]
    # every duplicate pair is adjacent and in id order
    S = U.astype(np.float64) @ P.astype(np.float64).T
    ref = np.lexsort((np.arange(8)[None].repeat(6, 0), -S), axis=1)
    assert np.array_equal(ids, ref)


def test_topk_ties_at_the_cut_keep_lower_id():
    """When the list is full, an equal value with a higher id must not displace the k-th."""
    u = np.array([[1.0, 0.0]], np.float32)
    P = np.array([[3, 0], [2, 1], [1, 5], [2, -1], [2, 7]], np.float32)   # scores 3, 2, 1, 2, 2
    vals, ids = oracle.topk(u, P, 2)
    assert ids[0].tolist() == [0, 1] and vals[0].tolist() == [3.0, 2.0]
