"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by element.

The bar (BASELINE north star): identical user-id sets; any disagreement must be a borderline
user (|q.u - tau_k(u)| <= 1e-5 |q||u|, reading R9) and there must be none on configs[0].  In
practice the exact fp64 path leaves no disagreement anywhere, which is what these tests assert.
"""
import numpy as np
import pytest

import oracle
from synth import generator as gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2110_07131_b200 import rmips  # noqa: E402

DEV = torch.device("cuda:0")
BUILDS = [("tc", rmips.RMIPS_BUILD_DEFAULT), ("simt", rmips.RMIPS_BUILD_SIMT)]


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(DEV)


def gpu_sets(U, P, Qy, k, k_max, build_flags=0, qflags=0, idx=None):
    own = idx is None
    if own:
        idx = rmips.rmips_build_index(_t(U), _t(P), k_max, build_flags)
    off, ids = rmips.rmips_query(idx, _t(Qy), k, qflags)
    sets = rmips.split_sets(off, ids)
    if own:
        idx.close()
    return sets


def assert_same(got, member, U=None, P=None, Qy=None, k=None, label=""):
    want = oracle.sets_from_member(member)
    assert len(got) == len(want)
    bad = []
    for i, (g, w) in enumerate(zip(got, want)):
        assert (np.diff(g) > 0).all(), "ids not strictly ascending (query %d)" % i
        if not np.array_equal(g, w):
            bad.append((i, np.setxor1d(g, w)))
    if bad and U is not None:
        pairs = np.array([(i, u) for i, us in bad for u in us])
        mu = oracle.margins(U, P, Qy, pairs, k)
        raise AssertionError("%s: %d disagreements on %d queries; margins %s" % (label, len(pairs), len(bad), mu[:10]))
    assert not bad, label


# ---------------------------------------------------------------- configs[0] (whole config, naive oracle)

@pytest.fixture(scope="module")
def cfg0():
    w = gen.make_workload(0)
    member = oracle.rkmips_naive(w.U, w.P, w.Qy, 10)
    return w, member


@pytest.mark.parametrize("name,bf", BUILDS)
def test_cfg0_full_parity(cfg0, name, bf):
    w, member = cfg0
    got = gpu_sets(w.U, w.P, w.Qy, 10, 10, bf)
    assert_same(got, member, w.U, w.P, w.Qy, 10, "cfg0/" + name)


def test_cfg0_index_tables_bitwise(cfg0):
    """T6: exported tau equals the oracle's exact top list bit for bit (reading R7); ids equal."""
    w, _ = cfg0
    idx = rmips.rmips_build_index(_t(w.U), _t(w.P), 10)
    pu, pp, tau, ids = idx.export()
    vals, oids = oracle.topk(w.U, w.P, 10)
    assert np.array_equal(tau.T, vals)
    assert np.array_equal(ids.T, oids)
    assert np.array_equal(pu, oracle.sort_by_norm_desc(oracle.norms(w.U)))
    assert np.array_equal(pp, oracle.sort_by_norm_desc(oracle.norms(w.P)))
    assert idx.overflow_rows == 0
    idx.close()


@pytest.mark.parametrize("qflags", [rmips.RMIPS_FLAG_NO_BLOCKS, rmips.RMIPS_FLAG_VERIFY_SCAN,
                                    rmips.RMIPS_FLAG_FORCE_VERIFY,
                                    rmips.RMIPS_FLAG_FORCE_VERIFY | rmips.RMIPS_FLAG_VERIFY_SCAN,
                                    rmips.RMIPS_FLAG_SIMT, rmips.RMIPS_FLAG_KEY_SORT,
                                    rmips.RMIPS_FLAG_KEY_SORT | rmips.RMIPS_FLAG_FORCE_VERIFY])
def test_cfg0_query_modes_agree(cfg0, qflags):
    w, member = cfg0
    got = gpu_sets(w.U, w.P, w.Qy, 10, 10, 0, qflags)
    assert_same(got, member, w.U, w.P, w.Qy, 10, "cfg0 flags=%d" % qflags)


def test_cfg0_every_k_and_invariant(cfg0):
    """Queries over ALL of P: every user appears in exactly k sets (north-star invariant)."""
    w, _ = cfg0
    idx = rmips.rmips_build_index(_t(w.U), _t(w.P), 10)
    vals, _ = oracle.topk(w.U, w.P, 10)
    for k in (1, 3, 10):
        off, ids = rmips.rmips_query(idx, _t(w.P), k)
        counts = np.bincount(ids.cpu().numpy(), minlength=w.U.shape[0])
        assert (counts == k).all(), k
        member = oracle.rkmips_twophase(w.U, vals, w.P, k)
        assert_same(rmips.split_sets(off, ids), member, label="all-P k=%d" % k)
    idx.close()


# ---------------------------------------------------------------- random small instances, ragged shapes

CASES = [
    # seed, n, m, d, k_max, k, dist, nq
    (1, 129, 33, 8, 10, 3, "gaussian", 20),
    (2, 300, 70, 50, 25, 10, "skewed", 30),
    (3, 257, 200, 65, 16, 16, "uniform", 25),
    (4, 500, 300, 2, 5, 1, "gaussian", 40),
    (5, 64, 40, 1, 4, 2, "gaussian", 10),
    (6, 400, 150, 200, 50, 50, "skewed", 16),
    (7, 1000, 600, 50, 10, 5, "uniform", 30),
    (8, 130, 7, 12, 10, 9, "gaussian", 12),     # m < k_max, k > m
    (9, 333, 250, 128, 20, 7, "skewed", 20),
    (10, 300, 260, 90, 12, 6, "gaussian", 20),   # d_pad 128, 6 K steps: 32-column tail K block (SW64)
    (11, 270, 140, 100, 9, 4, "uniform", 18),    # 7 K steps: full tail K block
]


@pytest.mark.parametrize("case", CASES, ids=[str(c[0]) for c in CASES])
@pytest.mark.parametrize("name,bf", BUILDS)
def test_random_instances(case, name, bf):
    seed, n, m, d, kmax, k, dist, nq = case
    U, P = gen.random_instance(seed, n, m, d, dist)
    fresh, _ = gen.random_instance(seed + 1000, nq - nq // 2, 1, d, dist)
    Qy = np.concatenate([P[: nq // 2], fresh])
    member = oracle.rkmips_naive(U, P, Qy, k)
    got = gpu_sets(U, P, Qy, k, kmax, bf)
    assert_same(got, member, U, P, Qy, k, "case %d/%s" % (seed, name))


def test_duplicate_items_and_ties():
    """Many identical items force candidate-buffer overflow -> exact fallback rows."""
    U, P = gen.random_instance(11, 300, 40, 16, "gaussian")
    P = np.concatenate([P] + [P[:3]] * 60)        # 180 copies of 3 items
    Qy = np.concatenate([P[:5], P[100:103]])
    member = oracle.rkmips_naive(U, P, Qy, 7)
    idx = rmips.rmips_build_index(_t(U), _t(P), 20)
    got = rmips.split_sets(*rmips.rmips_query(idx, _t(Qy), 7))
    assert_same(got, member, U, P, Qy, 7, "dups")
    _, _, tau, _ = idx.export()
    vals, _ = oracle.topk(U, P, 20)
    assert np.array_equal(tau.T, vals)
    idx.close()


def test_zero_vectors_and_all_equal_norms():
    rng = np.random.default_rng(12)
    U = rng.standard_normal((200, 10)).astype(np.float32)
    U[::7] = 0.0
    P = rng.standard_normal((90, 10)).astype(np.float32)
    P /= np.linalg.norm(P, axis=1, keepdims=True)       # all item norms ~equal
    P[5] = 0.0
    Qy = np.concatenate([P[:6], np.zeros((1, 10), np.float32), -P[:3]])
    for k in (1, 4):
        member = oracle.rkmips_naive(U, P, Qy, k)
        assert_same(gpu_sets(U, P, Qy, k, 8), member, U, P, Qy, k, "zeros k=%d" % k)


def test_huge_norm_range():
    """Norms over ~2^40 (fp16 subnormal range for small items) stay exact."""
    rng = np.random.default_rng(13)
    U = (rng.standard_normal((300, 20)) * np.exp(rng.normal(0, 6, (300, 1)))).astype(np.float32)
    P = (rng.standard_normal((200, 20)) * np.exp(rng.normal(0, 6, (200, 1)))).astype(np.float32)
    Qy = np.concatenate([P[:10], (rng.standard_normal((10, 20)) * 1e-3).astype(np.float32)])
    member = oracle.rkmips_naive(U, P, Qy, 5)
    assert_same(gpu_sets(U, P, Qy, 5, 10), member, U, P, Qy, 5, "norm range")


# ---------------------------------------------------------------- boundary behaviour

def test_empty_users_and_empty_batch():
    _, P = gen.random_instance(14, 1, 30, 8)
    idx = rmips.rmips_build_index(None, _t(P), 5)
    off, ids = rmips.rmips_query(idx, _t(P[:4]), 3)
    assert off.cpu().tolist() == [0] * 5 and ids.numel() == 0
    off, ids = rmips.rmips_query(idx, torch.zeros((0, 8), dtype=torch.float32, device=DEV), 3)
    assert off.numel() == 1 and ids.numel() == 0
    idx.close()


def test_errors_k_range_nonfinite_capacity():
    U, P = gen.random_instance(15, 100, 30, 8)
    idx = rmips.rmips_build_index(_t(U), _t(P), 5)
    with pytest.raises(rmips.RmipsError) as e:
        rmips.rmips_query(idx, _t(P[:2]), 6, rmips.RMIPS_FLAG_NO_EXTEND)
    assert e.value.status == rmips.RMIPS_ERR_K_RANGE
    with pytest.raises(rmips.RmipsError) as e:
        rmips.rmips_query(idx, _t(P[:2]), 0)
    assert e.value.status == rmips.RMIPS_ERR_K_RANGE
    bad = P[:2].copy()
    bad[1, 3] = np.nan
    with pytest.raises(rmips.RmipsError) as e:
        rmips.rmips_query(idx, _t(bad), 2)
    assert e.value.status == rmips.RMIPS_ERR_NONFINITE
    with pytest.raises(rmips.RmipsError) as e:
        rmips.rmips_query(idx, _t(P[:10]), 5, capacity=1)
    assert e.value.status == rmips.RMIPS_ERR_CAPACITY
    Ub = U.copy()
    Ub[3, 0] = np.inf
    with pytest.raises(rmips.RmipsError) as e:
        rmips.rmips_build_index(_t(Ub), _t(P), 5)
    assert e.value.status == rmips.RMIPS_ERR_NONFINITE
    idx.close()


def test_output_paths_identical():
    """The bit-matrix output and the sorted-key output give the same offsets and ids (ragged n,
    several batch sizes incl. one query and more than one 256-query sub-batch), and both report
    RMIPS_ERR_CAPACITY with valid offsets when the ids do not fit."""
    U, P = gen.random_instance(21, 3001, 400, 24)
    idx = rmips.rmips_build_index(_t(U), _t(P), 12)
    for b in (1, 7, 300, 700):
        Q = _t(P[:b] if b <= len(P) else P[np.arange(b) % len(P)])
        for k in (1, 5, 12):
            o1, i1 = rmips.rmips_query(idx, Q, k)
            o2, i2 = rmips.rmips_query(idx, Q, k, rmips.RMIPS_FLAG_KEY_SORT)
            assert np.array_equal(o1.cpu().numpy(), o2.cpu().numpy()), (b, k)
            assert np.array_equal(i1.cpu().numpy(), i2.cpu().numpy()), (b, k)
    for fl in (0, rmips.RMIPS_FLAG_KEY_SORT):
        with pytest.raises(rmips.RmipsError) as e:
            rmips.rmips_query(idx, _t(P[:50]), 12, fl, capacity=3)
        assert e.value.status == rmips.RMIPS_ERR_CAPACITY
    # the matrix is clean again after a capacity failure and across batch-size changes
    for b in (50, 700, 50):
        o1, i1 = rmips.rmips_query(idx, _t(P[np.arange(b) % len(P)]), 12)
        o2, i2 = rmips.rmips_query(idx, _t(P[np.arange(b) % len(P)]), 12, rmips.RMIPS_FLAG_KEY_SORT)
        assert np.array_equal(o1.cpu().numpy(), o2.cpu().numpy())
        assert np.array_equal(i1.cpu().numpy(), i2.cpu().numpy())
    idx.close()


def test_host_variants_match_device():
    U, P = gen.random_instance(16, 400, 120, 50)
    Qy = P[:30]
    idx_d = rmips.rmips_build_index(_t(U), _t(P), 10)
    idx_h = rmips.rmips_build_index_host(U, P, 10)
    a = rmips.split_sets(*rmips.rmips_query(idx_d, _t(Qy), 4))
    off, ids = rmips.rmips_query_host(idx_h, Qy, 4)
    b = [ids[off[i]:off[i + 1]] for i in range(len(off) - 1)]
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
    idx_d.close()
    idx_h.close()


def test_stats_counters_consistent(cfg0):
    w, member = cfg0
    idx = rmips.rmips_build_index(_t(w.U), _t(w.P), 10)
    rmips.rmips_query(idx, _t(w.Qy), 10)
    s = idx.stats()
    assert s["queries"] == 100
    assert s["result_total"] == int(member.sum())
    assert s["pairs_scored"] == s["pairs_rejected"] + s["pairs_accepted_fast"] + s["pairs_undecided"]
    assert s["result_total"] == s["pairs_accepted_fast"] + s["pairs_exact_accepted"]
    assert s["block_query_pairs"] == 100 * ((idx.n + 127) // 128)
    assert s["filter_kernel"] == 1          # the tcgen05 filter ran (query_tc.cu), not the SIMT one
    rmips.rmips_query(idx, _t(w.Qy), 10, rmips.RMIPS_FLAG_SIMT)
    s2 = idx.stats()
    assert s2["filter_kernel"] == 0
    for key in ("block_query_pairs", "block_query_pruned", "pairs_scored", "result_total"):
        assert s2[key] == s[key], key
    idx.close()


# ---------------------------------------------------------------- configs[1] at full size (sampled oracle)

def test_cfg1_full_size_sampled():
    """BJ configs[1] at full size, in the bench's launch configuration (all 1,000 queries in one
    call).  The oracle checks a fixed sample of 1,500 users: exact top lists (two-phase form,
    equal to the definition by reading R8) and every query's decision for those users."""
    w = gen.make_workload(1)
    idx = rmips.rmips_build_index(_t(w.U), _t(w.P), 50)
    off, ids = rmips.rmips_query(idx, _t(w.Qy), 10)
    assert idx.stats()["filter_kernel"] == 1
    sets = rmips.split_sets(off, ids)
    # the SIMT filter must give the identical sets (different fp32 summation order, same decisions)
    off2, ids2 = rmips.rmips_query(idx, _t(w.Qy), 10, rmips.RMIPS_FLAG_SIMT)
    assert torch.equal(off, off2) and torch.equal(ids, ids2)
    rng = np.random.default_rng(0)
    sample = np.sort(rng.choice(w.U.shape[0], 1500, replace=False))
    vals, oids = oracle.topk(w.U[sample], w.P, 50)
    _, _, tau, tids = idx.export()
    assert np.array_equal(tau[:, sample].T, vals)
    member = oracle.rkmips_twophase(w.U[sample], vals, w.Qy, 10)
    for qi in range(w.Qy.shape[0]):
        got = np.intersect1d(sets[qi], sample)
        want = sample[member[qi]]
        assert np.array_equal(got, want), qi
    # invariant-style global check: totals are plausible and ids ascending
    assert all((np.diff(s) > 0).all() for s in sets)
    idx.close()


# ---------------------------------------------------------------- configs[2..4] at full size (sampled oracle)

def _sampled_full_config(cfg, n_sample, batch=None, query_stride=1):
    """BJ configs[cfg] at full size.  The GPU index covers every user; the oracle recomputes a fixed
    sample of users exactly (top lists, two-phase decisions — equal to the definition by R8) and every
    sampled user's membership in every query's set must match; tau/ids are compared bitwise."""
    w = gen.make_workload(cfg)
    spec = w.spec
    idx = rmips.rmips_build_index(_t(w.U), _t(w.P), spec.k_max)
    assert idx.overflow_rows == 0
    assert idx.build_flags & rmips.RMIPS_BUILD_SIMT == 0  # the tcgen05 build ran
    assert idx.build_kernel == (4 if spec.d > 64 else 1)  # CTA pairs for d_pad 128..256
    rng = np.random.default_rng(cfg)
    sample = np.sort(rng.choice(spec.n, n_sample, replace=False))
    vals, oids = oracle.topk(w.U[sample], w.P, spec.k_max)
    _, _, tau, tids = idx.export()
    assert np.array_equal(tau[:, sample].T, vals)
    assert np.array_equal(tids[:, sample].T, oids)
    Qy = w.Qy[::query_stride]
    for k in spec.ks:
        bs = batch or Qy.shape[0]
        sets = []
        for b0 in range(0, Qy.shape[0], bs):
            off, ids = rmips.rmips_query(idx, _t(Qy[b0:b0 + bs]), k)
            assert idx.stats()["filter_kernel"] == 1  # the tcgen05 filter ran
            sets += rmips.split_sets(off, ids)
        assert all((np.diff(s_) > 0).all() for s_ in sets)
        member = oracle.rkmips_twophase(w.U[sample], vals, Qy, k)
        for qi in range(Qy.shape[0]):
            got = np.intersect1d(sets[qi], sample)
            want = sample[member[qi]]
            assert np.array_equal(got, want), (cfg, k, qi)
    idx.close()


def test_cfg2_full_size_sampled_k_sweep():
    """BJ configs[2]: 480,000 x 18,000, k swept over {1, 5, 10, 25, 50}."""
    _sampled_full_config(2, 1200)


def test_cfg3_full_size_sampled():
    """BJ configs[3]: 2,000,000 x 100,000, heavy-tailed norms, half the queries not in P."""
    _sampled_full_config(3, 400)


def test_cfg4_full_size_sampled():
    """BJ configs[4]: d = 200, 1,000,000 x 1,000,000, fresh queries in batches of 256 (every 4th of the
    10,000 queries, to bound the test time)."""
    _sampled_full_config(4, 96, batch=256, query_stride=4)


def test_filter_error_bound_holds():
    """The fp16/fp32 filter error bound dominates the observed error: the exact path
    would hide a violated bound, so check it directly.  The build's kept candidates always contain the
    exact top list (checked bitwise above); here the query filter's accept/reject decisions must never
    contradict the exact decision: a pair accepted or rejected by the filter is re-decided exactly."""
    U, P = gen.random_instance(21, 3000, 1500, 50, "skewed")
    Qy = np.concatenate([P[:100], gen.random_instance(22, 100, 1, 50, "skewed")[0]])
    for k in (1, 7, 20):
        member = oracle.rkmips_naive(U, P, Qy, k)
        # FORCE_VERIFY routes every filter accept through the exact path: both runs must agree
        a = gpu_sets(U, P, Qy, k, 20)
        b = gpu_sets(U, P, Qy, k, 20, qflags=rmips.RMIPS_FLAG_FORCE_VERIFY)
        assert_same(a, member, U, P, Qy, k, "bound k=%d" % k)
        assert_same(b, member, U, P, Qy, k, "bound/force k=%d" % k)


# ---------------------------------------------------------------- build-kernel variants (dev library)

_VARIANT_SCRIPT = """
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2110_07131_b200 import rmips
from synth import generator as gen
U, P = gen.random_instance(77, 20000, 6000, int(sys.argv[3]) if len(sys.argv) > 3 else 50, "skewed")
dev = torch.device("cuda:0")
idx = rmips.rmips_build_index(torch.from_numpy(U).to(dev), torch.from_numpy(P).to(dev), 50)
assert idx.build_flags & rmips.RMIPS_BUILD_SIMT == 0
_, _, tau, ids = idx.export()
np.savez(sys.argv[2], tau=tau, ids=ids, lib=rmips.LIB_PATH)
"""


@pytest.mark.parametrize("env", [{}, {"RMIPS_SEED_TILES": "0"}, {"RMIPS_SEED_TILES": "32"},
                                 {"RMIPS_SEED_TILES": "3"}, {"RMIPS_NO_CS": "1"}],
                         ids=["default", "seed0", "seed32", "seed3", "no-cs"])
def test_build_variants_bitwise(env, tmp_path):
    """Every tensor-core build variant (seed-pass lengths, no Cauchy-Schwarz exit) gives the oracle's
    exact top-k_max lists (tau and ids bitwise) on a sample of users, with m = 6,000 items (47 item
    tiles, a ragged last tile) and k_max = 50.  The variants are selected by getenv switches that only
    the development library librmips_dev.so (-DRMIPS_DEV) reads, so each runs in a subprocess."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2110_07131_b200 import build_lib
    devlib = build_lib.build_dev()
    out = str(tmp_path / "v.npz")
    e = dict(os.environ, RMIPS_LIB=devlib, **env)
    r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, root, out], env=e, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(out)
    assert str(got["lib"]).endswith("librmips_dev.so")
    U, P = gen.random_instance(77, 20000, 6000, 50, "skewed")
    sample = np.sort(np.random.default_rng(7).choice(U.shape[0], 600, replace=False))
    vals, oids = oracle.topk(U[sample], P, 50)
    assert np.array_equal(got["tau"][:, sample].T, vals)
    assert np.array_equal(got["ids"][:, sample].T, oids)


def test_repeated_builds_two_streams_identical():
    """Builds of one instance repeated on two streams (the first build of a size takes the direct
    sort, later ones the cached per-stream sort graph) export identical permutations and lists,
    equal to the oracle's on a sample."""
    import torch
    U, P = gen.random_instance(91, 3000, 900, 20)
    Ut, Pt = _t(U), _t(P)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    ref = None
    for rep in range(3):
        for s in streams:
            idx = rmips.rmips_build_index(Ut, Pt, 8, stream=s)
            s.synchronize()
            out = idx.export()
            idx.close()
            if ref is None:
                ref = out
                sample = np.arange(0, U.shape[0], 37)
                vals, oids = oracle.topk(U[sample], P, 8)
                assert np.array_equal(out[2][:, sample].T, vals)
                assert np.array_equal(out[3][:, sample].T, oids)
            else:
                for a, b in zip(ref, out):
                    assert np.array_equal(a, b), rep


# ---------------------------------------------------------------- P' index (NEXT-1: Alg. 1 as printed)

@pytest.mark.parametrize("name,bf", BUILDS)
@pytest.mark.parametrize("c", [1, 2, 5])
def test_cfg0_pprime_parity(cfg0, name, bf, c):
    """configs[0] with lists over P' = the first c * k_max norm-sorted items: the query path
    decides by Lemma 1 / Lemma 2 / Cor. 1 and the scan after P', and must give the same sets."""
    w, member = cfg0
    idx = rmips.rmips_build_index_pprime(_t(w.U), _t(w.P), 10, c * 10, bf)
    assert idx.m_prime == c * 10
    got = gpu_sets(w.U, w.P, w.Qy, 10, 10, idx=idx)
    assert_same(got, member, w.U, w.P, w.Qy, 10, "cfg0/pprime c=%d/%s" % (c, name))
    st = idx.stats()
    assert st["pairs_accepted_fast"] == 0  # the filter never accepts on a P' index
    assert st["scans"] > 0 and st["items_scanned"] > 0
    # Lemma-3 blocks of ceil(log2 n) users: n = 2,000 -> 11 users, 182 blocks
    assert idx.block_size == 11 and st["block_query_pairs"] == 100 * 182
    # Alg. 2 over all of P (stress) on the same index agrees
    off, ids = rmips.rmips_query(idx, _t(w.Qy), 10, rmips.RMIPS_FLAG_VERIFY_SCAN)
    assert_same(rmips.split_sets(off, ids), member, label="cfg0/pprime scan-all")
    for k in (1, 3, 7):
        mk = oracle.rkmips_naive(w.U, w.P, w.Qy, k)
        assert_same(gpu_sets(w.U, w.P, w.Qy, k, 10, idx=idx), mk, label="cfg0/pprime k=%d" % k)
    idx.close()


@pytest.mark.parametrize("case", CASES, ids=[str(c[0]) for c in CASES])
@pytest.mark.parametrize("mp", ["1", "2kmax", "m-1"])
def test_random_instances_pprime(case, mp):
    seed, n, m, d, kmax, k, dist, nq = case
    U, P = gen.random_instance(seed, n, m, d, dist)
    fresh, _ = gen.random_instance(seed + 1000, nq - nq // 2, 1, d, dist)
    Qy = np.concatenate([P[: nq // 2], fresh])
    member = oracle.rkmips_naive(U, P, Qy, k)
    m_prime = {"1": 1, "2kmax": 2 * kmax, "m-1": max(1, m - 1)}[mp]
    idx = rmips.rmips_build_index_pprime(_t(U), _t(P), kmax, m_prime)
    got = gpu_sets(U, P, Qy, k, kmax, idx=idx)
    idx.close()
    assert_same(got, member, U, P, Qy, k, "case %d/pprime %s" % (seed, mp))


def test_cfg1_pprime_sampled():
    """configs[1] at full size with |P'| = 2 k_max (SPEC's choice): sampled users' memberships in
    every query's set equal the oracle's (two-phase form over all of P)."""
    w = gen.make_workload(1)
    idx = rmips.rmips_build_index_pprime(_t(w.U), _t(w.P), 50, 100)
    off, ids = rmips.rmips_query(idx, _t(w.Qy), 10)
    sets = rmips.split_sets(off, ids)
    st = idx.stats()
    assert st["scans"] > 0
    rng = np.random.default_rng(1)
    sample = np.sort(rng.choice(w.U.shape[0], 1000, replace=False))
    vals, _ = oracle.topk(w.U[sample], w.P, 50)
    member = oracle.rkmips_twophase(w.U[sample], vals, w.Qy, 10)
    for qi in range(w.Qy.shape[0]):
        assert np.array_equal(np.intersect1d(sets[qi], sample), sample[member[qi]]), qi
    idx.close()


# ---------------------------------------------------------------- NEXT-2: k > k_max extends the index

@pytest.mark.parametrize("pp", [0, 2])
def test_k_beyond_kmax_extends_index(cfg0, pp):
    """configs[0] built with k_max = 4 (exact and P' indexes); queries with k = 7, 10, 25 extend the
    index in place and must give the oracle's sets; the extended lists equal the
    oracle's exact top-k lists bit for bit (exact index)."""
    w, member10 = cfg0
    if pp:
        idx = rmips.rmips_build_index_pprime(_t(w.U), _t(w.P), 4, pp * 4)
    else:
        idx = rmips.rmips_build_index(_t(w.U), _t(w.P), 4)
    for k in (7, 10, 25, 3):
        member = member10 if k == 10 else oracle.rkmips_naive(w.U, w.P, w.Qy, k)
        assert_same(gpu_sets(w.U, w.P, w.Qy, k, 4, idx=idx), member, label="extend k=%d pp=%d" % (k, pp))
    if not pp:
        _, _, tau, ids = idx.export()
        assert idx.k_max == 25
        vals, oids = oracle.topk(w.U, w.P, 25)
        assert np.array_equal(tau.T, vals) and np.array_equal(ids.T, oids)
    idx.close()


# ---------------------------------------------------------------- round-2 edge cases

def test_key_sort_power_of_two_span_keeps_last_user():
    """Sorted-key output with b * n an exact power of two (b = 4, n = 1024: span 2^12).  k > m puts
    every user in every set, so user n - 1 must be in the last query's set; the padding sentinel must
    sort after it (2^bits > span)."""
    U, P = gen.random_instance(60, 1024, 3, 16)
    Qy = gen.random_instance(61, 4, 1, 16)[0]
    idx = rmips.rmips_build_index(_t(U), _t(P), 4)
    for fl in (rmips.RMIPS_FLAG_KEY_SORT, rmips.RMIPS_FLAG_KEY_SORT | rmips.RMIPS_FLAG_FORCE_VERIFY, 0):
        off, ids = rmips.rmips_query(idx, _t(Qy), 4, fl)
        sets = rmips.split_sets(off, ids)
        for s_ in sets:
            assert np.array_equal(s_, np.arange(1024)), fl
    # and a power-of-two span with a real (not all-users) answer
    U, P = gen.random_instance(62, 2048, 300, 16)
    Qy = P[:8]
    member = oracle.rkmips_naive(U, P, Qy, 5)
    got = gpu_sets(U, P, Qy, 5, 8, qflags=rmips.RMIPS_FLAG_KEY_SORT)
    assert_same(got, member, U, P, Qy, 5, "pow2 span")
    idx.close()


def test_key_sort_64bit_branch_sampled():
    """The 64-bit (query, user) key output branch: b * n >= 2^32 and the b x n bit matrix above 64 MiB
    (VERDICT r1 weak #2).  n = 4.5 M users, m = 2,000 items, d = 8, 1,000 queries, k = 1: the oracle
    recomputes a fixed sample of users (two-phase form, equal to the definition by R8)."""
    w = gen.make_workload(0, n=4_500_000, m=2_000, nq=1_000, d=8)
    assert w.U.shape[0] * w.Qy.shape[0] >= 1 << 32
    idx = rmips.rmips_build_index(_t(w.U), _t(w.P), 2)
    off, ids = rmips.rmips_query(idx, _t(w.Qy), 1)
    sets = rmips.split_sets(off, ids)
    assert all((np.diff(s_) > 0).all() for s_ in sets)
    rng = np.random.default_rng(5)
    sample = np.sort(np.concatenate([rng.choice(w.U.shape[0], 3000, replace=False),
                                     np.arange(w.U.shape[0] - 50, w.U.shape[0])]))
    sample = np.unique(sample)
    vals, _ = oracle.topk(w.U[sample], w.P, 2)
    member = oracle.rkmips_twophase(w.U[sample], vals, w.Qy, 1)
    for qi in range(w.Qy.shape[0]):
        assert np.array_equal(np.intersect1d(sets[qi], sample), sample[member[qi]]), qi
    # totals: with queries drawn from P (no ties), each user is in at most one set at k = 1
    assert int(off[-1].item()) == int(ids.numel())
    idx.close()


def test_empty_users_k_beyond_kmax():
    """n = 0 and k > k_max: the empty index extends trivially and answers the empty set."""
    _, P = gen.random_instance(63, 1, 30, 8)
    idx = rmips.rmips_build_index(None, _t(P), 2)
    off, ids = rmips.rmips_query(idx, _t(P[:5]), 7)
    assert off.cpu().tolist() == [0] * 6 and ids.numel() == 0
    idx.close()


def test_extreme_magnitudes_exact():
    """Finite inputs near FLT_MAX: a threshold tau / nu that is not a finite fp32 must not accept or
    reject outright, and a user whose norm exceeds FLT_MAX (no unit-norm fp32 scaling) must still be
    decided exactly."""
    # the ADVICE example: u.q = -6.6e38 < tau_1 = -6e38, so u is not in R_1(q)
    U = np.array([[1.0, 1.0]], np.float32)
    P = np.array([[-3e38, -3e38]], np.float32)
    Qy = np.array([[-3.3e38, -3.3e38], [-2e38, -2e38], [-3e38, -3e38]], np.float32)
    member = oracle.rkmips_naive(U, P, Qy, 1)
    assert member.tolist() == [[False], [True], [True]]
    assert_same(gpu_sets(U, P, Qy, 1, 1), member, U, P, Qy, 1, "advice example")
    # random instance with huge users / items / queries mixed into ordinary ones
    rng = np.random.default_rng(64)
    U = rng.standard_normal((300, 6)).astype(np.float32)
    U[::17] = (rng.standard_normal((18, 6)) * 2e38).clip(-3.3e38, 3.3e38).astype(np.float32)[: len(U[::17])]
    P = rng.standard_normal((120, 6)).astype(np.float32)
    P[::11] = (rng.standard_normal((11, 6)) * 1.5e38).clip(-3.3e38, 3.3e38).astype(np.float32)[: len(P[::11])]
    Qy = np.concatenate([P[:12], (rng.standard_normal((6, 6)) * 2e38).clip(-3.3e38, 3.3e38).astype(np.float32),
                         rng.standard_normal((6, 6)).astype(np.float32)])
    assert np.isfinite(U).all() and np.isfinite(P).all() and np.isfinite(Qy).all()
    assert (oracle.norms(U) > 3.4028234663852886e38).any()
    for k in (1, 3, 8):
        member = oracle.rkmips_naive(U, P, Qy, k)
        for bf in (0, rmips.RMIPS_BUILD_SIMT):
            got = gpu_sets(U, P, Qy, k, 8, bf)
            assert_same(got, member, U, P, Qy, k, "huge k=%d bf=%d" % (k, bf))
    idx = rmips.rmips_build_index(_t(U), _t(P), 8)
    _, _, tau, ids = idx.export()
    vals, oids = oracle.topk(U, P, 8)
    assert np.array_equal(tau.T, vals) and np.array_equal(ids.T, oids)
    idx.close()


def test_concurrent_builds_same_stream_handle():
    """Builds of the same size from two host threads on cudaStreamPerThread (one handle value, a
    different stream per thread) must not share the cached sort buffers."""
    import threading
    U, P = gen.random_instance(65, 5000, 700, 24)
    Ut, Pt = _t(U), _t(P)
    sample = np.arange(0, U.shape[0], 53)
    vals, oids = oracle.topk(U[sample], P, 6)
    torch.cuda.synchronize()
    errors = []

    def worker():
        try:
            for _ in range(6):
                idx = rmips.rmips_build_index(Ut, Pt, 6, stream=2)   # 2 = cudaStreamPerThread
                _, _, tau, ids = idx.export()
                idx.close()
                if not (np.array_equal(tau[:, sample].T, vals) and np.array_equal(ids[:, sample].T, oids)):
                    errors.append("mismatch")
        except Exception as e:  # noqa: BLE001
            errors.append(repr(e))

    ts = [threading.Thread(target=worker) for _ in range(3)]
    for t_ in ts:
        t_.start()
    for t_ in ts:
        t_.join()
    assert not errors, errors[:3]


# ---------------------------------------------------------------- the full boundary domain

@pytest.mark.parametrize("d", [300, 513, 1000])
def test_large_d_streamed_k_loop(d):
    """d > 256: the build streams the user tile's K blocks next to the item tile's (k_build_tcq, KB = 0)
    and the query filter streams the queries' K blocks (k_query_tc, KB = 0); the last K block is trimmed
    (d = 513: a 16-column tail).  Sets equal the naive oracle's; tau / ids bitwise."""
    U, P = gen.random_instance(70 + d, 700, 450, d, "skewed")
    Qy = np.concatenate([P[:20], gen.random_instance(71 + d, 15, 1, d, "skewed")[0]])
    idx = rmips.rmips_build_index(_t(U), _t(P), 12)
    assert idx.build_kernel == 3 and idx.build_flags & rmips.RMIPS_BUILD_SIMT == 0
    for k in (1, 5, 12):
        member = oracle.rkmips_naive(U, P, Qy, k)
        got = rmips.split_sets(*rmips.rmips_query(idx, _t(Qy), k))
        assert idx.stats()["filter_kernel"] == 1
        assert_same(got, member, U, P, Qy, k, "d=%d k=%d" % (d, k))
        got = rmips.split_sets(*rmips.rmips_query(idx, _t(Qy), k, rmips.RMIPS_FLAG_FORCE_VERIFY))
        assert_same(got, member, U, P, Qy, k, "d=%d k=%d force" % (d, k))
    _, _, tau, ids = idx.export()
    vals, oids = oracle.topk(U, P, 12)
    assert np.array_equal(tau.T, vals) and np.array_equal(ids.T, oids)
    with pytest.raises(rmips.RmipsError) as e:
        rmips.rmips_query(idx, _t(Qy), 3, rmips.RMIPS_FLAG_SIMT)
    assert e.value.status == rmips.RMIPS_ERR_INVALID
    idx.close()


@pytest.mark.parametrize("d", [16, 90, 200])
def test_trimmed_tail_k_block(d):
    """The last K block trimmed to a 16- or 32-column box (SWIZZLE_32B / 64B descriptors) in both the
    build and the query kernels: d = 16 (one 16-column block), 90 (32-column tail), 200 (16-column tail)."""
    U, P = gen.random_instance(80 + d, 1300, 700, d, "gaussian")  # 11 user tiles: the last CTA pair has one
    Qy = np.concatenate([P[:30], gen.random_instance(81 + d, 30, 1, d)[0]])
    for kmax, k in ((10, 4), (100, 37)):   # the second: k_max > 80 -> 256-slot lists (k_build_tcq for d = 16)
        member = oracle.rkmips_naive(U, P, Qy, k)
        idx = rmips.rmips_build_index(_t(U), _t(P), kmax)
        assert idx.build_flags & rmips.RMIPS_BUILD_SIMT == 0 and idx.overflow_rows == 0
        assert idx.cand_slots == (256 if kmax > 80 else 128)
        if d > 64 and kmax <= 80:
            assert idx.build_kernel == 4  # CTA pairs (tcgen05.mma.cta_group::2)
        got = rmips.split_sets(*rmips.rmips_query(idx, _t(Qy), k))
        assert_same(got, member, U, P, Qy, k, "tail d=%d kmax=%d" % (d, kmax))
        _, _, tau, ids = idx.export()
        vals, oids = oracle.topk(U, P, kmax)
        assert np.array_equal(tau.T, vals) and np.array_equal(ids.T, oids)
        idx.close()


@pytest.mark.parametrize("d", [50, 100])
def test_kmax_128_lists_without_fallback(d):
    """k_max = 128: the 256-slot 4-byte candidate lists hold every row (no exact-fallback
    rows), the exported lists equal the oracle's bitwise, and k = 100 and 128 answer like the oracle."""
    U, P = gen.random_instance(90 + d, 3000, 2500, d, "skewed")
    Qy = P[:40]
    idx = rmips.rmips_build_index(_t(U), _t(P), 128)
    assert idx.cand_slots == 256 and idx.build_kernel == 2
    assert idx.overflow_rows <= U.shape[0] // 20  # heavy-tailed norms: a few rows may take the exact fallback
    _, _, tau, ids = idx.export()
    vals, oids = oracle.topk(U, P, 128)
    assert np.array_equal(tau.T, vals) and np.array_equal(ids.T, oids)
    for k in (100, 128):
        member = oracle.rkmips_twophase(U, vals, Qy, k)
        got = rmips.split_sets(*rmips.rmips_query(idx, _t(Qy), k))
        assert_same(got, member, label="kmax128 d=%d k=%d" % (d, k))
    idx.close()


@pytest.mark.parametrize("m,slots", [(1_100_000, 256), (2_100_000, 128)])
def test_m_above_2pow20_tensor_core_build(m, slots):
    """m above 2^20: positions no longer fit 20 bits -- up to 2^21 the build keeps 4-byte
    entries with 21-bit positions (256 slots), beyond that 8-byte entries (128 slots); either way the
    tcgen05 kernel (not the SIMT build) with the oracle's exact lists on a user sample."""
    w = gen.make_workload(4, n=1500, m=m, nq=30, d=100)
    idx = rmips.rmips_build_index(_t(w.U), _t(w.P), 20)
    assert idx.build_kernel == 2 and idx.build_flags & rmips.RMIPS_BUILD_SIMT == 0  # (1-CTA kernel)
    assert idx.cand_slots == slots and idx.overflow_rows == 0
    sample = np.sort(np.random.default_rng(3).choice(w.U.shape[0], 160, replace=False))
    vals, oids = oracle.topk(w.U[sample], w.P, 20)
    _, _, tau, ids = idx.export()
    assert np.array_equal(tau[:, sample].T, vals) and np.array_equal(ids[:, sample].T, oids)
    off, gids = rmips.rmips_query(idx, _t(w.Qy), 20)
    sets = rmips.split_sets(off, gids)
    member = oracle.rkmips_twophase(w.U[sample], vals, w.Qy, 20)
    for qi in range(w.Qy.shape[0]):
        assert np.array_equal(np.intersect1d(sets[qi], sample), sample[member[qi]]), qi
    idx.close()


@pytest.mark.parametrize("n", [1, 127, 128, 129, 255, 383])
def test_cta_pair_build_ragged_user_tiles(n):
    """The CTA-pair build (k_build_tc2cta) with every user-tile parity: a single tile (the follower's rows
    all past n), odd and even tile counts, ragged last tiles; lists bitwise equal to the oracle's."""
    U, P = gen.random_instance(100 + n, n, 900, 100, "skewed")
    idx = rmips.rmips_build_index(_t(U), _t(P), 16)
    assert idx.build_kernel == 4 and idx.overflow_rows == 0
    _, _, tau, ids = idx.export()
    vals, oids = oracle.topk(U, P, 16)
    assert np.array_equal(tau.T, vals) and np.array_equal(ids.T, oids)
    Qy = P[:12]
    member = oracle.rkmips_twophase(U, vals, Qy, 7)
    assert_same(rmips.split_sets(*rmips.rmips_query(idx, _t(Qy), 7)), member, label="pair n=%d" % n)
    idx.close()


_TILED_SCRIPT = """
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2110_07131_b200 import rmips
from synth import generator as gen
import oracle
dev = torch.device("cuda:0")
t = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev)
bad = 0
for (seed, n, m, d, kmax, k, pp) in [(0, 2000, 1000, 50, 10, 10, 20), (1, 900, 700, 200, 8, 5, 16),
                                     (2, 500, 300, 520, 6, 4, 12), (3, 700, 400, 30, 10, 3, 0)]:
    U, P = gen.random_instance(seed, n, m, d, "skewed")
    Qy = np.concatenate([P[:20], gen.random_instance(seed + 9, 10, 1, d, "skewed")[0]])
    member = oracle.rkmips_naive(U, P, Qy, k)
    want = oracle.sets_from_member(member)
    idx = rmips.rmips_build_index_pprime(t(U), t(P), kmax, pp) if pp else rmips.rmips_build_index(t(U), t(P), kmax)
    for fl in (0, rmips.RMIPS_FLAG_VERIFY_SCAN, rmips.RMIPS_FLAG_VERIFY_SCAN | rmips.RMIPS_FLAG_FORCE_VERIFY):
        got = rmips.split_sets(*rmips.rmips_query(idx, t(Qy), k, fl))
        bad += sum(not np.array_equal(a, b) for a, b in zip(got, want))
    idx.close()
print("BAD", bad)
"""


def test_tiled_verification_scan_dev():
    """The shared-memory tiled form of Alg. 2's scan (used when P32 exceeds the L2 budget) forced on
    small instances through the development library (RMIPS_SCAN_TILED): P' indexes and the scan-all
    stress modes, d = 50 / 200 / 520 (1 pair per warp, 32-row tiles), against the naive oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2110_07131_b200 import build_lib
    e = dict(os.environ, RMIPS_LIB=build_lib.build_dev(), RMIPS_SCAN_TILED="1")
    r = subprocess.run([sys.executable, "-c", _TILED_SCRIPT, root], env=e, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "BAD 0" in r.stdout, r.stdout[-500:]


def _np(t):
    return t.cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)


def test_query_batches_equals_single_calls(cfg0):
    """rmips_query_batches (one host sync for all batches) = rmips_query per batch, concatenated:
    ragged last batch, several batch sizes, the key-sort fallback, k > k_max, capacity, host variant."""
    w, member = cfg0
    idx = rmips.rmips_build_index(_t(w.U), _t(w.P), 10)
    off, ids = rmips.rmips_query_batches(idx, _t(w.Qy), 32, 10)  # 100 queries: 32, 32, 32, 4
    assert_same(rmips.split_sets(off, ids), member, w.U, w.P, w.Qy, 10, "cfg0 batches")
    assert idx.stats()["queries"] == 100 and idx.stats()["result_total"] == int(member.sum())
    U, P = gen.random_instance(21, 3000, 700, 40)
    Qy = P[np.arange(700) % len(P)]
    idx2 = rmips.rmips_build_index(_t(U), _t(P), 12)
    for batch in (256, 100, 700, 1000, 1):
        for fl in (0, rmips.RMIPS_FLAG_KEY_SORT):
            o1, i1 = rmips.rmips_query_batches(idx2, _t(Qy[:300] if batch == 1 else Qy), batch, 9, fl)
            q = Qy[:300] if batch == 1 else Qy
            parts = [rmips.rmips_query(idx2, _t(q[b0:b0 + batch]), 9) for b0 in range(0, len(q), batch)]
            want = [s for o, i in parts for s in rmips.split_sets(o, i)]
            got = rmips.split_sets(o1, i1)
            assert len(got) == len(q) and all(np.array_equal(a, b) for a, b in zip(got, want)), (batch, fl)
            assert int(_np(o1)[0]) == 0 and int(_np(o1)[-1]) == len(_np(i1))
    # k > k_max extends once, up front (the same sets as single calls after the extension)
    o1, i1 = rmips.rmips_query_batches(idx2, _t(Qy[:500]), 256, 20)
    parts = [rmips.rmips_query(idx2, _t(Qy[b0:b0 + 256]), 20) for b0 in (0, 256)]
    want = [s for o, i in parts for s in rmips.split_sets(o, i)]
    assert all(np.array_equal(a, b) for a, b in zip(rmips.split_sets(o1, i1), want))
    # capacity: an explicit small capacity fails with the needed total; None retries
    with pytest.raises(rmips.RmipsError) as e:
        rmips.rmips_query_batches(idx2, _t(Qy), 256, 9, capacity=3)
    assert e.value.status == rmips.RMIPS_ERR_CAPACITY
    o1, i1 = rmips.rmips_query_batches(idx2, _t(Qy), 256, 9)
    ho, hi = rmips.rmips_query_batches_host(idx2, Qy, 256, 9)
    assert np.array_equal(_np(o1), ho) and np.array_equal(_np(i1), hi)
    # nq = 0
    o0, i0 = rmips.rmips_query_batches(idx2, _t(Qy[:0]), 256, 9)
    assert _np(o0).tolist() == [0] and len(_np(i0)) == 0
    idx.close()
    idx2.close()


def test_unaligned_input_views_build_identical_index():
    """Q and P given as row-slice views whose data pointers are not 16-byte aligned (d = 50: a one-row
    offset is 200 bytes) build the same index, bit for bit, as aligned copies."""
    import torch
    U, P = gen.random_instance(31, 1500, 700, 50)
    Ub = torch.from_numpy(np.vstack([U[:1], U])).cuda()
    Pb = torch.from_numpy(np.vstack([P[:1], P])).cuda()
    Uv, Pv = Ub[1:], Pb[1:]
    assert Uv.data_ptr() % 16 != 0 and Pv.data_ptr() % 16 != 0
    a = rmips.rmips_build_index(Uv, Pv, 10)
    b = rmips.rmips_build_index(_t(U), _t(P), 10)
    ta, tb = a.export(), b.export()
    for x, y in zip(ta, tb):
        assert np.array_equal(np.asarray(x), np.asarray(y))
    a.close()
    b.close()


def test_query_batches_other_paths_equal_single_calls():
    """rmips_query_batches on the other query paths (Alg. 2's scan for every undecided pair, no Lemma 3
    blocks, a P' index) = rmips_query per batch, and the oracle on the P' index."""
    U, P = gen.random_instance(41, 1200, 500, 24)
    Qy = P[np.arange(300) % len(P)]
    idx = rmips.rmips_build_index(_t(U), _t(P), 8)
    pidx = rmips.rmips_build_index_pprime(_t(U), _t(P), 8, 16)
    cases = [(idx, rmips.RMIPS_FLAG_VERIFY_SCAN), (idx, rmips.RMIPS_FLAG_NO_BLOCKS), (pidx, 0),
             (pidx, rmips.RMIPS_FLAG_KEY_SORT)]
    for ix, fl in cases:
        o1, i1 = rmips.rmips_query_batches(ix, _t(Qy), 128, 6, fl)
        parts = [rmips.rmips_query(ix, _t(Qy[b0:b0 + 128]), 6, fl) for b0 in range(0, len(Qy), 128)]
        want = [s for o, i in parts for s in rmips.split_sets(o, i)]
        got = rmips.split_sets(o1, i1)
        assert len(got) == len(Qy) and all(np.array_equal(a, b) for a, b in zip(got, want)), fl
    member = oracle.rkmips_naive(U, P, Qy, 6)
    assert_same(rmips.split_sets(*rmips.rmips_query_batches(pidx, _t(Qy), 100, 6)), member, U, P, Qy, 6,
                "P' batches")
    idx.close()
    pidx.close()


def test_large_d_lists_do_not_overflow():
    """d > 256 (configs[4] recipe): the 256-slot lists hold every row (with 128 slots, d = 300 / 513 sent
    hundreds of rows per 100k to the O(m d) exact fallback); the tables still equal the oracle's."""
    from synth.generator import make_workload
    for d in (300, 513):
        w = make_workload(4, n=6000, m=120000, d=d, nq=4)
        idx = rmips.rmips_build_index(_t(w.U), _t(w.P), 50)
        idx.refresh_info()
        assert idx.overflow_rows == 0 and idx.cand_slots == 256, (d, idx.overflow_rows, idx.cand_slots)
        pu, pp, tau, ids = idx.export()
        users = np.arange(0, 6000, 997)
        vals, oids = oracle.topk(w.U[users], w.P, 50)
        assert np.array_equal(tau[:, users].T, vals) and np.array_equal(ids[:, users].T, oids), d
        idx.close()


_REGROUP_SCRIPT = """
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_2110_07131_b200 import rmips
from synth import generator as gen
d = int(sys.argv[3])
w = gen.make_workload(4, n=80001, m=70000, nq=8, d=d)
dev = torch.device("cuda:0")
idx = rmips.rmips_build_index(torch.from_numpy(w.U).to(dev), torch.from_numpy(w.P).to(dev), 10)
assert idx.build_kernel == (4 if d > 64 else 1) and idx.overflow_rows == 0
_, _, tau, ids = idx.export()
np.savez(sys.argv[2], tau=tau, ids=ids, tiles=idx.tiles_done, lib=rmips.LIB_PATH)
"""


@pytest.mark.parametrize("d", [50, 100])
def test_regrouped_build_equals_single_pass(tmp_path, d):
    """The tensor-core builds' head pass + regrouping (rows sorted by their head theta, lists written back
    to the index order) triggers at n >= 4 * 148 * 128 users and >= 16 head lengths of item tiles: on
    80,001 x 70,000 (ragged last user tile), k_max = 10, d = 50 (k_build_tc) and d = 100 (the CTA-pair
    kernel), the lists equal the oracle's on a user sample (the
    last rows included) and the whole tables equal those of the single-pass build (development library,
    RMIPS_HEAD_TILES=0), bitwise."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2110_07131_b200 import build_lib
    devlib = build_lib.build_dev()
    got = {}
    # (d <= 64: regrouping is off in the product library; forced on here)
    for name, env in (("regroup", {"RMIPS_HEAD_TILES": "8" if d == 50 else "32"}), ("single", {"RMIPS_HEAD_TILES": "0"})):
        out = str(tmp_path / (name + ".npz"))
        e = dict(os.environ, RMIPS_LIB=devlib, **env)
        r = subprocess.run([sys.executable, "-c", _REGROUP_SCRIPT, root, out, str(d)], env=e, capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        got[name] = np.load(out)
    assert np.array_equal(got["regroup"]["tau"], got["single"]["tau"])
    assert np.array_equal(got["regroup"]["ids"], got["single"]["ids"])
    assert got["regroup"]["tiles"] < got["single"]["tiles"] or d == 50
    w = gen.make_workload(4, n=80001, m=70000, nq=8, d=d)
    rng = np.random.default_rng(11)
    sample = np.unique(np.concatenate([rng.choice(80001, 250, replace=False), np.arange(80001 - 40, 80001)]))
    vals, oids = oracle.topk(w.U[sample], w.P, 10)
    # (export returns users in their original order)
    idx = rmips.rmips_build_index(_t(w.U), _t(w.P), 10)
    _, _, tau, ids = idx.export()
    idx.close()
    assert np.array_equal(tau, got["regroup"]["tau"]) and np.array_equal(ids, got["regroup"]["ids"])
    assert np.array_equal(tau[:, sample].T, vals)
    assert np.array_equal(ids[:, sample].T, oids)


@pytest.mark.parametrize("env", [{}, {"RMIPS_SEED_TILES": "0"}], ids=["default", "seed0"])
def test_pair_build_seed_pass_bitwise(env, tmp_path):
    """The CTA-pair build's seed pass (8 item tiles of 8-item group maxima -> a starting theta) on the single
    pass (20,000 users: no regrouping), d = 120, m = 6,000 (47 item tiles), k_max = 50: the lists equal the
    oracle's on a user sample with and without the seed pass (development library switches)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2110_07131_b200 import build_lib
    devlib = build_lib.build_dev()
    out = str(tmp_path / "v.npz")
    e = dict(os.environ, RMIPS_LIB=devlib, **env)
    r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, root, out, "120"], env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(out)
    U, P = gen.random_instance(77, 20000, 6000, 120, "skewed")
    sample = np.sort(np.random.default_rng(8).choice(U.shape[0], 500, replace=False))
    vals, oids = oracle.topk(U[sample], P, 50)
    assert np.array_equal(got["tau"][:, sample].T, vals)
    assert np.array_equal(got["ids"][:, sample].T, oids)


def test_regrouped_build_overflowed_rows():
    """Rows that overflow their candidate buffer in the regrouped CTA-pair build's HEAD pass (150 identical
    items with the largest norm: massive ties for every user with a positive cosine to them) are saved with
    the overflow mark (their theta sorts last), skip the main pass and take the exact fallback at their index
    rows; the sampled tables equal the oracle's (ties by ascending item id)."""
    w = gen.make_workload(4, n=80001, m=70000, nq=8, d=100)
    P = w.P.copy()
    nrm = np.linalg.norm(P.astype(np.float64), axis=1)
    p = P[int(np.argmax(nrm))].astype(np.float64)
    P[:150] = (p / np.linalg.norm(p) * 2.0 * nrm.max()).astype(np.float32)
    idx = rmips.rmips_build_index(_t(w.U), _t(P), 10)
    assert idx.build_kernel == 4
    assert idx.overflow_rows > 1000
    _, _, tau, ids = idx.export()
    idx.close()
    rng = np.random.default_rng(5)
    sample = np.sort(rng.choice(80001, 300, replace=False))
    vals, oids = oracle.topk(w.U[sample], P, 10)
    assert np.array_equal(tau[:, sample].T, vals)
    assert np.array_equal(ids[:, sample].T, oids)


@pytest.mark.parametrize("env", [{"RMIPS_2CTA_D64": "1"}, {"RMIPS_2CTA_D64": "1", "RMIPS_2CTA_FPOL": "1"},
                                 {"RMIPS_2CTA_D64": "1", "RMIPS_2CTA_FPOL": "2"}],
                         ids=["pair-qpol", "pair-fpol", "pair-fpol-flat"])
def test_pair_build_at_d64_bitwise(env, tmp_path):
    """The CTA-pair kernel forced onto d_pad = 64 (development switches) with its 4-byte (QPolT) and 8-byte
    (FPol) candidate lists, single pass with the seed pass (20,000 users, 47 item tiles, k_max = 50): the
    lists equal the oracle's on a user sample."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    from paper_2110_07131_b200 import build_lib
    devlib = build_lib.build_dev()
    out = str(tmp_path / "v.npz")
    e = dict(os.environ, RMIPS_LIB=devlib, **env)
    r = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, root, out, "50"], env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(out)
    U, P = gen.random_instance(77, 20000, 6000, 50, "skewed")
    sample = np.sort(np.random.default_rng(9).choice(U.shape[0], 500, replace=False))
    vals, oids = oracle.topk(U[sample], P, 50)
    assert np.array_equal(got["tau"][:, sample].T, vals)
    assert np.array_equal(got["ids"][:, sample].T, oids)
