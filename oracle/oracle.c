/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for exact reverse k-MIPS.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library.  The product path
 * (paper_2110_07131_b200/) never includes, links or calls anything in oracle/.
 * It shares no code, header, table or constant with the CUDA path.
 *
 * Citations: P:n = /root/reference/PAPER.md line n (Amagata & Hara, "Reverse
 * Maximum Inner Product Search", arXiv 2110.07131).  Readings of the paper that
 * this file takes are listed in DESIGN.md §3 ("Readings").
 *
 * Arithmetic rules (reading R7):
 *   - inputs are the caller's fp32 values, widened to fp64 (exact);
 *   - ONE dot routine, orc_dot(), a left-to-right fp64 sum, used for BOTH q.u and p.u
 *     (compiled with -ffp-contract=off; each product of two fp32 values is exact in fp64,
 *     so the only rounding is the sequential sum);
 *   - norms are sqrt(orc_dot(a, a)).
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fPIC -shared oracle.c -o liboracle.so -lm
 *
 * Parity status of each entry point:
 *   orc_dot, orc_norms, orc_sort_by_norm_desc, orc_topk, orc_rkmips_naive,
 *   orc_rkmips_twophase, orc_linear_scan, orc_block_bounds,
 *   orc_margin (Table 1 hand margins, exclusion of copies of q), orc_margin_lists (equals
 *   orc_margin by brute force)                                     -- pinned by tests/test_oracle_pins.py
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* u.p -- the inner product of Def. 1.  Left-to-right fp64 sum. */
double orc_dot(const float* a, const float* b, int d) {
    double s = 0.0;
    for (int j = 0; j < d; ++j) s += (double)a[j] * (double)b[j];
    return s;
}

/* ||x|| for every row (Alg. 1 lines 1-4). */
void orc_norms(const float* X, int64_t n, int d, double* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = sqrt(orc_dot(X + i * d, X + i * d, d));
}

/* Alg. 1 line 5: "Sort Q and P in descending order of norm size".
 * Ties by ascending original id (reading R6).  perm[rank] = original id.
 * Plain insertion-free approach: qsort on (norm desc, id asc). */
static const double* g_sort_keys;
static int cmp_desc(const void* x, const void* y) {
    int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
    if (g_sort_keys[a] > g_sort_keys[b]) return -1;
    if (g_sort_keys[a] < g_sort_keys[b]) return 1;
    return (a < b) ? -1 : (a > b);
}
void orc_sort_by_norm_desc(const double* norms, int64_t n, int64_t* perm) {
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    g_sort_keys = norms;
    qsort(perm, (size_t)n, sizeof(int64_t), cmp_desc);
}

/* k-MIPS (Def. 1) for every user: the kk largest inner products u.p over
 * ALL of P (BASELINE north_star: full-P lower-bound arrays, so L_i^j = tau_j(u)),
 * value-descending, ties by ascending item id.  Rows with kk > m are padded with
 * -inf / -1.  Plain per-user selection by repeated insertion into a sorted list. */
void orc_topk(const float* U, int64_t n, const float* P, int64_t m, int d, int kk,
              double* vals, int32_t* ids, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
    for (int64_t i = 0; i < n; ++i) {
        double* v = vals + i * kk;
        int32_t* id = ids + i * kk;
        int cnt = 0;
        for (int t = 0; t < kk; ++t) { v[t] = -INFINITY; id[t] = -1; }
        for (int64_t j = 0; j < m; ++j) {
            double s = orc_dot(U + i * d, P + j * d, d);
            /* insert (s, j) if it beats the current kk-th entry; equal values keep the
             * lower id first because j increases monotonically */
            if (cnt == kk && !(s > v[kk - 1])) continue;
            int pos = (cnt < kk) ? cnt : kk - 1;
            while (pos > 0 && s > v[pos - 1]) {
                v[pos] = v[pos - 1]; id[pos] = id[pos - 1]; --pos;
            }
            v[pos] = s; id[pos] = (int32_t)j;
            if (cnt < kk) ++cnt;
        }
    }
}

/* Reverse k-MIPS by its definition (Def. 2), strict-greater convention
 * (reading R1): c(u,q) = |{p in P : p.u > q.u}|,  u in R_k(q)  <=>  c(u,q) < k.
 * member[qi * n + i] = 1 iff user i is in R_k(query qi).  O(nq * n * m * d). */
void orc_rkmips_naive(const float* U, int64_t n, const float* P, int64_t m, int d,
                      const float* Qy, int64_t nq, int k, uint8_t* member, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for collapse(2) schedule(dynamic, 64)
#endif
    for (int64_t qi = 0; qi < nq; ++qi) {
        for (int64_t i = 0; i < n; ++i) {
            double g = orc_dot(Qy + qi * d, U + i * d, d);
            int64_t c = 0;
            for (int64_t j = 0; j < m && c < k; ++j)
                if (orc_dot(P + j * d, U + i * d, d) > g) ++c;
            member[qi * n + i] = (uint8_t)(c < k);
        }
    }
}

/* The same decision from a user's exact top-kk list (kk >= k):
 *   c'(u,q) = |{listed j : vals_j > q.u}|,  u in R_k(q) <=> c' < k.
 * Equal to the naive count for k <= kk: if c' >= k then k items strictly beat q;
 * if c' < k then vals_k <= q.u and every unlisted item is <= vals_kk <= vals_k <= q.u.
 * (reading R8.) */
void orc_rkmips_twophase(const float* U, int64_t n, int d, const double* topvals, int kk,
                         const float* Qy, int64_t nq, int k, uint8_t* member, int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for collapse(2) schedule(static)
#endif
    for (int64_t qi = 0; qi < nq; ++qi) {
        for (int64_t i = 0; i < n; ++i) {
            double g = orc_dot(Qy + qi * d, U + i * d, d);
            int c = 0;
            for (int t = 0; t < kk; ++t)
                if (topvals[i * kk + t] > g) ++c;
            member[qi * n + i] = (uint8_t)(c < k);
        }
    }
}

/* Alg. 2 Linear-scan(u) with Corollaries 1-2, as corrected by
 * readings R3 (tau starts at -inf, not 0) and R4 (falling off the end returns yes).
 * P_sorted / pnorm_sorted: items in norm-descending order (Alg. 1 line 5).
 * Returns 1 (yes) / 0 (no); *scanned = number of items whose u.p was evaluated.
 * I is kept as the multiset of the k largest values seen (including u.q). */
int orc_linear_scan(const float* u, double unorm, const float* q, const float* P_sorted,
                    const double* pnorm_sorted, int64_t m, int d, int k, int64_t* scanned) {
    double uq = orc_dot(q, u, d);
    double* I = (double*)malloc(sizeof(double) * (size_t)(k + 1));
    int cnt = 0;
    double tau = -INFINITY;
    int64_t sc = 0;
    int ans = 1; /* R4: surviving the whole scan means yes */
    I[cnt++] = uq; /* line 1: I <- {u.q} */
    for (int64_t i = 0; i < m; ++i) {
        if (uq >= unorm * pnorm_sorted[i]) { ans = 1; break; } /* line 3, Corollary 1 */
        double gam = orc_dot(P_sorted + i * d, u, d); /* line 5 */
        ++sc;
        if (gam > tau) { /* line 6 */
            /* line 7: I <- I u {gam}; keep sorted descending */
            int pos = cnt;
            I[cnt++] = gam;
            while (pos > 0 && I[pos] > I[pos - 1]) { double t = I[pos]; I[pos] = I[pos - 1]; I[pos - 1] = t; --pos; }
            if (cnt > k) { /* lines 8-10 */
                cnt = k;                /* delete the (k+1)-th */
                tau = I[k - 1];         /* tau <- k-th value of I */
            }
            if (tau > uq) { ans = 0; break; } /* lines 11-12, Corollary 2 */
        }
    }
    free(I);
    if (scanned) *scanned = sc;
    return ans;
}

/* Eq. (1) / Alg. 1 lines 10-16: blocks of b consecutive norm-sorted
 * users, L^j(B) = min over members of L_i^j.  L is [n][kk] in sorted-user order;
 * out is [nblocks][kk]. */
void orc_block_bounds(const double* L, int64_t n, int kk, int64_t b, double* out) {
    int64_t nb = (n + b - 1) / b;
    for (int64_t B = 0; B < nb; ++B) {
        for (int j = 0; j < kk; ++j) {
            double mn = INFINITY;
            for (int64_t i = B * b; i < n && i < (B + 1) * b; ++i)
                if (L[i * kk + j] < mn) mn = L[i * kk + j];
            out[B * kk + j] = mn;
        }
    }
}

/* Parity bookkeeping (BASELINE north_star borderline rule; reading R9): relative margin
 * mu = (q.u - tau'_k(u)) / (||q|| ||u||), tau'_k = k-th largest p.u over p in P that are
 * not bitwise-equal to q.  Computed for listed (qi, i) pairs.  "parity unpinned". */
void orc_margin(const float* U, int64_t n, const float* P, int64_t m, int d,
                const float* Qy, const int64_t* pairs, int64_t npairs, int k, double* mu,
                int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
    for (int64_t t = 0; t < npairs; ++t) {
        int64_t qi = pairs[2 * t], i = pairs[2 * t + 1];
        const float* q = Qy + qi * d;
        const float* u = U + i * d;
        double* top = (double*)malloc(sizeof(double) * (size_t)k);
        int cnt = 0;
        for (int64_t j = 0; j < m; ++j) {
            if (memcmp(P + j * d, q, sizeof(float) * (size_t)d) == 0) continue;
            double s = orc_dot(P + j * d, u, d);
            if (cnt == k && !(s > top[k - 1])) continue;
            int pos = (cnt < k) ? cnt : k - 1;
            while (pos > 0 && s > top[pos - 1]) { top[pos] = top[pos - 1]; --pos; }
            top[pos] = s;
            if (cnt < k) ++cnt;
        }
        double tau = (cnt == k) ? top[k - 1] : -INFINITY;
        double g = orc_dot(q, u, d);
        double nq = sqrt(orc_dot(q, q, d)), nu = sqrt(orc_dot(u, u, d));
        double den = nq * nu;
        mu[t] = (den > 0) ? (g - tau) / den : (g - tau);
        free(top);
    }
}

/* The same margin (reading R9) from a user's exact top-kk list over P (orc_topk output:
 * values descending, item ids; -1 padding), so that it costs O(d + kk) per pair instead of a
 * scan of P: tau'_k(u) is the k-th listed value whose item is not bitwise-equal to q.  Items
 * outside the list score <= the last listed value, so the k-th surviving listed value IS the
 * k-th largest over P minus the copies of q whenever k survivors exist; when fewer survive and
 * the list is full (copies of q used up the slack), the pair falls back to orc_margin's scan.
 * Used by the bench and the parity tests for the BASELINE borderline bookkeeping. */
void orc_margin_lists(const float* U, int64_t n, const float* P, int64_t m, int d,
                      const float* Qy, const double* topvals, const int32_t* topids, int kk,
                      const int64_t* pairs, int64_t npairs, int k, double* mu, int threads) {
    (void)n;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic, 256)
#endif
    for (int64_t t = 0; t < npairs; ++t) {
        int64_t qi = pairs[2 * t], i = pairs[2 * t + 1];
        const float* q = Qy + qi * d;
        const float* u = U + i * d;
        const double* v = topvals + i * kk;
        const int32_t* id = topids + i * kk;
        double tau = -INFINITY;
        int seen = 0, full = 1, found = 0;
        for (int j = 0; j < kk; ++j) {
            if (id[j] < 0) { full = 0; break; }
            if (memcmp(P + (int64_t)id[j] * d, q, sizeof(float) * (size_t)d) == 0) continue;
            if (++seen == k) { tau = v[j]; found = 1; break; }
        }
        if (!found && full && kk < m) { /* not resolvable from the list: the definition */
            orc_margin(U, n, P, m, d, Qy, pairs + 2 * t, 1, k, mu + t, 1);
            continue;
        }
        double g = orc_dot(q, u, d);
        double nq = sqrt(orc_dot(q, q, d)), nu = sqrt(orc_dot(u, u, d));
        double den = nq * nu;
        mu[t] = (den > 0) ? (g - tau) / den : (g - tau);
    }
}
