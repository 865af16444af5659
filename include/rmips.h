/*
 * rmips.h -- C ABI of the B200 (sm_100a) exact reverse k-MIPS library.
 *
 * Problem (Def. 2): given user vectors Q (n x d), item vectors
 * P (m x d), a query item q and k, return every user u in Q such that q is in u's
 * k-MIPS result over P u {q}.  Tie convention (reading R1): u is returned iff
 * fewer than k items p in P satisfy p.u > q.u (strictly).  Results are EXACT: every
 * reduced-precision tensor-core score is only a conservative filter, and every pair the
 * filter cannot decide is decided from fp64 values.
 *
 * Method (§4): Alg. 1 (lines 267-298) pre-processing, generalised per
 * BASELINE.json's north star to the exact top-k_max inner products over ALL of P
 * (lower-bound arrays L_i, Def. 4, become exact); blocks with Eq. (1) minima
 * (line 260); Alg. 3 (lines 499-524) queries with Lemma 3 block pruning (417-426),
 * Lemma 1 rejection (389-396) and exact decision of undecided users; Alg. 2's linear
 * scan (475-498) is available as the verification path (RMIPS_FLAG_VERIFY_SCAN).
 *
 * Conventions common to every call:
 *   - Matrices are contiguous, row-major fp32, d floats per row, no padding.
 *   - "device" pointers are CUDA device (or managed) memory; "host" pointers are
 *     ordinary or pinned host memory.
 *   - cuda_stream is a cudaStream_t (NULL = legacy default stream).  All work is
 *     enqueued on it; each call synchronises that stream once before returning (to
 *     report device-detected errors and result sizes).
 *   - Nothing throws across this ABI; every entry point returns an rmips_status_t.
 *   - Not re-entrant on one index: rmips_query uses per-index workspace.  Distinct
 *     indexes may be used concurrently from different threads/streams.
 */
#ifndef RMIPS_H_
#define RMIPS_H_

#include <stdint.h>

#if defined(__GNUC__)
#define RMIPS_API __attribute__((visibility("default")))
#else
#define RMIPS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rmips_index_s* rmips_index_t; /* opaque; immutable after build */

typedef enum {
  RMIPS_OK = 0,
  RMIPS_ERR_INVALID = 1,   /* null pointer, n < 0, m < 1, d < 1 or d > 1024, b < 0, bad flags */
  RMIPS_ERR_NONFINITE = 2, /* a NaN/Inf in Q, P or a query vector */
  RMIPS_ERR_K_RANGE = 3,   /* k < 1, k_max < 1, or k > k_max with RMIPS_FLAG_NO_EXTEND */
  RMIPS_ERR_CAPACITY = 4,  /* result ids exceed `capacity`; *total_out and offsets hold the needed size */
  RMIPS_ERR_CUDA = 5,      /* a CUDA runtime error (message via rmips_last_error) */
  RMIPS_ERR_OOM = 6        /* device allocation failed */
} rmips_status_t;

/* Optional behaviour flags for rmips_query_ex. */
enum {
  RMIPS_FLAG_NONE = 0,
  RMIPS_FLAG_NO_BLOCKS = 1,     /* skip Lemma 3 (the paper's "without blocks" ablation) */
  RMIPS_FLAG_VERIFY_SCAN = 2,   /* decide undecided pairs with Alg. 2's early-terminating scan over
                                   norm-sorted P (Cor. 1-2) instead of the exact top list */
  RMIPS_FLAG_FORCE_VERIFY = 4,  /* stress mode: every pair that Lemma 1 does not reject goes to the
                                   undecided path (with VERIFY_SCAN: through the scan kernel) */
  RMIPS_FLAG_SIMT = 8,          /* use the SIMT (CUDA-core) filter kernels instead of tcgen05 */
  RMIPS_FLAG_TIMING = 16,       /* record per-phase CUDA-event times (rmips_phase_times) */
  RMIPS_FLAG_NO_EXTEND = 32,    /* k > k_max fails with RMIPS_ERR_K_RANGE instead of extending the index */
  RMIPS_FLAG_KEY_SORT = 64      /* output through the sorted (query, user) key list even when the
                                   b x n bit matrix (b * ceil(n/32) * 4 bytes <= 64 MiB) would be used */
};

/* Per-index build options (rmips_build_index_ex). */
enum {
  RMIPS_BUILD_DEFAULT = 0,
  RMIPS_BUILD_SIMT = 1,         /* score the build contraction on CUDA cores instead of tcgen05 */
  RMIPS_BUILD_TIMING = 2        /* record per-phase CUDA-event times (rmips_phase_times) */
};

/* Counters of the most recent rmips_query on an index (Theorem 3 instrumentation,
 * alpha = pruned (block, query) pairs / all; m' = items_scanned / scans). */
typedef struct {
  int64_t queries;              /* queries in the call */
  int64_t block_query_pairs;    /* (user block, query) pairs considered */
  int64_t block_query_pruned;   /* ... pruned by Lemma 3 */
  int64_t pairs_scored;         /* (user, query) filter scores computed */
  int64_t pairs_rejected;       /* rejected by the filter (Lemma 1 with the error bound) */
  int64_t pairs_accepted_fast;  /* accepted by the filter (u.q >= tau_k with the error bound) */
  int64_t pairs_undecided;      /* handed to the exact path */
  int64_t pairs_exact_accepted; /* ... of which accepted */
  int64_t scans;                /* Alg. 2 scans run (VERIFY_SCAN) */
  int64_t items_scanned;        /* items whose u.p the scans evaluated */
  int64_t result_total;         /* sum over queries of |R(q)| */
  int64_t filter_kernel;        /* 1 = tcgen05 filter (query_tc.cu), 0 = SIMT filter */
  int64_t tiles_scored;         /* (128-user tile, query sub-batch) work items not pruned whole by Lemma 3 */
  int64_t scan_exact;           /* scanned items re-evaluated in fp64 (inside the scan's fp32 error band) */
} rmips_stats_t;

/* rmips_build_index -- Alg. 1 (PAPER.md 267-298) with L_i over all of P.
 *   Q       device, n x d fp32 user vectors (may be NULL iff n == 0)
 *   n       number of users, >= 0
 *   P       device, m x d fp32 item vectors
 *   m       number of items, 1 <= m < 2^31 (m > 2^20 with d > 64 uses 8-byte candidate entries, slower)
 *   d       dimensionality, 1 <= d <= 1024 (the tensor-core kernels cover every d in that range: K blocks
 *           of 64 columns, the last one trimmed to 16/32/64 columns; for d > 256 the build and query
 *           K loops stream the user and query K blocks from L2 instead of keeping them on chip;
 *           RMIPS_BUILD_SIMT covers d <= 256 only)
 *   k_max   largest k the index answers, >= 1 (lists are padded with -inf when k_max > m).  The
 *           build's candidate filter keeps 128 slots per user row for k_max <= 80 and d <= 240 (m <=
 *           2^20), and 256 slots for larger k_max or d, and for 2^20 < m <= 2^21 (4-byte entries with 21-bit
 *           positions); beyond m = 2^21, and with RMIPS_BUILD_SIMT, 128 slots of 8-byte entries.  A row
 *           whose list cannot be compacted into its slots (k_max above ~220 with 256 slots; k_max above
 *           ~60 or crowded scores at large d with 128 8-byte slots; massive ties) is recomputed exactly
 *           by a fallback kernel that costs O(k_max m d) per row: correct, slow (overflow rows are
 *           reported by rmips_index_info)
 *   out     receives the new index handle (NULL on failure)
 * The library copies what it needs; Q and P may be freed after the call returns.
 * Errors: INVALID, NONFINITE, K_RANGE (k_max < 1), OOM, CUDA. */
RMIPS_API rmips_status_t rmips_build_index(const float* Q, int64_t n, const float* P, int64_t m, int32_t d,
                                 int32_t k_max, void* cuda_stream, rmips_index_t* out);
RMIPS_API rmips_status_t rmips_build_index_ex(const float* Q, int64_t n, const float* P, int64_t m, int32_t d,
                                    int32_t k_max, int32_t build_flags, void* cuda_stream,
                                    rmips_index_t* out);
/* rmips_build_index_pprime -- Alg. 1 as printed (PAPER.md 267-298): the lists L_i^j are the
 * k_max largest u_i.p over P' = the first m_prime items of the norm-sorted P (line 6, P:280,
 * "the first O(k_max) vectors"; SPEC uses m_prime = 2 k_max), so they are LOWER bounds of the
 * k-th largest over P (Def. 4).  Queries on such an index decide a pair by Lemma 1 (reject
 * when u.q < L^k), Lemma 2 (accept when u.q >= ||u|| ||p_k||), Cor. 1 at item m_prime
 * (accept when u.q >= ||u|| ||p_{m_prime+1}||: no item outside P' can beat q), and otherwise
 * Alg. 2's early-terminating scan over the items after P', started with the count of
 * P' items that beat q (exact: the list holds P''s exact top k_max).
 *   m_prime  1 <= m_prime; values >= m build the exact index (same as rmips_build_index_ex)
 * Other arguments and errors as rmips_build_index_ex. */
RMIPS_API rmips_status_t rmips_build_index_pprime(const float* Q, int64_t n, const float* P, int64_t m, int32_t d,
                                        int32_t k_max, int64_t m_prime, int32_t build_flags,
                                        void* cuda_stream, rmips_index_t* out);
/* Same, with Q and P in HOST memory (copied to the device inside the call). */
RMIPS_API rmips_status_t rmips_build_index_host(const float* Q, int64_t n, const float* P, int64_t m, int32_t d,
                                      int32_t k_max, void* cuda_stream, rmips_index_t* out);

/* rmips_query -- Alg. 3 (PAPER.md 499-524) for a batch of b query items.
 *   idx        index from rmips_build_index
 *   q_batch    device, b x d fp32 query vectors (may be NULL iff b == 0)
 *   b          number of queries, >= 0 (any size; processed internally in tiles of 256)
 *   k          k >= 1.  k > k_max first EXTENDS the index in place to k_max = k (the paper's
 *              "re-builds the data structures"): the lists, the block
 *              table and the candidate filter are rebuilt from the index's own sorted operands
 *              (no caller rebuild; the cost of one build without its prep phase).  With
 *              RMIPS_FLAG_NO_EXTEND it fails with RMIPS_ERR_K_RANGE instead.
 *   offsets    device, b + 1 int64: query i's users are user_ids[offsets[i] .. offsets[i+1])
 *   user_ids   device, capacity int32: 0-based ORIGINAL row indices of Q, ascending per query
 *   capacity   number of int32 slots in user_ids
 *   total_out  host: receives sum_i |R(q_i)| (also on RMIPS_ERR_CAPACITY, with offsets valid)
 * Output assembly: accepted pairs are set as bits of a b x n matrix in the query workspace when
 * b * ceil(n/32) * 4 <= 64 MiB (read back chunk by chunk: no sort, one host sync per call), else
 * appended as (query, user) keys and radix-sorted.  Same offsets and ids either way.
 * Errors: INVALID, NONFINITE (non-finite query), K_RANGE, CAPACITY, OOM, CUDA. */
RMIPS_API rmips_status_t rmips_query(rmips_index_t idx, const float* q_batch, int32_t b, int32_t k,
                           int64_t* offsets, int32_t* user_ids, int64_t capacity, int64_t* total_out,
                           void* cuda_stream);
RMIPS_API rmips_status_t rmips_query_ex(rmips_index_t idx, const float* q_batch, int32_t b, int32_t k,
                              int32_t flags, int64_t* offsets, int32_t* user_ids, int64_t capacity,
                              int64_t* total_out, void* cuda_stream);
/* Same, with q_batch, offsets and user_ids in HOST memory (copied inside the call). */
RMIPS_API rmips_status_t rmips_query_host(rmips_index_t idx, const float* q_batch, int32_t b, int32_t k,
                                int64_t* offsets, int32_t* user_ids, int64_t capacity,
                                int64_t* total_out, void* cuda_stream);

/* rmips_query_batches -- a stream of queries answered in consecutive batches of `batch` (BASELINE
 * configs[4]: "10,000 freshly generated queries in batches of 256"): the result equals calling
 * rmips_query_ex on q_all[0 .. batch), q_all[batch .. 2 batch), ... and concatenating the sets in
 * query order, but the batches run back to back on the stream with ONE host synchronisation at the
 * end (each batch's output offsets continue from a device-side running total).
 *   q_all      device, nq x d fp32 (may be NULL iff nq == 0); nq >= 0, batch >= 1
 *   offsets    device, nq + 1 int64 (global: query i's users are user_ids[offsets[i] .. offsets[i+1]))
 *   user_ids, capacity, total_out, flags, k: as rmips_query_ex (k > k_max extends once, up front)
 * Shapes outside the bit-matrix output (RMIPS_FLAG_KEY_SORT, batch * ceil(n/32) * 4 > 64 MiB, n == 0)
 * run as one rmips_query_ex per batch (one synchronisation each); same results.  The counters of
 * rmips_query_stats are summed over the batches.  A batch that outgrows the pair workspace makes the
 * call run every batch again with a larger one (the results never depend on it).
 * Errors: as rmips_query_ex. */
RMIPS_API rmips_status_t rmips_query_batches(rmips_index_t idx, const float* q_all, int64_t nq, int32_t batch,
                                   int32_t k, int32_t flags, int64_t* offsets, int32_t* user_ids,
                                   int64_t capacity, int64_t* total_out, void* cuda_stream);
/* Same, with q_all, offsets and user_ids in HOST memory (one copy each way inside the call). */
RMIPS_API rmips_status_t rmips_query_batches_host(rmips_index_t idx, const float* q_all, int64_t nq,
                                        int32_t batch, int32_t k, int64_t* offsets, int32_t* user_ids,
                                        int64_t capacity, int64_t* total_out, void* cuda_stream);

/* Counters of the last rmips_query on idx (host struct filled). */
RMIPS_API rmips_status_t rmips_query_stats(rmips_index_t idx, rmips_stats_t* out);

/* Index introspection (for tests and tools).  All outputs are HOST buffers.
 *   info[0..9] = n, m, d, k_max, d_pad, block_size, overflow_rows, build_flags,
 *                candidates kept by the build filter (sum over rows),
 *                (128-user tile, item tile) contractions issued by the tensor-core build (0 for the
 *                SIMT build; fewer than all when the Cauchy-Schwarz early exit fired),
 *                m_prime (items the lists are built over; = m for the exact index),
 *                build kernel (0 SIMT, 1 k_build_tc (d <= 64), 2 k_build_tcq with the user tile in
 *                tensor memory, 3 k_build_tcq with streamed user K blocks (d > 256), 4 k_build_tc2cta
 *                (CTA pairs, tcgen05.mma.cta_group::2, 64 < d <= 256)),
 *                candidate slots per row (128 or 256);  info[13..15] reserved, 0
 *   perm_u[n], perm_p[m]: sorted position -> original id (norm descending, ties by id)
 *   tau[k_max * n] fp64 and ids[k_max * n] int32: column-major by rank, users in ORIGINAL
 *   order: tau[j * n + u] = (j+1)-th largest u.p over P (over P' for a P' index), ids = its
 *   original item id.
 *   Any of perm_u/perm_p/tau/ids may be NULL to skip it. */
RMIPS_API rmips_status_t rmips_index_info(rmips_index_t idx, int64_t info[16]);
RMIPS_API rmips_status_t rmips_index_export(rmips_index_t idx, int64_t* perm_u, int64_t* perm_p, double* tau,
                                  int32_t* ids);

/* Per-phase device times (ms, CUDA events recorded on the call's stream) of the last build /
 * query made with RMIPS_BUILD_TIMING / RMIPS_FLAG_TIMING, and kernel launch counts:
 *   ms[0] build prep (norms, sort, convert)   ms[1] build contraction + candidate epilogue
 *   ms[2] exact select + fallback + blocks     ms[3] build total
 *   ms[8] query prep   ms[9] query filter contraction   ms[10] exact decide / scan
 *   ms[11] output (sort, offsets, copy)       ms[12] query total
 *   ms[13] the tcgen05 query filter kernel alone (k_query_tc, events right around its launch)
 *   ms[14] kernels launched by the last build  ms[15] kernels launched by the last query
 * Entries not measured are -1.  ms must hold 16 doubles. */
RMIPS_API rmips_status_t rmips_phase_times(rmips_index_t idx, double ms[16]);

/* Frees the index (stream-ordered on the stream of the index's last call; no host sync).  Call it
 * before destroying that stream. */
RMIPS_API void rmips_free_index(rmips_index_t idx);
RMIPS_API const char* rmips_status_string(rmips_status_t s);
RMIPS_API const char* rmips_last_error(void);  /* thread-local detail of the last failure */
RMIPS_API const char* rmips_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RMIPS_H_ */
