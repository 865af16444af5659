// query.cu -- batched query evaluation (Alg. 3) except the tcgen05 filter.
//
//   Q1 k_query_prep      ||q|| (Alg. 3 line 1), norm sort of each 256-query tile, fp16 q*2^eq
//   Q2+Q3 k_query_simt   Lemma 3 prefix + SIMT filter with Lemma 1
//                        against tau_k, accept / reject / undecided (tcgen05 version: query_tc.cu)
//   Q4 k_exact_decide    exact decision of undecided pairs from the exact top list (reading R8)
//   Q5 k_verify_scan     Alg. 2 with Cor. 1-2, readings R3/R4 -- used
//                        with RMIPS_FLAG_VERIFY_SCAN
//   Q6 output            sort (query, original user id) keys; CSR offsets; copy to the caller
#include <cub/cub.cuh>

#include "common.cuh"
#include "internal.h"

namespace rmips {

// ------------------------------------------------------------------------------ Q1
// Two launches over warps, one warp per query (kPrepWarps per CTA):
//   k_query_norms   ||q|| with coalesced row reads (lanes over the row, fp64 sum; only its rounded-up
//                   value is used, so the order does not matter), the finite check, and each CTA's
//                   max |q_j| for the sub-batch's power-of-two scale
//   k_query_finish  the query's rank in (norm desc, index asc) order within its 256-query sub-batch
//                   (Alg. 3 line 1 sorts by ||q||), its slot's metadata, and its fp16 row q * 2^eq
//                   (zero-padded to ldh) in that slot
constexpr int kPrepWarps = 8;
constexpr int kPrepCtas = kQB / kPrepWarps;  // CTAs per sub-batch
__global__ void __launch_bounds__(32 * kPrepWarps)
k_query_norms(const float* __restrict__ q, int b, int d, double* __restrict__ nrm, float* __restrict__ cmax,
              int* __restrict__ flags) {
  pdl_enter();  // (PDL: see launch_pdl)
  __shared__ float smax[kPrepWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t qi = (int64_t)blockIdx.x * kPrepWarps + wid;  // sub-batch slot of the INPUT order
  float mx = 0.f;
  double acc = 0.0;
  bool fin = true;
  if (qi < b) {
    const float* x = q + qi * d;
    for (int e = lane; e < d; e += 32) {
      const float v = x[e];
      fin &= isfinite(v);
      mx = fmaxf(mx, fabsf(v));
      acc = __fma_rn((double)v, (double)v, acc);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  fin = __all_sync(0xffffffffu, fin);
  if (lane == 0) {
    double nr = qi < b ? sqrt(acc) : -1.0;
    if (qi < b && !fin) atomicOr(flags, kFlagNonfinite), nr = 0.0;
    nrm[qi] = nr;
    smax[wid] = isfinite(mx) ? mx : 0.f;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m2 = 0.f;
    for (int w = 0; w < kPrepWarps; ++w) m2 = fmaxf(m2, smax[w]);
    cmax[blockIdx.x] = m2;
  }
}

__global__ void __launch_bounds__(32 * kPrepWarps)
k_query_finish(const float* __restrict__ q, int b, int d, int ldh, double c1, double c2,
               const double* __restrict__ nrm, const float* __restrict__ cmax, __half* __restrict__ Q16,
               float* __restrict__ qn, float* __restrict__ qerr, float* __restrict__ qscale,
               int32_t* __restrict__ qperm, int32_t* __restrict__ qcount) {
  pdl_enter();  // (PDL: see launch_pdl)
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int s = blockIdx.x / kPrepCtas;
  const int t = (blockIdx.x - s * kPrepCtas) * kPrepWarps + wid;  // query t of sub-batch s (input order)
  const int cnt = min(kQB, b - s * kQB);
  // the sub-batch's scale 2^e: max |q_j| < 2^14 after scaling (the filter's fp16 range)
  float m2 = lane < kPrepCtas ? cmax[s * kPrepCtas + lane] : 0.f;
#pragma unroll
  for (int o = 16; o; o >>= 1) m2 = fmaxf(m2, __shfl_xor_sync(0xffffffffu, m2, o));
  int ex = 0;
  if (m2 > 0.f) frexpf(m2, &ex);
  const float scale = ldexpf(1.f, max(-126, min(126, 14 - ex)));
  const double* nr_s = nrm + (int64_t)s * kQB;
  const double nr = nr_s[t];
  int rank = t;  // padding (t >= cnt) keeps its own slot
  if (t < cnt) {
    int r = 0;
    for (int j = lane; j < cnt; j += 32) {
      const double o = nr_s[j];
      r += (o > nr) || (o == nr && j < t);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    rank = r;
  }
  const int64_t slot = (int64_t)s * kQB + rank;
  if (lane == 0) {
    if (t < cnt) {
      qperm[slot] = s * kQB + t;
      qn[slot] = __double2float_ru(nr * (1.0 + 1e-12));
      qerr[slot] = __double2float_ru((c1 * nr * (double)scale + c2) * (1.0 + 1e-6));
    } else {
      qperm[slot] = -1;
      qn[slot] = -CUDART_INF_F;
      qerr[slot] = 0.f;
    }
    if (t == 0) {
      qscale[s] = scale;
      qcount[s] = cnt;
    }
  }
  const float* x = q + (int64_t)(s * kQB + (t < cnt ? t : 0)) * d;
  __half2* out = reinterpret_cast<__half2*>(Q16 + slot * ldh);
  for (int e = 2 * lane; e < ldh; e += 64) {
    float v0 = 0.f, v1 = 0.f;
    if (t < cnt) {
      if (e < d) v0 = x[e] * scale;
      if (e + 1 < d) v1 = x[e + 1] * scale;
    }
    out[e >> 1] = __halves2half2(__float2half_rn(v0), __float2half_rn(v1));
  }
}

// Lemma 3 prefix of a (tile, sub-batch): #{slots < cnt : qn[slot] >= tbv}.  Queries are sorted
// by norm descending, so the kept queries are exactly this prefix.
__device__ __forceinline__ int lemma3_prefix(const float* qn_sub, int cnt, float tbv) {
  int lo = 0, hi = cnt;  // first slot with qn < tbv
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (qn_sub[mid] >= tbv) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Classification of one (user, query) filter score.  acc ~ (u/nu).(q*2^eq);
// thr_s = (tau_k/nu)*2^eq; E = qerr + |thr_s| 2^-22 (fp32 rounding of thr).
// returns 0 reject (Lemma 1: u.q < tau_k), 1 accept (u.q >= tau_k), 2 undecided.
__device__ __forceinline__ int classify(float acc, float thr_s, float qe) {
  float E = __fadd_ru(qe, fabsf(thr_s) * 2.384185791015625e-07f);
  if (__fadd_ru(acc, E) < thr_s) return 0;
  if (__fsub_rd(acc, E) >= thr_s) return 1;
  return 2;
}

// ------------------------------------------------------------------------------ Q2 + Q3 (SIMT)
template <int DPAD>
__global__ void __launch_bounds__(128)
k_query_simt(const __half* __restrict__ U16, int ldh, const float* __restrict__ thrk, const float* __restrict__ tbk,
             int bsz, int64_t nlb,
             const int32_t* __restrict__ perm_u, int64_t n, const __half* __restrict__ Q16,
             const float* __restrict__ qn, const float* __restrict__ qerr, const float* __restrict__ qscale,
             const int32_t* __restrict__ qperm, const int32_t* __restrict__ qcount, int flags,
             unsigned long long* __restrict__ ctr, AccSink acc_list, uint64_t* __restrict__ und_list,
             int64_t cap) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __half2* us = reinterpret_cast<__half2*>(smem_raw);        // [DPAD/2][128]
  __half2* qs = us + (DPAD / 2) * 128;                        // [kQB][DPAD/2]
  __shared__ int s_len;
  const int tile = blockIdx.x, s = blockIdx.y, tid = threadIdx.x;
  const int cnt = qcount[s];
  const float* qn_sub = qn + (int64_t)s * kQB;
  if (tid == 0) {
    unsigned long long pairs = 0, pruned = 0;
    const int len = tile_lemma3(tile, bsz, nlb, cnt, (flags & RMIPS_FLAG_NO_BLOCKS) != 0, tbk,
                                [&](float tbv) { return lemma3_prefix(qn_sub, cnt, tbv); }, pairs, pruned);
    s_len = len;
    atomicAdd(ctr + C_BLOCK_PAIRS, pairs);
    atomicAdd(ctr + C_BLOCK_PRUNED, pruned);
  }
  __syncthreads();
  const int len = s_len;
  if (len == 0) return;
  if (tid == 0) atomicAdd(ctr + C_TILES_SCORED, 1ull);
  const int64_t row = (int64_t)tile * 128 + tid;
  const bool live = row < n;
  for (int i = tid; i < 128 * (DPAD / 2); i += 128) {
    int r = i / (DPAD / 2), k2 = i % (DPAD / 2);
    int64_t gr = (int64_t)tile * 128 + r;
    us[k2 * 128 + r] = gr < n && 2 * k2 < ldh ? reinterpret_cast<const __half2*>(U16)[gr * (ldh / 2) + k2]
                                              : __floats2half2_rn(0.f, 0.f);
  }
  const __half2* qsrc = reinterpret_cast<const __half2*>(Q16) + (int64_t)s * kQB * (ldh / 2);
  for (int i = tid; i < len * (DPAD / 2); i += 128) {
    const int qr = i / (DPAD / 2), k2 = i - qr * (DPAD / 2);
    qs[i] = 2 * k2 < ldh ? qsrc[qr * (ldh / 2) + k2] : __floats2half2_rn(0.f, 0.f);
  }
  __syncthreads();
  const float sc = qscale[s];
  const float thr_s = live ? thrk[row] * sc : 0.f;
  const uint64_t uo = live ? (uint64_t)(uint32_t)perm_u[row] : 0;
  for (int q0 = 0; q0 < len; q0 += 8) {
    float a8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a8[j] = 0.f;
    for (int k2 = 0; k2 < DPAD / 2; ++k2) {
      float2 a = __half22float2(us[k2 * 128 + tid]);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int qq = min(q0 + j, len - 1);
        float2 bq = __half22float2(qs[qq * (DPAD / 2) + k2]);
        a8[j] = fmaf(a.x, bq.x, a8[j]);
        a8[j] = fmaf(a.y, bq.y, a8[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int slot = q0 + j;
      const bool ok = live && slot < len;
      int cls = ok ? classify(a8[j], thr_s, qerr[(int64_t)s * kQB + slot]) : 0;
      if ((flags & RMIPS_FLAG_FORCE_VERIFY) && cls == 1) cls = 2;
      const uint64_t qin = ok ? (uint64_t)(uint32_t)qperm[(int64_t)s * kQB + slot] : 0;
      warp_count(ok, ctr + C_SCORED);
      warp_count(ok && cls == 0, ctr + C_REJECTED);
      warp_count(ok && cls == 1, ctr + C_ACCEPT_FAST);
      acc_list.put(ok && cls == 1, (qin << 32) | uo, ctr + C_ACCEPTED_TOTAL, cap);
      warp_count(ok && cls == 1, ctr + C_ACC_REAL);
      warp_append_u64(ok && cls == 2, (qin << 32) | (uint64_t)row, ctr + C_UND_TOTAL, und_list, cap);
    }
  }
}

// ------------------------------------------------------------------------------ Q4
// u in R_k(q) <=> dot64(q, u) >= tau_k(u)  (reading R8; same dot routine as the build).
// One warp per undecided pair of the DENSE list (k_scan_compact packs the real records first: the filter
// reserves list slots in blocks, so the real pairs cluster, and a warp per slot window would run its
// cluster's pairs one after another): the lanes load 32 coordinates of q and u at a time (coalesced) and
// form their exact fp64 products; every lane then adds the products in index order, taking each one by
// a broadcast shuffle, so the sum is dot64's left-to-right fp64 sum bit for bit (each product of two fp32
// values is exact in fp64, so fma(a, b, s) and s + a*b round identically).
constexpr int C_SCAN_LIST = kNumCounters;      // (spare counter slot) pairs in the dense list
constexpr int C_SCAN_NEXT = kNumCounters + 1;  // (spare, zeroed per call) next pair for k_verify_scan_warp
__global__ void __launch_bounds__(256)
k_exact_decide(const float* __restrict__ q, const float* __restrict__ U32, const double* __restrict__ tauk,
               const int32_t* __restrict__ perm_u, int d, unsigned long long* __restrict__ ctr,
               const uint64_t* __restrict__ dense, AccSink acc_list, int64_t cap) {
  pdl_enter();  // (PDL: see launch_pdl)
  const int64_t total = (int64_t)min((unsigned long long)cap, ctr[C_SCAN_LIST]);
  const int lane = threadIdx.x & 31;
  const int64_t wstride = (int64_t)gridDim.x * (blockDim.x >> 5);
  unsigned n_und = 0, n_yes = 0;
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < total; i += wstride) {
    const uint64_t rec = dense[i];
    const uint32_t qin = (uint32_t)(rec >> 32);
    const int64_t row = (int64_t)(rec & 0xffffffffu);
    const float* qa = q + (int64_t)qin * d;
    const float* ua = U32 + row * d;
    double g = 0.0;
    // the first kPre chunks' products are loaded before the first add (one memory latency per pair
    // instead of one per 32 coordinates; a call's few hundred pairs are latency-bound)
    constexpr int kPre = 8;
    double pcs[kPre];
#pragma unroll
    for (int i = 0; i < kPre; ++i) {
      const int t = 32 * i + lane;
      pcs[i] = t < d ? (double)__ldg(qa + t) * (double)__ldg(ua + t) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < kPre; ++i) {
      if (32 * i >= d) break;
      const int nj = min(32, d - 32 * i);
#pragma unroll 8
      for (int jj = 0; jj < nj; ++jj) g = __dadd_rn(g, __shfl_sync(0xffffffffu, pcs[i], jj));
    }
    for (int c = 32 * kPre; c < d; c += 32) {
      const double pc = c + lane < d ? (double)__ldg(qa + c + lane) * (double)__ldg(ua + c + lane) : 0.0;
      const int nj = min(32, d - c);
#pragma unroll 8
      for (int jj = 0; jj < nj; ++jj) g = __dadd_rn(g, __shfl_sync(0xffffffffu, pc, jj));
    }
    ++n_und;
    if (g >= tauk[row]) {  // u in R_k(q) <=> dot64(q, u) >= tau_k(u)  (reading R8)
      ++n_yes;
      if (lane == 0) acc_list.put_one(((uint64_t)qin << 32) | (uint64_t)(uint32_t)perm_u[row], ctr + C_ACCEPTED_TOTAL, cap);
    }
  }
  if (lane == 0 && n_und) {
    atomicAdd(ctr + C_UNDECIDED, (unsigned long long)n_und);
    if (n_yes) {
      atomicAdd(ctr + C_EXACT_ACCEPT, (unsigned long long)n_yes);
      atomicAdd(ctr + C_ACC_REAL, (unsigned long long)n_yes);
    }
  }
}

// Q4 on a P' index (lists = exact top k_max over the first mprime norm-sorted items, reading
// NEXT-1 / DESIGN.md §8).  g = dot64(q, u); c' = #{listed j : L^j > g}:
//   g < L^k                                  -> no   (Lemma 1: k items of P' beat q)
//   k > m, or g >= ||u|| ||p_k|| (rounded up) -> yes  (Lemma 2)
//   g >= ||u|| ||p_{mprime+1}||  (rounded up) -> yes  (Cor. 1 at the first item after P': no item
//                                               outside P' can beat q, and c' < k inside it)
//   otherwise the pair goes to the scan over the items after P' with beats = c' (exact: P' items
//   outside the list score <= L^{k_max} <= L^k <= g, so exactly c' items of P' beat q).
// Decided records are overwritten with the sentinel; undecided ones keep theirs for k_verify_scan.
__global__ void k_exact_decide_pp(const float* __restrict__ q, const float* __restrict__ U32,
                                  const double* __restrict__ unorm, const double* __restrict__ pnorm,
                                  const double* __restrict__ tau, int64_t n, int64_t m, int64_t mprime, int k,
                                  const int32_t* __restrict__ perm_u, int d, unsigned long long* __restrict__ ctr,
                                  uint64_t* __restrict__ und_list, int32_t* __restrict__ scan_cnt,
                                  AccSink acc_list, int64_t cap) {
  const int64_t total = (int64_t)min((unsigned long long)cap, ctr[C_UND_TOTAL]);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const double slack = 1.0 + (d + 8) * 2.220446049250313e-16;  // as k_verify_scan's Cor. 1 test
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < total; base += stride) {
    const int64_t i = base + threadIdx.x;
    bool ok = i < total;
    bool yes = false, scan = false;
    uint64_t key = 0;
    uint64_t rec = ok ? und_list[i] : kSentinel;
    if (rec == kSentinel) ok = false;  // unused reserved slot
    if (ok) {
      const uint32_t qin = (uint32_t)(rec >> 32);
      const int64_t row = (int64_t)(rec & 0xffffffffu);
      const double g = dot64(q + (int64_t)qin * d, U32 + row * d, d);
      if (g >= tau[(int64_t)(k - 1) * n + row]) {
        const double un = unorm[row] * slack;
        if (k > m || g >= un * pnorm[k - 1] * slack || g >= un * pnorm[mprime] * slack) {
          yes = true;
        } else {
          int c = 0;
          for (int j = 0; j < k - 1; ++j) c += tau[(int64_t)j * n + row] > g;
          scan_cnt[i] = c;
          scan = true;
        }
      }
      key = ((uint64_t)qin << 32) | (uint64_t)(uint32_t)perm_u[row];
      if (!scan) und_list[i] = kSentinel;
    }
    warp_count(ok, ctr + C_UNDECIDED);
    warp_count(yes, ctr + C_EXACT_ACCEPT);
    acc_list.put(yes, key, ctr + C_ACCEPTED_TOTAL, cap);
    warp_count(yes, ctr + C_ACC_REAL);
  }
}

// ------------------------------------------------------------------------------ Q5
// Alg. 2 with Corollaries 1-2, readings R3/R4, for the undecided pairs.
// Items are visited in norm-descending order (Alg. 1 line 5).  Corollary 1 (yes): u.q >= ||u|| ||p_j||
// (both rounded up to cover the fp64 rounding of every later gamma) means no later item can beat q.
// Corollary 2 (no): once k items have gamma = p.u > u.q.  Falling off the end: yes (R4).
// Each gamma is first scored in fp32 (four independent FMA chains over the zero-padded row) with a
// rigorous bound |s - dot64(p, u)| <= E = (gamma32(pd/4 + 2) + gamma64(d)) ||p|| ||u|| (rounded up,
// plus an absolute term for subnormal products); only items with |s - u.q| <= E (or a non-finite s)
// are re-evaluated with the left-to-right fp64 sum, so every "beats" decision is the oracle's (R7).
//
// Layout (north star (d)): the scan streams the norm-sorted P32 through SHARED MEMORY, one tile of
// kScanRows rows at a time, and every warp of the CTA scores its pairs against the staged tile: a CTA
// batch of up to 32 pairs reads each tile from L2 / HBM once instead of once per pair.  Lane l scores
// item row l of a 32-row step (rows staged at an odd number of float4s per row: conflict-free 128-bit
// loads); the pair's u is broadcast from shared memory.  The batch ends when every pair decided.
// k_scan_compact first packs the real pairs (the exact-decide pass leaves sentinels) densely.
// start / beats0: the scan begins at item `start` with beats0 items already known to beat q (P' index:
// start = mprime, beats0 = c' from k_exact_decide_pp); 0 / NULL scans all of P.
constexpr int kScanWarps = 8;
__global__ void k_scan_compact(const uint64_t* __restrict__ und_list, const int32_t* __restrict__ beats0,
                               unsigned long long* __restrict__ ctr, int64_t cap, uint64_t* __restrict__ out_rec,
                               int32_t* __restrict__ out_beats) {
  pdl_enter();  // (PDL: see launch_pdl)
  const int64_t total = (int64_t)min((unsigned long long)cap, ctr[C_UND_TOTAL]);
  const int lane = threadIdx.x & 31;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x; i0 < total; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const uint64_t rec = i < total ? und_list[i] : kSentinel;
    const bool live = rec != kSentinel;
    const uint32_t bal = __ballot_sync(0xffffffffu, live);
    if (!bal) continue;
    unsigned long long base = 0;
    if (lane == __ffs(bal) - 1) base = atomicAdd(ctr + C_SCAN_LIST, (unsigned long long)__popc(bal));
    base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
    if (live) {
      const unsigned long long pos = base + __popc(bal & lanemask_lt());
      out_rec[pos] = rec;
      out_beats[pos] = beats0 ? beats0[i] : 0;
    }
  }
}

// Warp-per-pair form (P32 small enough to stay in L2, m pd 4 <= kScanL2Bytes): lane j scores item
// base + j straight from the sector-padded P32 rows (consecutive lanes read consecutive rows), so a pair
// stops at its own depth -- the tiled form's CTA batches run to their deepest pair, which costs more than
// it saves when the rows are L2 hits anyway (configs[1] P': 19 vs 29 ms).
constexpr int64_t kScanL2Bytes = (int64_t)64 << 20;
__global__ void __launch_bounds__(32 * kScanWarps)
k_verify_scan_warp(const float* __restrict__ q, const float* __restrict__ U32, const double* __restrict__ unorm,
                   const float* __restrict__ P32, const double* __restrict__ pnorm, const int32_t* __restrict__ perm_u,
                   int64_t m, int d, int pd, int k, unsigned long long* __restrict__ ctr,
                   const uint64_t* __restrict__ scan_rec, const int32_t* __restrict__ scan_beats, AccSink acc_list,
                   int64_t cap, int64_t start, bool count_undecided) {
  extern __shared__ __align__(16) float sw[];  // [kScanWarps][pd]: the pair's u, fp32, zero-padded to pd
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float* uw = sw + (size_t)w * pd;
  const int64_t npairs = (int64_t)min((unsigned long long)cap, ctr[C_SCAN_LIST]);
  const double slack = 1.0 + (d + 8) * 2.220446049250313e-16;
  const double n32 = pd / 4 + 2, g32 = n32 * 5.9604644775390625e-08 / (1.0 - n32 * 5.9604644775390625e-08);
  const double g64 = (d + 2) * 1.1102230246251565e-16 / (1.0 - (d + 2) * 1.1102230246251565e-16);
  const double efac = (g32 + g64) * slack * slack * (1.0 + 1e-6);
  const int nq4 = pd / 4;
  // pairs are taken one at a time from a counter: scan lengths differ by orders of magnitude (each pair
  // stops at its own depth), and a static stride left each launch waiting on its longest warps
  for (;;) {
    unsigned long long gi = 0;
    if (lane == 0) gi = atomicAdd(ctr + C_SCAN_NEXT, 1ull);
    const int64_t i = (int64_t)__shfl_sync(0xffffffffu, gi, 0);
    if (i >= npairs) break;
    const uint64_t rec = scan_rec[i];
    const uint32_t qin = (uint32_t)(rec >> 32);
    const int64_t row = (int64_t)(rec & 0xffffffffu);
    const float* u = U32 + row * d;
    __syncwarp();
    for (int t = lane; t < pd; t += 32) uw[t] = t < d ? __ldg(u + t) : 0.f;
    __syncwarp();
    const double uq = dot64(q + (int64_t)qin * d, u, d);
    const double un = unorm[row];
    const double unc = un * slack;
    int beats = scan_beats[i];
    int64_t scanned = 0, exact = 0;
    bool yes = true, decided = false;
    for (int64_t base = start; base < m && !decided; base += 32) {
      const int nrow = (int)min((int64_t)32, m - base);
      const int64_t j = base + lane;
      const bool in = lane < nrow;
      const double pn = in ? pnorm[j] : 0.0;
      const bool cor1 = in && (uq >= unc * pn * slack);
      const uint32_t ycut = __ballot_sync(0xffffffffu, cor1);  // first lane where Cor. 1 fires
      const int lim = ycut ? (__ffs(ycut) - 1) : nrow;
      bool beat = false;
      if (lane < lim) {
        const float4* pr = reinterpret_cast<const float4*>(P32 + j * pd);
        const float4* u4 = reinterpret_cast<const float4*>(uw);
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 4
        for (int t = 0; t < nq4; ++t) {
          const float4 x = __ldg(pr + t), y = u4[t];
          a0 = fmaf(x.x, y.x, a0);
          a1 = fmaf(x.y, y.y, a1);
          a2 = fmaf(x.z, y.z, a2);
          a3 = fmaf(x.w, y.w, a3);
        }
        const float sc = (a0 + a1) + (a2 + a3);
        const double E = efac * pn * un + 1e-40;
        const double sd = (double)sc;
        if (isfinite(sc) && sd - E > uq) {
          beat = true;
        } else if (!(isfinite(sc) && sd + E <= uq)) {  // inside the band: the exact fp64 value
          double g = 0.0;
          const float* prf = P32 + j * pd;
          for (int t = 0; t < d; ++t) g = __fma_rn((double)__ldg(prf + t), (double)uw[t], g);
          beat = g > uq;
          ++exact;
        }
      }
      scanned += lim;
      const uint32_t bb = __ballot_sync(0xffffffffu, beat);
      const int nb = __popc(bb);
      if (beats + nb >= k) { yes = false; decided = true; }
      else if (ycut) { yes = true; decided = true; }
      beats += nb;
    }
    for (int o = 16; o; o >>= 1) exact += __shfl_xor_sync(0xffffffffu, exact, o);
    if (lane == 0) {
      atomicAdd(ctr + C_SCANS, 1ull);
      atomicAdd(ctr + C_ITEMS_SCANNED, (unsigned long long)scanned);
      atomicAdd(ctr + C_SCAN_EXACT, (unsigned long long)exact);
      if (count_undecided) atomicAdd(ctr + C_UNDECIDED, 1ull);
      if (yes) {
        atomicAdd(ctr + C_EXACT_ACCEPT, 1ull);
        atomicAdd(ctr + C_ACC_REAL, 1ull);
        acc_list.put_one(((uint64_t)qin << 32) | (uint64_t)(uint32_t)perm_u[row], ctr + C_ACCEPTED_TOTAL, cap);
      }
    }
  }
}

// Tiled form (P32 larger than kScanL2Bytes): pw pairs per warp (4 for pd <= 256, else 1); rows staged
// per tile: 64 (pd <= 256) or 32
__global__ void __launch_bounds__(32 * kScanWarps)
k_verify_scan(const float* __restrict__ q, const float* __restrict__ U32, const double* __restrict__ unorm,
              const float* __restrict__ P32, const double* __restrict__ pnorm, const int32_t* __restrict__ perm_u,
              int64_t m, int d, int pd, int k, unsigned long long* __restrict__ ctr,
              const uint64_t* __restrict__ scan_rec, const int32_t* __restrict__ scan_beats, AccSink acc_list,
              int64_t cap, int64_t start, bool count_undecided, int pw, int rows) {
  extern __shared__ __align__(16) float ssc[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int s4 = (pd / 4) | 1;                      // row stride in float4 (odd: conflict-free LDS.128)
  float4* tile = reinterpret_cast<float4*>(ssc);    // [rows][s4]
  float* su = ssc + (size_t)rows * s4 * 4;          // [kScanWarps * pw][pd]
  __shared__ int s_live;
  const int64_t npairs = (int64_t)min((unsigned long long)cap, ctr[C_SCAN_LIST]);
  const double slack = 1.0 + (d + 8) * 2.220446049250313e-16;
  const double n32 = pd / 4 + 2, g32 = n32 * 5.9604644775390625e-08 / (1.0 - n32 * 5.9604644775390625e-08);
  const double g64 = (d + 2) * 1.1102230246251565e-16 / (1.0 - (d + 2) * 1.1102230246251565e-16);
  const double efac = (g32 + g64) * slack * slack * (1.0 + 1e-6);
  const int nq4 = pd / 4;
  const int per_cta = kScanWarps * pw;
  constexpr int kMaxPw = 4;
  for (int64_t b0 = (int64_t)blockIdx.x * per_cta; b0 < npairs; b0 += (int64_t)gridDim.x * per_cta) {
    // this warp's pairs: u staged, u.q and ||u|| computed, state in registers (lane-uniform)
    uint32_t qin[kMaxPw];
    int64_t row[kMaxPw];
    double uq[kMaxPw], un[kMaxPw];
    int beats[kMaxPw];
    bool active[kMaxPw], yes[kMaxPw];
    int64_t scanned = 0, exact = 0;
#pragma unroll
    for (int p = 0; p < kMaxPw; ++p) {
      const int64_t i = b0 + w * pw + p;
      active[p] = p < pw && i < npairs;
      yes[p] = true;
      qin[p] = 0, row[p] = 0, uq[p] = 0.0, un[p] = 0.0, beats[p] = 0;
      if (active[p]) {
        const uint64_t rec = scan_rec[i];
        qin[p] = (uint32_t)(rec >> 32);
        row[p] = (int64_t)(rec & 0xffffffffu);
        const float* u = U32 + row[p] * d;
        float* uw = su + (size_t)(w * pw + p) * pd;
        for (int t = lane; t < pd; t += 32) uw[t] = t < d ? __ldg(u + t) : 0.f;
        uq[p] = dot64(q + (int64_t)qin[p] * d, u, d);
        un[p] = unorm[row[p]];
        beats[p] = scan_beats[i];
      }
    }
    __syncwarp();
    for (int64_t base = start; base < m; base += rows) {
      // any pair of the CTA still undecided?  (also orders the previous tile's reads before the reload)
      const bool mine = active[0] | active[1] | active[2] | active[3];
      if (threadIdx.x == 0) s_live = 0;
      __syncthreads();
      if (mine && lane == 0) s_live = 1;
      __syncthreads();
      if (!s_live) break;
      const int nrow = (int)min((int64_t)rows, m - base);
      for (int r = w; r < nrow; r += kScanWarps) {  // stage the tile: one warp per row, float4 over the row
        const float4* src = reinterpret_cast<const float4*>(P32 + (base + r) * pd);
        for (int t = lane; t < nq4; t += 32) tile[r * s4 + t] = __ldg(src + t);
      }
      __syncthreads();
      for (int st = 0; st < nrow; st += 32) {
        const int nr = min(32, nrow - st);
        const int64_t j = base + st + lane;
        const bool in = lane < nr;
        const double pn = in ? pnorm[j] : 0.0;
        const float4* pr = tile + (st + lane) * s4;
#pragma unroll
        for (int p = 0; p < kMaxPw; ++p) {
          if (!active[p]) continue;  // (warp-uniform)
          const double unc = un[p] * slack;
          const bool cor1 = in && (uq[p] >= unc * pn * slack);
          const uint32_t ycut = __ballot_sync(0xffffffffu, cor1);  // first lane where Cor. 1 fires
          const int lim = ycut ? (__ffs(ycut) - 1) : nr;
          const float4* u4 = reinterpret_cast<const float4*>(su + (size_t)(w * pw + p) * pd);
          bool beat = false;
          if (lane < lim) {
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 4
            for (int t = 0; t < nq4; ++t) {
              const float4 x = pr[t], y = u4[t];
              a0 = fmaf(x.x, y.x, a0);
              a1 = fmaf(x.y, y.y, a1);
              a2 = fmaf(x.z, y.z, a2);
              a3 = fmaf(x.w, y.w, a3);
            }
            const float sc = (a0 + a1) + (a2 + a3);
            const double E = efac * pn * un[p] + 1e-40;
            const double sd = (double)sc;
            if (isfinite(sc) && sd - E > uq[p]) {
              beat = true;
            } else if (!(isfinite(sc) && sd + E <= uq[p])) {  // inside the band: the exact fp64 value
              const float* prf = reinterpret_cast<const float*>(pr);
              const float* uf = su + (size_t)(w * pw + p) * pd;
              double g = 0.0;
              for (int t = 0; t < d; ++t) g = __fma_rn((double)prf[t], (double)uf[t], g);
              beat = g > uq[p];
              ++exact;
            }
          }
          scanned += lim;
          const uint32_t bb = __ballot_sync(0xffffffffu, beat);
          // Alg. 2 visits items in order: the k-th beat (if any) decides "no"
          const int nb = __popc(bb);
          if (beats[p] + nb >= k) {
            yes[p] = false;
            active[p] = false;
          } else if (ycut) {
            active[p] = false;  // yes
          }
          beats[p] += nb;
        }
      }
    }
    for (int o = 16; o; o >>= 1) exact += __shfl_xor_sync(0xffffffffu, exact, o);
    if (lane == 0) {
      int nsc = 0, nyes = 0;
#pragma unroll
      for (int p = 0; p < kMaxPw; ++p) {
        const int64_t i = b0 + w * pw + p;
        if (p >= pw || i >= npairs) continue;
        ++nsc;
        if (yes[p]) {
          ++nyes;
          acc_list.put_one(((uint64_t)qin[p] << 32) | (uint64_t)(uint32_t)perm_u[row[p]], ctr + C_ACCEPTED_TOTAL, cap);
        }
      }
      if (nsc) {
        atomicAdd(ctr + C_SCANS, (unsigned long long)nsc);
        atomicAdd(ctr + C_ITEMS_SCANNED, (unsigned long long)scanned);
        atomicAdd(ctr + C_SCAN_EXACT, (unsigned long long)exact);
        if (count_undecided) atomicAdd(ctr + C_UNDECIDED, (unsigned long long)nsc);  // (P': counted already)
        if (nyes) {
          atomicAdd(ctr + C_EXACT_ACCEPT, (unsigned long long)nyes);
          atomicAdd(ctr + C_ACC_REAL, (unsigned long long)nyes);
        }
      }
    }
  }
}

// ------------------------------------------------------------------------------ Q6
__global__ void k_offsets(const uint64_t* __restrict__ keys, int64_t total, int b, int64_t* __restrict__ offsets) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > b) return;
  uint64_t target = (uint64_t)i << 32;
  int64_t lo = 0, hi = total;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if (keys[mid] < target) lo = mid + 1; else hi = mid;
  }
  offsets[i] = lo;
}

__global__ void k_copy_ids(const uint64_t* __restrict__ keys, int64_t total, int32_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < total) out[i] = (int32_t)(keys[i] & 0xffffffffu);
}

// ------------------------------------------------------------------------------ host side
static inline unsigned nblk(int64_t work, int t) { return (unsigned)((work + t - 1) / t); }

cudaError_t query_prep(QueryCtx& c, cudaStream_t st) {
  rmips_index_s* x = c.idx;
  const unsigned grid = (unsigned)(c.nsub * kPrepCtas);
  CK_PDL(launch_pdl(k_query_norms, dim3(grid), dim3(32 * kPrepWarps), 0, st, c.q, c.b, x->d, c.qnrm, c.qcmax, c.flags_dev));
  count_launch();
  CK_PDL(launch_pdl(k_query_finish, dim3(grid), dim3(32 * kPrepWarps), 0, st, c.q, c.b, x->d, x->ldh, x->c1, x->c2, c.qnrm, c.qcmax, c.Q16, c.qn,
                                                   c.qerr, c.qscale, c.qperm, c.qcount));
  count_launch();
  return cudaGetLastError();
}

template <int DPAD>
static cudaError_t launch_query_simt(QueryCtx& c, cudaStream_t st) {
  rmips_index_s* x = c.idx;
  size_t smem = (size_t)(DPAD / 2) * 128 * 4 + (size_t)kQB * (DPAD / 2) * 4;
  cudaError_t e = set_smem_attr((const void*)k_query_simt<DPAD>, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)x->nblocks, (unsigned)c.nsub);
  k_query_simt<DPAD><<<grid, 128, smem, st>>>(x->U16, x->ldh, x->thr + (int64_t)(c.k - 1) * x->n,
                                              x->tb + (int64_t)(c.k - 1) * x->nlb, x->bsz, x->nlb, x->perm_u, x->n, c.Q16, c.qn,
                                              c.qerr, c.qscale, c.qperm, c.qcount, c.flags, c.counters, AccSink{c.acc, c.bits, c.nw, c.dirty, c.nbr}, c.und,
                                              c.cap); count_launch();
  return cudaGetLastError();
}

cudaError_t query_filter_simt(QueryCtx& c, cudaStream_t st) {
  if (c.idx->n == 0) return cudaSuccess;
  switch (c.idx->dpad) {
    case 64: return launch_query_simt<64>(c, st);
    case 128: return launch_query_simt<128>(c, st);
    case 192: return launch_query_simt<192>(c, st);
    case 256: return launch_query_simt<256>(c, st);
    default: return cudaErrorInvalidValue;
  }
}

#define CK_RET(expr)                     \
  do {                                   \
    const cudaError_t e_ = (expr);       \
    if (e_ != cudaSuccess) return e_;    \
  } while (0)

// Alg. 2 over the undecided pairs: compaction into the dense scan list, then the tiled scan.
static cudaError_t launch_scan(QueryCtx& c, int64_t start, const int32_t* beats0, bool count_und, cudaStream_t st) {
  rmips_index_s* x = c.idx;
  k_scan_compact<<<148 * 4, 256, 0, st>>>(c.und, beats0, c.counters, c.cap, c.scan_rec, c.scan_beats);
  count_launch();
  bool tiled = (int64_t)x->m * x->pd * 4 > kScanL2Bytes;
#ifdef RMIPS_DEV
  if (getenv("RMIPS_SCAN_TILED")) tiled = true;  // (development library: the tiled form on small P)
#endif
  if (!tiled) {
    const size_t smem = (size_t)kScanWarps * x->pd * sizeof(float);
    if (smem > 48 * 1024)
      CK_RET(set_smem_attr((const void*)k_verify_scan_warp, (int)smem));
    k_verify_scan_warp<<<148 * 8, 32 * kScanWarps, smem, st>>>(c.q, x->U32, x->unorm, x->P32, x->pnorm, x->perm_u,
                                                                x->m, x->d, x->pd, c.k, c.counters, c.scan_rec,
                                                                c.scan_beats, AccSink{c.acc, c.bits, c.nw, c.dirty, c.nbr}, c.cap, start,
                                                                count_und);
    count_launch();
    return cudaGetLastError();
  }
  const int pw = x->pd <= 256 ? 4 : 1, rows = x->pd <= 256 ? 64 : 32;
  const int s4 = (x->pd / 4) | 1;
  const size_t smem = (size_t)rows * s4 * 16 + (size_t)kScanWarps * pw * x->pd * sizeof(float);
  if (smem > 48 * 1024) CK_RET(set_smem_attr((const void*)k_verify_scan, (int)smem));
  k_verify_scan<<<148 * 2, 32 * kScanWarps, smem, st>>>(c.q, x->U32, x->unorm, x->P32, x->pnorm, x->perm_u, x->m, x->d,
                                                        x->pd, c.k, c.counters, c.scan_rec, c.scan_beats,
                                                        AccSink{c.acc, c.bits, c.nw, c.dirty, c.nbr}, c.cap, start, count_und, pw, rows);
  count_launch();
  return cudaGetLastError();
}

cudaError_t query_exact(QueryCtx& c, cudaStream_t st) {
  rmips_index_s* x = c.idx;
  if (x->n == 0) return cudaSuccess;
  if (c.flags & RMIPS_FLAG_VERIFY_SCAN) {  // every undecided pair scans all of P (Alg. 2)
    CK_RET(launch_scan(c, 0, nullptr, true, st));
  } else if (x->mprime < x->m) {  // P' index: Lemmas 1-2 / Cor. 1 per pair, then the scan after P'
    k_exact_decide_pp<<<148 * 8, 256, 0, st>>>(c.q, x->U32, x->unorm, x->pnorm, x->tau, x->n, x->m, x->mprime, c.k,
                                               x->perm_u, x->d, c.counters, c.und, c.scan_cnt, AccSink{c.acc, c.bits, c.nw, c.dirty, c.nbr}, c.cap);
    count_launch();
    CK_RET(launch_scan(c, x->mprime, c.scan_cnt, false, st));
  } else {
    CK_PDL(launch_pdl(k_scan_compact, dim3(148 * 4), dim3(256), 0, st, c.und, nullptr, c.counters, c.cap, c.scan_rec,
                      c.scan_beats));
    count_launch();
    CK_PDL(launch_pdl(k_exact_decide, dim3(148 * 4), dim3(256), 0, st, c.q, x->U32, x->tau + (int64_t)(c.k - 1) * x->n, x->perm_u, x->d,
                                            c.counters, c.scan_rec, AccSink{c.acc, c.bits, c.nw, c.dirty, c.nbr}, c.cap));
    count_launch();
  }
  return cudaGetLastError();
}

// Fast output path when b * n < 2^32: accepted (q, user) pairs packed as one 32-bit key q * n + u,
// so the radix sort needs ceil(log2(b n)) bits (4 passes) instead of 64.
__global__ void k_pack32(const uint64_t* __restrict__ acc, int64_t total, uint32_t n, uint32_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < total) {
    const uint64_t r = acc[i];
    out[i] = r == kSentinel ? 0xffffffffu : (uint32_t)(r >> 32) * n + (uint32_t)(r & 0xffffffffu);
  }
}
__global__ void k_offsets32(const uint32_t* __restrict__ keys, int64_t total, int b, uint32_t n,
                            int64_t* __restrict__ offsets) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > b) return;
  const uint64_t target = (uint64_t)i * n;
  int64_t lo = 0, hi = total;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((uint64_t)keys[mid] < target) lo = mid + 1; else hi = mid;
  }
  offsets[i] = lo;
}
__global__ void k_copy_ids32(const uint32_t* __restrict__ keys, int64_t total, uint32_t n, int32_t* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < total) out[i] = (int32_t)(keys[i] % n);
}

// Bit-matrix output (QueryCtx::bits): the b x n matrix is cut into warp chunks of kChunkWords words of
// one query row; lane l of a chunk's warp owns block l (32 consecutive words, 1024 users).  Only blocks
// whose dirty byte is set (AccSink::set) are read: a 256-query batch of configs[4] sets ~11,000 of
// 256 M bits, so the passes read the 0.25 MB of dirty bytes and ~1 MB of words instead of the 32 MB
// matrix.  Pass 1 counts the set bits of every chunk, a scan gives every chunk's first output position
// (the chunks are in (query, user) order), and pass 2 re-reads the dirty blocks, writes the ids in
// ascending user order (a warp prefix sum over the lanes' block counts) and clears the words and dirty
// bytes it read, so both are all zero again for the next batch (they are memset only when their place
// in the workspace changes).  Every warp works independently.
constexpr int kChunkWords = 1024;
constexpr int kBitsThreads = 256;
constexpr int C_BITS_TICKET = kNumCounters + 2;  // (spare, zeroed per call / batch) k_bits_count CTAs done
__global__ void __launch_bounds__(kBitsThreads)
k_bits_count(const uint32_t* __restrict__ bits, const uint8_t* __restrict__ dirty, int64_t nw, int64_t nbr,
             int64_t nchunk_total, int64_t* __restrict__ counts, int64_t* __restrict__ local_off,
             int64_t* __restrict__ cta_sum, int64_t* __restrict__ cta_off,
             unsigned long long* __restrict__ ticket) {  // ticket: zeroed before the launch
  pdl_enter();  // (PDL: see launch_pdl)
  constexpr int kWarps = kBitsThreads / 32;
  __shared__ int last;
  __shared__ int64_t wsum[kWarps];
  const int64_t g = (blockIdx.x * (int64_t)kBitsThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int cnt = 0;
  if (g < nchunk_total) {  // (no early return: the CTA sync and the last CTA's scan below need every thread)
    const int64_t per_row = (nw + kChunkWords - 1) / kChunkWords;
    const int64_t q = g / per_row, c = g - q * per_row;
    const int64_t blk = c * 32 + lane;  // this lane's block of the row
    if (blk < nbr && dirty[q * nbr + blk]) {
      const uint32_t* wp = bits + q * nw + blk * 32;
      const int nwb = (int)min((int64_t)32, nw - blk * 32);
#pragma unroll
      for (int i = 0; i < 32; ++i) cnt += i < nwb ? __popc(wp[i]) : 0;  // (all 32 loads in flight)
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  }
  // two levels: each chunk's offset within its CTA (local_off) and every CTA's total (cta_sum); the last
  // CTA to finish scans the CTA totals (cta_off), k_bits_emit adds the two
  if (lane == 0) wsum[wid] = cnt;
  __syncthreads();
  if (lane == 0 && g < nchunk_total) {
    int64_t pre = 0;
    for (int i = 0; i < wid; ++i) pre += wsum[i];
    counts[g] = cnt;
    local_off[g] = pre;
  }
  if (threadIdx.x == 0) {
    int64_t tot = 0;
    for (int i = 0; i < kWarps; ++i) tot += wsum[i];
    cta_sum[blockIdx.x] = tot;
    __threadfence();  // (every write the last CTA reads is thread 0's, published before its ticket)
    last = atomicAdd(ticket, 1ull) == (unsigned long long)gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // exclusive scan of the gridDim.x CTA totals: thread t owns the contiguous run [t per, (t + 1) per)
  const int64_t nc = gridDim.x;
  const int t = threadIdx.x;
  const int64_t per = (nc + kBitsThreads - 1) / kBitsThreads;
  const int64_t a = (int64_t)t * per, e = a + per < nc ? a + per : nc;
  int64_t sum = 0;
  for (int64_t i = a; i < e; ++i) sum += __ldcg(cta_sum + i);
  int64_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  __syncthreads();  // (wsum is reused)
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  int64_t run = incl - sum;
#pragma unroll
  for (int i = 0; i < kWarps; ++i) run += i < wid ? wsum[i] : 0;
  for (int64_t i = a; i < e; ++i) {
    cta_off[i] = run;
    run += __ldcg(cta_sum + i);
  }
}
__global__ void __launch_bounds__(kBitsThreads)
k_bits_emit(uint32_t* __restrict__ bits, uint8_t* __restrict__ dirty, int64_t nw, int64_t nbr, int b,
            int64_t nchunk_total, const int64_t* __restrict__ counts, const int64_t* __restrict__ local_off,
            const int64_t* __restrict__ cta_sum, const int64_t* __restrict__ cta_off,
            int64_t capacity, int64_t* __restrict__ offsets, int32_t* __restrict__ out,
            const int64_t* __restrict__ obase, int64_t* __restrict__ obase_next,
            const unsigned long long* __restrict__ ctr, const int* __restrict__ flags_dev,
            unsigned long long* __restrict__ fold) {
  pdl_enter();  // (PDL: see launch_pdl)
  const int64_t g = (blockIdx.x * (int64_t)kBitsThreads + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (g >= nchunk_total) return;
  if (fold && g == nchunk_total - 1) {
    // batched calls: this batch's counters folded into the call's (sums; the largest pair-workspace
    // need; the OR of the error flags), read by the host once after the last batch
    for (int i = lane; i < kNumCounters; i += 32) fold[i] += ctr[i];
    if (lane == 0) {
      const unsigned long long need = ctr[C_ACCEPTED_TOTAL] > ctr[C_UND_TOTAL] ? ctr[C_ACCEPTED_TOTAL] : ctr[C_UND_TOTAL];
      if (need > fold[kNumCounters]) fold[kNumCounters] = need;
      fold[kNumCounters + 1] |= (unsigned long long)(unsigned)flags_dev[0];
    }
  }
  const int64_t per_row = (nw + kChunkWords - 1) / kChunkWords;
  const int64_t q = g / per_row, c = g - q * per_row;
  // obase (batched calls, rmips_query_batches): the ids of the earlier batches already in `out`; this
  // batch's running total goes to obase_next (a different word: every block reads obase)
  const int64_t b0 = obase ? *obase : 0;
  const int64_t lc = (nchunk_total - 1) / (kBitsThreads / 32);  // the last CTA of the count pass
  const int64_t total = b0 + cta_off[lc] + cta_sum[lc];
  const bool fits = total <= capacity;  // ids only when all of them fit (as the sorted-key path)
  const int64_t base = b0 + cta_off[g / (kBitsThreads / 32)] + local_off[g];
  if (lane == 0) {
    if (c == 0) offsets[q] = base;
    if (g == nchunk_total - 1) {
      offsets[b] = total;
      if (obase_next) *obase_next = total;
    }
  }
  if (counts[g] == 0) return;  // (warp-uniform) nothing set in this chunk
  const int64_t blk = c * 32 + lane;
  const bool mine = blk < nbr && dirty[q * nbr + blk];
  uint32_t* wp = bits + q * nw + blk * 32;
  const int nwb = mine ? (int)min((int64_t)32, nw - blk * 32) : 0;
  int cnt = 0;
  uint32_t wv[32];  // the block's words, every load in flight at once
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    wv[i] = i < nwb ? wp[i] : 0u;
    cnt += __popc(wv[i]);
  }
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += x;
  }
  if (mine) {
    int64_t pos = base + incl - cnt;
    const int32_t u_blk = (int32_t)(blk * 1024);
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      uint32_t w = wv[i];
      if (!w) continue;
      wp[i] = 0u;
      if (fits) {
        const int32_t u0 = u_blk + 32 * i;
        while (w) {
          const int bit = __ffs(w) - 1;
          w &= w - 1;
          out[pos++] = u0 + bit;
        }
      }
    }
    dirty[q * nbr + blk] = 0;
  }
}

size_t query_scan_bytes(int64_t items) {
  size_t a = 0;
  cub::DeviceScan::ExclusiveSum((void*)nullptr, a, (const int64_t*)nullptr, (int64_t*)nullptr, (int)items);
  return a;
}
int64_t query_bits_chunks(int b, int64_t nw) { return (int64_t)b * ((nw + kChunkWords - 1) / kChunkWords); }

cudaError_t query_output_bits(QueryCtx& c, int64_t* offsets, int32_t* user_ids, int64_t capacity, cudaStream_t st,
                              const int64_t* obase, int64_t* obase_next, unsigned long long* fold) {
  const int64_t nch = query_bits_chunks(c.b, c.nw);
  // (the sort's space is unused on this path: 2 nch + 2 grid <= 3 nch words, ensure_ws)
  const unsigned grid = (unsigned)((nch * 32 + kBitsThreads - 1) / kBitsThreads);
  int64_t* counts = reinterpret_cast<int64_t*>(c.acc_sorted);
  int64_t* local_off = counts + nch;
  int64_t* cta_sum = local_off + nch;
  int64_t* cta_off = cta_sum + grid;
  // the CTA totals are scanned by the count kernel's last CTA (no separate scan launch)
  CK_PDL(launch_pdl(k_bits_count, dim3(grid), dim3(kBitsThreads), 0, st, c.bits, c.dirty, c.nw, c.nbr, nch, counts,
                    local_off, cta_sum, cta_off, c.counters + C_BITS_TICKET));
  count_launch();
  CK_PDL(launch_pdl(k_bits_emit, dim3(grid), dim3(kBitsThreads), 0, st, c.bits, c.dirty, c.nw, c.nbr, c.b, nch, counts,
                    local_off, cta_sum, cta_off, capacity,
                                              offsets, user_ids, obase, obase_next, c.counters, c.flags_dev, fold));
  count_launch();
  return cudaGetLastError();
}

static bool use_keys32(const QueryCtx& c) { return c.idx->n > 0 && (uint64_t)c.b * (uint64_t)c.idx->n < (1ull << 32); }

size_t query_cub_bytes(int64_t cap) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortKeys((void*)nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int)cap, 0, 64);
  cub::DeviceRadixSort::SortKeys((void*)nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)cap, 0, 32);
  return a > b ? a : b;
}

// total = number of accepted keys (host-known after the mid-call sync).
cudaError_t query_sort(QueryCtx& c, int64_t total, int end_bit, cudaStream_t st) {
  size_t tb = c.cub_bytes;
  c.sorted_n = total;
  if (total == 0) return cudaSuccess;
  if (use_keys32(c)) {
    // packed keys in the first half of acc_sorted's space, sorted into the second half (both fit: the
    // workspace holds cap 8-byte records)
    uint32_t* kin = reinterpret_cast<uint32_t*>(c.acc_sorted);
    uint32_t* kout = kin + total;
    k_pack32<<<nblk(total, 256), 256, 0, st>>>(c.acc, total, (uint32_t)c.idx->n, kin);
    count_launch();
    // real keys are < span; the sentinel 0xffffffff must sort after them on the low `bits` bits,
    // so 2^bits > span (a power-of-two span would otherwise tie its largest key with the sentinel)
    const uint64_t span = (uint64_t)c.b * (uint64_t)c.idx->n;
    int bits = 1;
    while (bits < 32 && (1ull << bits) <= span) ++bits;
    count_launch(kCubSortKernels);
    return cub::DeviceRadixSort::SortKeys(c.cub_tmp, tb, kin, kout, (int)total, 0, bits, st);
  }
  count_launch(kCubSortKernels);
  return cub::DeviceRadixSort::SortKeys(c.cub_tmp, tb, c.acc, c.acc_sorted, (int)total, 0, end_bit, st);
}

cudaError_t query_output(QueryCtx& c, int64_t* offsets, int32_t* user_ids, int64_t capacity, cudaStream_t st) {
  // offsets from the sorted keys; ids copied only if they fit
  const int64_t total = c.idx->stats.result_total;
  if (use_keys32(c)) {
    const uint32_t* keys = reinterpret_cast<const uint32_t*>(c.acc_sorted) + c.sorted_n;
    const uint32_t n32 = (uint32_t)c.idx->n;
    k_offsets32<<<nblk(c.b + 1, 256), 256, 0, st>>>(keys, total, c.b, n32, offsets); count_launch();
    if (total <= capacity && total > 0) {
      k_copy_ids32<<<nblk(total, 256), 256, 0, st>>>(keys, total, n32, user_ids);
      count_launch();
    }
    return cudaGetLastError();
  }
  k_offsets<<<nblk(c.b + 1, 256), 256, 0, st>>>(c.acc_sorted, total, c.b, offsets); count_launch();
  if (total <= capacity && total > 0) k_copy_ids<<<nblk(total, 256), 256, 0, st>>>(c.acc_sorted, total, user_ids); count_launch();
  return cudaGetLastError();
}

}  // namespace rmips
