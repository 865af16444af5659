// cand.cuh -- per-user-row top-k_max CANDIDATE filter, the epilogue of the build contraction.
//
// Alg. 1 lines 7-9 compute, for every user, the k_max largest inner products.
// On the GPU the |Q| x |P| score matrix is produced tile by tile (tensor cores or FFMA) in a
// reduced precision whose error is bounded per item by perr[p] (common.cuh).
// Each epilogue thread owns one user row r and keeps
//   theta_r : a valid lower bound (scaled units) of the k_max-th largest TRUE score seen so far
//             = the k_max-th largest lower bound lo = s~ - perr among its candidates;
//   a candidate buffer (value s~, item position) in shared memory, kCand slots.
// An item is appended iff s~ + perr >= theta_r (it may still be in the final top-k_max); when a
// row's buffer nears full, the warp cooperatively recomputes theta_r (radix select of the
// k_max-th largest lo) and drops candidates whose upper bound s~ + perr < theta_r.  Every true
// top-k_max item has s >= tau_kmax >= theta_r at all times, so it is never rejected or dropped
// (DESIGN.md §5 proof).  A row whose buffer cannot be compacted below kCand - 32 (massive ties)
// is flagged and recomputed exactly by the fallback kernel.
#pragma once
#include "common.cuh"

namespace rmips {

struct CandRow {
  float theta;   // running lower bound (scaled units); +inf once the row overflowed
  int cnt;       // live candidates in this row's buffer
};

// Warp-cooperative refresh of lane L's row.  All 32 lanes must call it (warp-uniform L).
// cv/ci: this warp's rows' buffers; row of lane L is cv + L*kCandPitch.
__device__ __forceinline__ void cand_refresh_lane(int L, CandRow& me, float* cv, int* ci,
                                                  const float* __restrict__ perr, int kmax,
                                                  bool* overflow_me) {
  const int lane = threadIdx.x & 31;
  const int cn = __shfl_sync(0xffffffffu, me.cnt, L);
  const float th = __shfl_sync(0xffffffffu, me.theta, L);
  float* vr = cv + L * kCandPitch;
  int* ir = ci + L * kCandPitch;
  float v[kCand / 32], e[kCand / 32];
  int id[kCand / 32];
  bool valid[kCand / 32];
#pragma unroll
  for (int t = 0; t < kCand / 32; ++t) {
    int i = lane + 32 * t;
    valid[t] = i < cn;
    v[t] = valid[t] ? vr[i] : 0.f;
    id[t] = valid[t] ? ir[i] : 0;
    e[t] = valid[t] ? __ldg(perr + id[t]) : 0.f;
  }
  float thn = th;
  if (cn >= kmax) {
    // radix select: largest key T (20 significant bits) with #{lo >= T} >= kmax.
    uint32_t key[kCand / 32];
#pragma unroll
    for (int t = 0; t < kCand / 32; ++t) key[t] = valid[t] ? f2key(__fsub_rd(v[t], e[t])) : 0u;
    uint32_t T = 0;
#pragma unroll 1
    for (int b = 31; b >= 12; --b) {
      uint32_t c = T | (1u << b);
      int count = 0;
#pragma unroll
      for (int t = 0; t < kCand / 32; ++t) count += __popc(__ballot_sync(0xffffffffu, key[t] >= c));
      if (count >= kmax) T = c;
    }
    thn = fmaxf(th, key2f(T));  // T <= key(k-th lo): a valid lower bound of tau_kmax
  }
  __syncwarp();
  int base = 0;
#pragma unroll
  for (int t = 0; t < kCand / 32; ++t) {
    bool keep = valid[t] && (__fadd_ru(v[t], e[t]) >= thn);
    uint32_t bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      int pos = base + __popc(bal & lanemask_lt());
      vr[pos] = v[t];
      ir[pos] = id[t];
    }
    base += __popc(bal);
  }
  __syncwarp();
  if (lane == L) {
    me.cnt = base;
    me.theta = thn;
    if (base > kCand - 32) {  // cannot make room for another chunk: exact fallback for this row
      *overflow_me = true;
      me.theta = __int_as_float(0x7f800000);  // +inf: append nothing more
    }
  }
}

// Process one chunk of 32 scores of this thread's row: s[j] is the score of item position
// pos0 + j (s = -inf for padding).  E = perr[pos0] >= perr of every item in the chunk (items
// are norm-sorted descending, so perr is non-increasing).  All 32 lanes must call it.
template <typename ScoreFn>
__device__ __forceinline__ void cand_chunk(ScoreFn s_of, float mx, float E, int pos0, CandRow& me,
                                           float* cv, int* ci, const float* __restrict__ perr,
                                           int kmax, bool* overflow_me) {
  const int lane = threadIdx.x & 31;
  const bool pass = __fadd_ru(mx, E) >= me.theta;
  if (!__any_sync(0xffffffffu, pass)) return;
  if (pass) {
    float* vr = cv + lane * kCandPitch;
    int* ir = ci + lane * kCandPitch;
    const float thr = fmaxf(__fsub_rd(me.theta, E), -3.402823466e38f);  // padding (-inf) never passes
    int c = me.cnt;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      float sj = s_of(j);
      if (sj >= thr) {
        vr[c] = sj;
        ir[c] = pos0 + j;
        ++c;
      }
    }
    me.cnt = c;
  }
  uint32_t need = __ballot_sync(0xffffffffu, me.cnt > kCand - 32);
  while (need) {
    int L = __ffs(need) - 1;
    need &= need - 1;
    cand_refresh_lane(L, me, cv, ci, perr, kmax, overflow_me);
  }
}

// Final compaction of every row of the warp, then write the candidates out.
__device__ __forceinline__ void cand_finish(CandRow& me, float* cv, int* ci, const float* __restrict__ perr,
                                            int kmax, bool* overflow_me, int64_t row, int64_t n,
                                            int32_t* __restrict__ cand, int32_t* __restrict__ ccount,
                                            int32_t* __restrict__ ovf_list, int* __restrict__ ovf_count) {
  const int lane = threadIdx.x & 31;
  for (int L = 0; L < 32; ++L) {
    bool skip = __shfl_sync(0xffffffffu, (int)*overflow_me, L);
    if (!skip) cand_refresh_lane(L, me, cv, ci, perr, kmax, overflow_me);
  }
  __syncwarp();
  if (row < n) {
    if (*overflow_me) {
      ccount[row] = -1;
      int slot = atomicAdd(ovf_count, 1);
      ovf_list[slot] = (int32_t)row;
    } else {
      ccount[row] = me.cnt;
    }
  }
  // coalesced-ish write: each lane copies its own row (rows are kCand-strided in global)
  if (row < n && !*overflow_me) {
    const int* ir = ci + lane * kCandPitch;
    for (int i = 0; i < me.cnt; ++i) cand[row * kCand + i] = ir[i];
  }
}

}  // namespace rmips
