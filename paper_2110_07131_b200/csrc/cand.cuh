// cand.cuh -- per-user-row top-k_max CANDIDATE filter, the epilogue of the build contraction.
//
// Alg. 1 lines 7-9 compute, for every user, the k_max largest inner products.
// On the GPU the |Q| x |P| score matrix is produced tile by tile (tensor cores or FFMA) in a
// reduced precision whose error is bounded per item by perr[p] (common.cuh).
// Each epilogue thread owns one user row and keeps
//   theta : a valid lower bound (scaled units) of the k_max-th largest TRUE score seen so far;
//   a candidate buffer in shared memory, slot-major ([slot][128 rows]) so that every lane
//   writes/reads its own row conflict-free: lo = s~ - E (rounded down) and the item position.
// An item is appended iff s~ + E >= theta (it may still be in the final top-k_max).  When any
// row of a warp nears full, the whole warp refreshes at once, every thread on its own row:
// theta <- a value with at least k_max entries lo >= theta (bisection, 8 halvings of
// [theta_old, max lo]), then entries with upper bound lo + 2E < theta are dropped.  Refreshes
// are synchronized because the 32 rows of a warp see the same item stream and fill at similar
// rates (SURVEY cfg1 simulation: 4.75 warp refreshes per sweep of P).
// Every true top-k_max item has s >= tau_kmax >= theta at all times, so it is never rejected
// or dropped.  A row that cannot be compacted below kCand - 32 entries (massive
// ties) is flagged and recomputed exactly by the fallback kernel.
#pragma once
#include "common.cuh"

namespace rmips {

constexpr int kCandRows = 128;  // rows per CTA buffer (slot stride)

struct CandRow {
  float theta;   // running lower bound (scaled units); +inf for dead / overflowed rows
  int cnt;       // live candidates in this row's buffer
  bool ovf;      // overflowed: exact fallback
};

// Per-thread refresh of this thread's row (called by all 32 lanes together).
// clo/cid: slot-major buffers, entry i of this row at [i * kCandRows + rloc].
// perr_of(pos) returns the chunk error bound E used when the entry was appended.
__device__ __forceinline__ void cand_refresh_row(CandRow& me, float* __restrict__ clo, int* __restrict__ cid,
                                                 int rloc, const float* __restrict__ perr, int kmax) {
  if (me.ovf) return;
  const int cn = me.cnt;
  float vmax = -__int_as_float(0x7f800000), vmin = __int_as_float(0x7f800000);
  for (int i = 0; i < cn; ++i) {
    float v = clo[i * kCandRows + rloc];
    vmax = fmaxf(vmax, v);
    vmin = fminf(vmin, v);
  }
  float th = me.theta;
  if (cn >= kmax) {
    // invariant: #{lo >= L} >= kmax  (L = theta_old holds for the survivors of the last refresh)
    float L = fmaxf(th, vmin), U = vmax;
#pragma unroll 1
    for (int it = 0; it < 8; ++it) {
      const float mid = 0.5f * (L + U);
      int c = 0;
      for (int i = 0; i < cn; ++i) c += clo[i * kCandRows + rloc] >= mid;
      if (c >= kmax) L = mid; else U = mid;
    }
    th = fmaxf(th, L);
  }
  int w = 0;
  for (int i = 0; i < cn; ++i) {
    const float lo = clo[i * kCandRows + rloc];
    const int id = cid[i * kCandRows + rloc];
    const float E = __ldg(perr + (id & ~31));         // chunk bound used at append time
    if (__fadd_ru(lo, 2.f * E) >= th) {
      clo[w * kCandRows + rloc] = lo;
      cid[w * kCandRows + rloc] = id;
      ++w;
    }
  }
  me.cnt = w;
  me.theta = th;
  if (w > kCand - 32) {
    me.ovf = true;
    me.theta = __int_as_float(0x7f800000);
  }
}

// Append pass of one 32-column chunk (scores via s_of(j), positions pos0 + j) for a thread
// whose chunk max passed.  Works in groups of 4 columns using the group maxima g4[8].
template <typename ScoreFn>
__device__ __forceinline__ void cand_append_chunk(ScoreFn s_of, const float (&g4)[8], float E, int pos0,
                                                  CandRow& me, float* __restrict__ clo, int* __restrict__ cid,
                                                  int rloc) {
  const float thr = fmaxf(__fsub_rd(me.theta, E), -3.402823466e38f);  // padding (-inf) never passes
  int c = me.cnt;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    if (g4[g] >= thr) {
#pragma unroll
      for (int j = 4 * g; j < 4 * g + 4; ++j) {
        const float sj = s_of(j);
        if (sj >= thr) {
          clo[c * kCandRows + rloc] = __fsub_rd(sj, E);
          cid[c * kCandRows + rloc] = pos0 + j;
          ++c;
        }
      }
    }
  }
  me.cnt = c;
}

// After a chunk: if any row of the warp may not have room for another chunk, refresh all.
__device__ __forceinline__ void cand_maybe_refresh(CandRow& me, float* clo, int* cid, int rloc,
                                                   const float* __restrict__ perr, int kmax) {
  if (__any_sync(0xffffffffu, me.cnt > kCand - 32)) cand_refresh_row(me, clo, cid, rloc, perr, kmax);
}

// Process one chunk of 32 scores: group maxima, one compare, appends only if needed.
template <typename ScoreFn>
__device__ __forceinline__ void cand_chunk(ScoreFn s_of, float E, int pos0, CandRow& me, float* clo, int* cid,
                                           int rloc, const float* __restrict__ perr, int kmax) {
  float g4[8];
#pragma unroll
  for (int g = 0; g < 8; ++g)
    g4[g] = fmaxf(fmaxf(s_of(4 * g), s_of(4 * g + 1)), fmaxf(s_of(4 * g + 2), s_of(4 * g + 3)));
  const float mx = fmaxf(fmaxf(fmaxf(g4[0], g4[1]), fmaxf(g4[2], g4[3])), fmaxf(fmaxf(g4[4], g4[5]), fmaxf(g4[6], g4[7])));
  const bool pass = __fadd_ru(mx, E) >= me.theta;
  if (!__any_sync(0xffffffffu, pass)) return;
  if (pass) cand_append_chunk(s_of, g4, E, pos0, me, clo, cid, rloc);
  cand_maybe_refresh(me, clo, cid, rloc, perr, kmax);
}

// Final compaction of every row of the warp, then write the candidates out.
__device__ __forceinline__ void cand_finish(CandRow& me, float* clo, int* cid, int rloc,
                                            const float* __restrict__ perr, int kmax, int64_t row, int64_t n,
                                            int32_t* __restrict__ cand, int32_t* __restrict__ ccount,
                                            int32_t* __restrict__ ovf_list, int* __restrict__ ovf_count) {
  cand_refresh_row(me, clo, cid, rloc, perr, kmax);
  if (row < n) {
    if (me.ovf) {
      ccount[row] = -1;
      int slot = atomicAdd(ovf_count, 1);
      ovf_list[slot] = (int32_t)row;
    } else {
      ccount[row] = me.cnt;
      for (int i = 0; i < me.cnt; ++i) cand[row * kCand + i] = cid[i * kCandRows + rloc];
    }
  }
}

}  // namespace rmips
