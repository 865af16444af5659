// cand.cuh -- per-user-row top-k_max CANDIDATE filter, the epilogue of the build contraction.
//
// Alg. 1 lines 7-9 compute, for every user, the k_max largest inner products.
// On the GPU the |Q| x |P| score matrix is produced tile by tile (tensor cores or FFMA) in a
// reduced precision whose error is bounded per item by perr[p] (common.cuh).
// Each epilogue thread owns one user row and keeps
//   theta : a valid lower bound (scaled units) of the k_max-th largest TRUE score seen so far
//           (at least k_max buffered entries have lo >= theta, and lo <= true score);
//   vmax  : the largest lo in its buffer;
//   a candidate buffer in shared memory, slot-major ([slot][128 rows]) so that every lane
//   reads/writes its own row conflict-free: lo = s~ - E (rounded down) and the item position.
// An item is appended iff s~ >= theta - E (it may still be in the final top-k_max).  When any
// row of a warp may not have room for another 32-column chunk, the whole warp refreshes at
// once, every thread on its own row: theta <- the largest of a 4-level quaternary search
// (3 thresholds per pass over the buffer, 256-way resolution of [theta, vmax]) that keeps at
// least k_max entries lo >= theta; then entries whose upper bound lo + 2 E0 (E0 = perr of the
// largest-norm item >= every E) is below theta are dropped.  Every true top-k_max item has
// s >= tau_kmax >= theta at all times, so it is never rejected or dropped.
// A row that cannot be compacted below kCand - 32 entries (massive ties) is flagged and
// recomputed exactly by the fallback kernel.
#pragma once
#include "common.cuh"

namespace rmips {

constexpr int kCandRows = 128;  // rows per CTA buffer (slot stride)

struct CandRow {
  float theta;   // running lower bound (scaled units); +inf for dead / overflowed rows
  float vmax;    // max lo in the buffer (-inf when empty)
  int cnt;       // live candidates in this row's buffer
  bool ovf;      // overflowed: exact fallback
};

__device__ __forceinline__ CandRow cand_init(bool live) {
  const float inf = __int_as_float(0x7f800000);
  return CandRow{live ? -inf : inf, -inf, 0, false};
}

// Per-thread refresh of this thread's row (called by all 32 lanes together).
// clo/cid: slot-major buffers, entry i of this row at [i * kCandRows + rloc].
// e0x2 >= 2 * (every chunk error bound E used at append time), rounded up.
// Not inlined (one copy per kernel keeps the hot loops inside the instruction cache); the row
// state travels in registers (by value).
static __device__ __noinline__ CandRow cand_refresh(CandRow me, float* __restrict__ clo, int* __restrict__ cid,
                                                    int rloc, float e0x2, int kmax) {
  if (me.ovf) return me;
  const int cn = me.cnt;
  float th = me.theta;
  if (cn >= kmax) {
    // invariant: #{lo >= L} >= kmax (L = theta_old holds for the survivors of the last refresh)
    float L = th, U = me.vmax;
    if (!(L > -3.402823466e38f)) {  // first refresh: bracket from the smallest entry
      L = U;
#pragma unroll 8
      for (int i = 0; i < cn; ++i) L = fminf(L, clo[i * kCandRows + rloc]);
    }
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
      const float w = U - L;
      const float t1 = fmaf(w, 0.25f, L), t2 = fmaf(w, 0.5f, L), t3 = fmaf(w, 0.75f, L);
      int c1 = 0, c2 = 0, c3 = 0;
      int i = 0;
      // 8 independent shared loads in flight per step (the loop is latency-, not issue-bound)
      for (; i + 8 <= cn; i += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = clo[(i + u) * kCandRows + rloc];
#pragma unroll
        for (int u = 0; u < 8; ++u) c1 += v[u] >= t1, c2 += v[u] >= t2, c3 += v[u] >= t3;
      }
      for (; i < cn; ++i) {
        const float v0 = clo[i * kCandRows + rloc];
        c1 += v0 >= t1, c2 += v0 >= t2, c3 += v0 >= t3;
      }
      if (c3 >= kmax) L = t3;
      else if (c2 >= kmax) L = t2, U = t3;
      else if (c1 >= kmax) L = t1, U = t2;
      else U = t1;
    }
    th = fmaxf(th, L);
  }
  const float keep = __fsub_rd(th, e0x2);  // lo < keep  =>  lo + 2E < theta: the item cannot be top-k_max
  int w = 0, i = 0;
  for (; i + 8 <= cn; i += 8) {
    float v[8];
    int id[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = clo[(i + u) * kCandRows + rloc], id[u] = cid[(i + u) * kCandRows + rloc];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (v[u] >= keep) {  // w <= i + u: the write never overtakes an unread entry
        clo[w * kCandRows + rloc] = v[u];
        cid[w * kCandRows + rloc] = id[u];
        ++w;
      }
    }
  }
  for (; i < cn; ++i) {
    const float lo = clo[i * kCandRows + rloc];
    const int id = cid[i * kCandRows + rloc];
    if (lo >= keep) {
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
  return me;
}

// Append pass of one 32-column chunk (scores via s_of(j), positions pos0 + j), called by the
// whole warp when any lane's chunk max passed; g4[8] are the 4-column group maxima.  Groups are
// skipped warp-uniformly; inside a group the 4 slots are computed from a prefix of predicates
// so the stores are independent of each other.
template <typename ScoreFn>
__device__ __forceinline__ void cand_append_chunk(ScoreFn s_of, const float (&g4)[8], float E, int pos0,
                                                  CandRow& me, float* __restrict__ clo, int* __restrict__ cid,
                                                  int rloc) {
  const float thr = fmaxf(__fsub_rd(me.theta, E), -3.402823466e38f);  // padding (-inf) never passes
  int c = me.cnt;
  float vmax = me.vmax;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const bool gp = g4[g] >= thr;
    if (__any_sync(0xffffffffu, gp)) {
      const float s0 = s_of(4 * g), s1 = s_of(4 * g + 1), s2 = s_of(4 * g + 2), s3 = s_of(4 * g + 3);
      const bool p0 = s0 >= thr, p1 = s1 >= thr, p2 = s2 >= thr, p3 = s3 >= thr;
      const int o1 = c + p0, o2 = o1 + p1, o3 = o2 + p2;
      if (p0) clo[c * kCandRows + rloc] = __fsub_rd(s0, E), cid[c * kCandRows + rloc] = pos0 + 4 * g;
      if (p1) clo[o1 * kCandRows + rloc] = __fsub_rd(s1, E), cid[o1 * kCandRows + rloc] = pos0 + 4 * g + 1;
      if (p2) clo[o2 * kCandRows + rloc] = __fsub_rd(s2, E), cid[o2 * kCandRows + rloc] = pos0 + 4 * g + 2;
      if (p3) clo[o3 * kCandRows + rloc] = __fsub_rd(s3, E), cid[o3 * kCandRows + rloc] = pos0 + 4 * g + 3;
      c = o3 + p3;
      if (gp) vmax = fmaxf(vmax, __fsub_rd(g4[g], E));
    }
  }
  me.cnt = c;
  me.vmax = vmax;
}

// After a chunk: if any row of the warp may not have room for another chunk, refresh all.
__device__ __forceinline__ void cand_maybe_refresh(CandRow& me, float* clo, int* cid, int rloc, float e0x2,
                                                   int kmax) {
  if (__any_sync(0xffffffffu, me.cnt > kCand - 32)) me = cand_refresh(me, clo, cid, rloc, e0x2, kmax);
}

// Process one chunk of 32 scores: group maxima, one compare, appends only if needed.
template <typename ScoreFn>
__device__ __forceinline__ void cand_chunk(ScoreFn s_of, float E, int pos0, CandRow& me, float* clo, int* cid,
                                           int rloc, float e0x2, int kmax) {
  float g4[8];
#pragma unroll
  for (int g = 0; g < 8; ++g)
    g4[g] = fmaxf(fmaxf(s_of(4 * g), s_of(4 * g + 1)), fmaxf(s_of(4 * g + 2), s_of(4 * g + 3)));
  const float mx = fmaxf(fmaxf(fmaxf(g4[0], g4[1]), fmaxf(g4[2], g4[3])), fmaxf(fmaxf(g4[4], g4[5]), fmaxf(g4[6], g4[7])));
  const bool pass = __fadd_ru(mx, E) >= me.theta;
  if (!__any_sync(0xffffffffu, pass)) return;
  cand_append_chunk(s_of, g4, E, pos0, me, clo, cid, rloc);
  cand_maybe_refresh(me, clo, cid, rloc, e0x2, kmax);
}

// Final compaction of every row of the warp, then write the candidates out.
__device__ __forceinline__ void cand_finish(CandRow& me, float* clo, int* cid, int rloc, float e0x2, int kmax,
                                            int64_t row, int64_t n, int32_t* __restrict__ cand,
                                            int32_t* __restrict__ ccount, int32_t* __restrict__ ovf_list,
                                            int* __restrict__ ovf_count) {
  me = cand_refresh(me, clo, cid, rloc, e0x2, kmax);
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

// 2 * E0 rounded up, E0 = perr[0] >= every item's bound (perr is non-increasing along the
// norm-sorted items).
__device__ __forceinline__ float cand_e0x2(const float* __restrict__ perr) {
  const float e0 = __ldg(perr);
  return __fadd_ru(e0, e0);
}

}  // namespace rmips
