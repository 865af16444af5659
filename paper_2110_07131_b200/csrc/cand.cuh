// cand.cuh -- per-user-row top-k_max CANDIDATE filter, the epilogue of the build contraction.
//
// Alg. 1 lines 7-9 compute, for every user, the k_max largest inner products.
// On the GPU the |Q| x |P| score matrix is produced tile by tile (tensor cores or FFMA) in a
// reduced precision whose error is bounded per item by perr[p] (common.cuh).
// Each epilogue thread owns one user row and keeps
//   theta : a valid lower bound (scaled units) of the k_max-th largest TRUE score seen so far
//           (at least k_max buffered entries have lo >= theta, and lo <= true score);
//   vmax  : the largest lo in its buffer;
//   a candidate buffer in shared memory, slot-major ([slot][128 rows], 8-byte entries
//   {lo bits, item position}) so that every lane reads/writes its own row conflict-free;
//   lo = s~ - E rounded down.
// An item is appended iff s~ >= theta - E (it may still be in the final top-k_max).  When any
// row of a warp may not have room for another 32-column chunk, the whole warp refreshes at
// once, every thread on its own row:
//   1. theta' = the largest of 4 quaternary search levels over [theta, vmax] (3 thresholds per
//      pass; 256-way resolution) that keeps at least k_max entries lo >= theta' (exact counts of
//      the fp32 thresholds themselves, so theta' is valid by construction);
//   2. one compaction pass that drops entries whose upper bound lo + 2 E0 (E0 = perr of the
//      largest-norm item >= every E) is below theta' and re-counts #{lo >= theta'} (a
//      belt-and-braces check: were it ever below k_max the row would go to the exact fallback).
// Every true top-k_max item has s >= tau_kmax >= theta at all times, so it is never rejected
// or dropped.  A row that cannot be compacted below kCand - 32 entries (massive
// ties) is likewise flagged and recomputed exactly by the fallback kernel.
#pragma once
#include "common.cuh"
#include "sm100.cuh"

namespace rmips {

constexpr int kCandRows = 128;  // rows per CTA buffer (slot stride)
// shared-memory bytes the filter needs for 128 rows
constexpr int kCandSmemBytes = kCand * kCandRows * 8;

// Shared-memory pointers.  Functions that are not inlined re-assert the state space
// (__builtin_assume(__isShared(..))) so that they still compile to LDS/STS.
struct CandSmem {
  uint2* buf;       // [kCand][kCandRows] {lo bits, item position}
  __device__ __forceinline__ static CandSmem at(uint8_t* base) { return CandSmem{reinterpret_cast<uint2*>(base)}; }
  __device__ __forceinline__ void assume_shared() const { __builtin_assume(__isShared(buf)); }
};

struct CandRow {
  float theta;   // running lower bound (scaled units); +inf for dead / overflowed rows
  float vmax;    // max lo in the buffer (-inf when empty)
  int cnt;       // live candidates in this row's buffer
  int ovf;       // overflowed: exact fallback
};

__device__ __forceinline__ CandRow cand_init(bool live) {
  const float inf = __int_as_float(0x7f800000);
  return CandRow{live ? -inf : inf, -inf, 0, 0};
}

// Per-thread refresh of this thread's row (called by all 32 lanes together).  Not inlined (one
// copy per kernel keeps the hot loops inside the instruction cache); the row state travels in
// registers.  e0x2 >= 2 * (every chunk error bound E used at append time), rounded up.
// theta_only (the build kernels' stale-theta checkpoints): the search starts at the current theta and only
// theta moves (no compaction).
static __device__ __noinline__ CandRow cand_refresh(CandRow me, CandSmem sm, int rloc, float e0x2, int kmax,
                                                    bool theta_only = false) {
  if (me.ovf) return me;
  const int cn = me.cnt;
  sm.assume_shared();
  uint2* b = sm.buf + rloc;
  const float th = me.theta;
  float nth = th;  // proposed new theta
  if (cn >= kmax) {
    float L = th;
    const float U = me.vmax;
    if (theta_only && L > -3.402823466e38f && L < U) {
      // (#{lo >= theta} >= k_max since the last full refresh: theta is a valid lower end)
    } else if (!(L > -3.402823466e38f)) {  // first refresh: bracket from the smallest entry
      float m0 = U, m1 = U, m2 = U, m3 = U;
      int i = 0;
      for (; i + 4 <= cn; i += 4) {
        m0 = fminf(m0, __uint_as_float(b[i * kCandRows].x));
        m1 = fminf(m1, __uint_as_float(b[(i + 1) * kCandRows].x));
        m2 = fminf(m2, __uint_as_float(b[(i + 2) * kCandRows].x));
        m3 = fminf(m3, __uint_as_float(b[(i + 3) * kCandRows].x));
      }
      for (; i < cn; ++i) m0 = fminf(m0, __uint_as_float(b[i * kCandRows].x));
      L = fminf(fminf(m0, m1), fminf(m2, m3));
    }
    // 4 quaternary passes (3 thresholds each, 256-way resolution of [L, U]); the counts are
    // kept in 4 independent accumulators per threshold so the loop is not a dependency chain
    float U2 = U;
#pragma unroll 1
    for (int pass = 0; pass < 4; ++pass) {
      const float w = U2 - L;
      const float t1 = fmaf(w, 0.25f, L), t2 = fmaf(w, 0.5f, L), t3 = fmaf(w, 0.75f, L);
      int a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0}, a3[4] = {0, 0, 0, 0};
      int i = 0;
      for (; i + 8 <= cn; i += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __uint_as_float(b[(i + u) * kCandRows].x);
#pragma unroll
        for (int u = 0; u < 8; ++u) a1[u & 3] += v[u] >= t1, a2[u & 3] += v[u] >= t2, a3[u & 3] += v[u] >= t3;
      }
      for (; i < cn; ++i) {
        const float v0 = __uint_as_float(b[i * kCandRows].x);
        a1[0] += v0 >= t1, a2[0] += v0 >= t2, a3[0] += v0 >= t3;
      }
      const int c1 = (a1[0] + a1[1]) + (a1[2] + a1[3]), c2 = (a2[0] + a2[1]) + (a2[2] + a2[3]),
                c3 = (a3[0] + a3[1]) + (a3[2] + a3[3]);
      if (c3 >= kmax) L = t3;
      else if (c2 >= kmax) L = t2, U2 = t3;
      else if (c1 >= kmax) L = t1, U2 = t2;
      else U2 = t1;
    }
    nth = L;
    nth = fmaxf(nth, th);
  }
  if (theta_only) {
    me.theta = nth;
    return me;
  }
  const float keep = __fsub_rd(nth, e0x2);  // lo < keep  =>  lo + 2E < theta: cannot be top-k_max
  int wpos = 0, ge = 0, i = 0;
  for (; i + 8 <= cn; i += 8) {
    uint2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = b[(i + u) * kCandRows];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float lo = __uint_as_float(v[u].x);
      ge += lo >= nth;
      if (lo >= keep) {  // wpos <= i + u: never overtakes an unread entry
        b[wpos * kCandRows] = v[u];
        ++wpos;
      }
    }
  }
  for (; i < cn; ++i) {
    const uint2 v = b[i * kCandRows];
    const float lo = __uint_as_float(v.x);
    ge += lo >= nth;
    if (lo >= keep) {
      b[wpos * kCandRows] = v;
      ++wpos;
    }
  }
  me.theta = nth;
  me.cnt = wpos;
  if (wpos > kCand - 32 || (nth > th && ge < kmax)) {  // no room / unverified theta: exact fallback
    me.ovf = 1;
    me.theta = __int_as_float(0x7f800000);
  }
  return me;
}

// Seed threshold (build_tc.cu, seed pass): slots [0, me.cnt) of this thread's row hold, in both
// halves of each entry, lower bounds of the maxima of disjoint item groups (lo = group max of s~
// minus E, rounded down, so lo <= the true score of a distinct item).  The k_max-th largest lo is
// therefore a valid lower bound of tau_kmax; this returns the largest level of a 5-pass
// quaternary search over [min lo, me.vmax] that keeps at least k_max of them (-inf if there are
// fewer than k_max).
static __device__ __noinline__ float cand_seed(CandRow me, CandSmem sm, int rloc, int kmax) {
  const int cn = me.cnt;
  if (2 * cn < kmax) return -__int_as_float(0x7f800000);
  sm.assume_shared();
  const uint2* b = sm.buf + rloc;
  float m0 = me.vmax, m1 = me.vmax;
  for (int i = 0; i < cn; ++i) {
    const uint2 v = b[i * kCandRows];
    m0 = fminf(m0, __uint_as_float(v.x)), m1 = fminf(m1, __uint_as_float(v.y));
  }
  float L = fminf(m0, m1), U2 = me.vmax;
#pragma unroll 1
  for (int pass = 0; pass < 5; ++pass) {
    const float w = U2 - L;
    const float t1 = fmaf(w, 0.25f, L), t2 = fmaf(w, 0.5f, L), t3 = fmaf(w, 0.75f, L);
    int a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0}, a3[4] = {0, 0, 0, 0};
    int i = 0;
    for (; i + 4 <= cn; i += 4) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint2 e = b[(i + u) * kCandRows];
        v[2 * u] = __uint_as_float(e.x), v[2 * u + 1] = __uint_as_float(e.y);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) a1[u & 3] += v[u] >= t1, a2[u & 3] += v[u] >= t2, a3[u & 3] += v[u] >= t3;
    }
    for (; i < cn; ++i) {
      const uint2 e = b[i * kCandRows];
      const float v0 = __uint_as_float(e.x), v1 = __uint_as_float(e.y);
      a1[0] += v0 >= t1, a2[0] += v0 >= t2, a3[0] += v0 >= t3;
      a1[1] += v1 >= t1, a2[1] += v1 >= t2, a3[1] += v1 >= t3;
    }
    const int c1 = (a1[0] + a1[1]) + (a1[2] + a1[3]), c2 = (a2[0] + a2[1]) + (a2[2] + a2[3]),
              c3 = (a3[0] + a3[1]) + (a3[2] + a3[3]);
    if (c3 >= kmax) L = t3;
    else if (c2 >= kmax) L = t2, U2 = t3;
    else if (c1 >= kmax) L = t1, U2 = t2;
    else U2 = t1;
  }
  return L;
}

// Append pass of one 32-column chunk (scores via s_of(j), positions pos0 + j), called by the
// whole warp when any lane's chunk max passed; g4[8] are the 4-column group maxima.  Groups are
// skipped warp-uniformly; inside a group the 4 slots are computed from a prefix of predicates
// so the stores are independent of each other.
template <typename ScoreFn>
__device__ __forceinline__ void cand_append_chunk(ScoreFn s_of, const float (&g4)[8], float E, int pos0,
                                                  CandRow& me, CandSmem sm, int rloc) {
  sm.assume_shared();
  const float thr = fmaxf(__fsub_rd(me.theta, E), -3.402823466e38f);  // padding (-inf) never passes
  uint2* b = sm.buf + rloc;
  int c = me.cnt;
  float vmax = me.vmax;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const bool gp = g4[g] >= thr;
    if (__any_sync(0xffffffffu, gp)) {
      const float s0 = s_of(4 * g), s1 = s_of(4 * g + 1), s2 = s_of(4 * g + 2), s3 = s_of(4 * g + 3);
      const bool p0 = s0 >= thr, p1 = s1 >= thr, p2 = s2 >= thr, p3 = s3 >= thr;
      const int o1 = c + p0, o2 = o1 + p1, o3 = o2 + p2;
      if (p0) b[c * kCandRows] = make_uint2(__float_as_uint(__fsub_rd(s0, E)), (uint32_t)(pos0 + 4 * g));
      if (p1) b[o1 * kCandRows] = make_uint2(__float_as_uint(__fsub_rd(s1, E)), (uint32_t)(pos0 + 4 * g + 1));
      if (p2) b[o2 * kCandRows] = make_uint2(__float_as_uint(__fsub_rd(s2, E)), (uint32_t)(pos0 + 4 * g + 2));
      if (p3) b[o3 * kCandRows] = make_uint2(__float_as_uint(__fsub_rd(s3, E)), (uint32_t)(pos0 + 4 * g + 3));
      c = o3 + p3;
      if (gp) vmax = fmaxf(vmax, __fsub_rd(g4[g], E));
    }
  }
  me.cnt = c;
  me.vmax = vmax;
}

// Branch-free append of one 32-column chunk (dense chunks: no per-group votes); the slot of
// column j is cnt + #{passing columns < j}.
template <typename ScoreFn>
__device__ __forceinline__ void cand_append_flat(ScoreFn s_of, float mx, float E, int pos0, CandRow& me, CandSmem sm,
                                                 int rloc) {
  sm.assume_shared();
  const float thr = fmaxf(__fsub_rd(me.theta, E), -3.402823466e38f);  // padding (-inf) never passes
  uint2* b = sm.buf + rloc;
  int c = me.cnt;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    const float sj = s_of(j);
    const bool p = sj >= thr;
    if (p) b[c * kCandRows] = make_uint2(__float_as_uint(__fsub_rd(sj, E)), (uint32_t)(pos0 + j));
    c += p;
  }
  if (mx >= thr) me.vmax = fmaxf(me.vmax, __fsub_rd(mx, E));
  me.cnt = c;
}

// After a chunk: if any row of the warp may not have room for another chunk, refresh all.
__device__ __forceinline__ void cand_maybe_refresh(CandRow& me, CandSmem sm, int rloc, float e0x2, int kmax) {
  if (__any_sync(0xffffffffu, me.cnt > kCand - 32)) me = cand_refresh(me, sm, rloc, e0x2, kmax);
}

// Process one chunk of 32 scores: group maxima, one compare, appends only if needed.
template <typename ScoreFn>
__device__ __forceinline__ void cand_chunk(ScoreFn s_of, float E, int pos0, CandRow& me, CandSmem sm, int rloc,
                                           float e0x2, int kmax) {
  float g4[8];
#pragma unroll
  for (int g = 0; g < 8; ++g)
    g4[g] = fmaxf(fmaxf(s_of(4 * g), s_of(4 * g + 1)), fmaxf(s_of(4 * g + 2), s_of(4 * g + 3)));
  const float mx = fmaxf(fmaxf(fmaxf(g4[0], g4[1]), fmaxf(g4[2], g4[3])), fmaxf(fmaxf(g4[4], g4[5]), fmaxf(g4[6], g4[7])));
  const bool pass = __fadd_ru(mx, E) >= me.theta;
  if (!__any_sync(0xffffffffu, pass)) return;
  cand_append_chunk(s_of, g4, E, pos0, me, sm, rloc);
  cand_maybe_refresh(me, sm, rloc, e0x2, kmax);
}

// Final compaction of every row of the warp, then write the candidates out.  A live row always
// holds at least min(k_max, m) entries (see qrow_finish, candq.cuh); fewer means NaN scores (a user
// whose norm exceeds FLT_MAX) and the row takes the exact fallback.
__device__ __forceinline__ void cand_finish(CandRow& me, CandSmem sm, int rloc, float e0x2, int kmax, int64_t m,
                                            int64_t row, int64_t n, int32_t* __restrict__ cand, int cstride,
                                            int32_t* __restrict__ ccount, int32_t* __restrict__ ovf_list,
                                            int* __restrict__ ovf_count) {
  me = cand_refresh(me, sm, rloc, e0x2, kmax);
  if (row < n) {
    if (me.ovf || (int64_t)me.cnt < (m < kmax ? m : (int64_t)kmax)) {
      ccount[row] = -1;
      int slot = atomicAdd(ovf_count, 1);
      ovf_list[slot] = (int32_t)row;
    } else {
      ccount[row] = me.cnt;
      const uint2* b = sm.buf + rloc;
      for (int i = 0; i < me.cnt; ++i) cand[row * cstride + i] = (int32_t)b[i * kCandRows].y;
    }
  }
}

// Row state of a two-pass (regrouped) build: entries row-major at ent[row * kCand ..], {theta, vmax, cnt,
// ovf} at meta[row].
__device__ __forceinline__ void cand_save(const CandRow& me, CandSmem sm, int rloc, uint2* __restrict__ ent,
                                          uint4* __restrict__ meta, int64_t row) {
  sm.assume_shared();
  const uint2* b = sm.buf + rloc;
  uint2* o = ent + row * kCand;
  for (int i = 0; i < me.cnt; ++i) o[i] = b[i * kCandRows];
  meta[row] = make_uint4(__float_as_uint(me.theta), __float_as_uint(me.vmax), (uint32_t)me.cnt, (uint32_t)me.ovf);
}
__device__ __forceinline__ void cand_load(CandRow& me, CandSmem sm, int rloc, const uint2* __restrict__ ent,
                                          const uint4* __restrict__ meta, int64_t row) {
  const uint4 mt = __ldg(meta + row);
  me.theta = __uint_as_float(mt.x);
  me.vmax = __uint_as_float(mt.y);
  me.cnt = (int)mt.z;
  me.ovf = (int)mt.w;
  sm.assume_shared();
  uint2* b = sm.buf + rloc;
  const uint2* s = ent + row * kCand;
  for (int i = 0; i < me.cnt; ++i) b[i * kCandRows] = __ldg(s + i);
}

// 2 * E0 rounded up, E0 = perr[0] >= every item's bound (perr is non-increasing along the
// norm-sorted items).
__device__ __forceinline__ float cand_e0x2(const float* __restrict__ perr) {
  const float e0 = __ldg(perr);
  return __fadd_ru(e0, e0);
}

}  // namespace rmips
