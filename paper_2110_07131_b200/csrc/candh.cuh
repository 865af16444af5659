// candh.cuh -- per-user-row top-k_max CANDIDATE filter with 4-byte entries for item sets of at
// most 65,536 items: entry = (bf16 lower bound << 16) | 16-bit item position.  Same invariant as
// cand.cuh; the 4-byte entries let one CTA keep 256 rows (two user tiles sharing
// every item tile, eight epilogue warps) next to the operand ring.
//
// Alg. 1 lines 7-9: every user's k_max largest inner products over P.  Each thread
// owns one user row and keeps theta, a valid lower bound of the k_max-th largest TRUE score seen
// so far, and a slot-major shared-memory buffer of entries whose value
//   v(e) = float(e & 0xffff0000) = lo rounded DOWN to bf16  <=  lo = s~ - E  <=  s,
// and lo < up(v) = v + |v| 2^-7 (the next bf16 value, rounded up).  An item is appended iff
// s~ >= theta - E; an entry is dropped only when its upper bound up(v) + 2 E0 (E0 >= every E) is
// below theta.  Every true top-k_max item has s >= tau_kmax >= theta, so it is never rejected or
// dropped.  Refresh = 4 quaternary passes on v (256-way resolution of [theta, vmax]) for the
// largest threshold keeping >= k_max entries, then one compaction pass.
#pragma once
#include "common.cuh"

namespace rmips {

constexpr int kHSlots = 128;  // entries per row

struct HRow {
  float theta;  // valid lower bound of the k_max-th largest true score (scaled units)
  float vmax;   // largest appended lower bound
  int cnt;      // entries in the buffer
  int ovf;      // overflowed: exact fallback
};

// Buffer of R rows: entry i of row r at buf[i * R + r].
struct HBuf {
  uint32_t* buf;
  int R;
  __device__ __forceinline__ void assume_shared() const { __builtin_assume(__isShared(buf)); }
};

// x rounded down to bf16, as the high half of an entry
__device__ __forceinline__ uint32_t bf16_down_bits(float x) {
  uint32_t u = __float_as_uint(x);
  if ((int32_t)u < 0 && (u & 0xffffu)) u += 0x10000u;  // negative: round the magnitude up
  return u & 0xffff0000u;
}
__device__ __forceinline__ float hval(uint32_t e) { return __uint_as_float(e & 0xffff0000u); }

__device__ __forceinline__ HRow hrow_init(bool live) {
  const float inf = __int_as_float(0x7f800000);
  return HRow{live ? -inf : inf, -inf, 0, 0};
}

// Refresh of this thread's row (all 32 lanes of the warp call it together).  Not inlined: one
// copy per kernel keeps the hot loops in the instruction cache.
static __device__ __noinline__ HRow hrow_refresh(HRow me, HBuf sb, int rr, float e0x2, int kmax) {
  if (me.ovf) return me;
  sb.assume_shared();
  uint32_t* b = sb.buf + rr;
  const int R = sb.R;
  const int cn = me.cnt;
  const float th = me.theta;
  float nth = th;
  if (cn >= kmax) {
    float L = th;
    const float U = me.vmax;
    if (!(L > -3.402823466e38f)) {  // first refresh: bracket from the smallest entry
      float m0 = U, m1 = U;
      int i = 0;
      for (; i + 2 <= cn; i += 2) m0 = fminf(m0, hval(b[i * R])), m1 = fminf(m1, hval(b[(i + 1) * R]));
      if (i < cn) m0 = fminf(m0, hval(b[i * R]));
      L = fminf(m0, m1);
    }
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
        for (int u = 0; u < 8; ++u) v[u] = hval(b[(i + u) * R]);
#pragma unroll
        for (int u = 0; u < 8; ++u) a1[u & 3] += v[u] >= t1, a2[u & 3] += v[u] >= t2, a3[u & 3] += v[u] >= t3;
      }
      for (; i < cn; ++i) {
        const float v0 = hval(b[i * R]);
        a1[0] += v0 >= t1, a2[0] += v0 >= t2, a3[0] += v0 >= t3;
      }
      const int c1 = (a1[0] + a1[1]) + (a1[2] + a1[3]), c2 = (a2[0] + a2[1]) + (a2[2] + a2[3]),
                c3 = (a3[0] + a3[1]) + (a3[2] + a3[3]);
      if (c3 >= kmax) L = t3;
      else if (c2 >= kmax) L = t2, U2 = t3;
      else if (c1 >= kmax) L = t1, U2 = t2;
      else U2 = t1;
    }
    nth = fmaxf(L, th);
  }
  int wpos = 0, ge = 0, i = 0;
  auto keep = [&](float v) {  // up(v) + 2 E0 >= theta: the item may still be in the top k_max
    return __fadd_ru(__fadd_ru(v, fabsf(v) * 0.0078125f + 1e-30f), e0x2) >= nth;
  };
  for (; i + 8 <= cn; i += 8) {
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = b[(i + u) * R];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float x = hval(v[u]);
      ge += x >= nth;
      if (keep(x)) {  // wpos <= i + u: never overtakes an unread entry
        b[wpos * R] = v[u];
        ++wpos;
      }
    }
  }
  for (; i < cn; ++i) {
    const uint32_t v0 = b[i * R];
    const float x = hval(v0);
    ge += x >= nth;
    if (keep(x)) {
      b[wpos * R] = v0;
      ++wpos;
    }
  }
  me.theta = nth;
  me.cnt = wpos;
  if (wpos > kHSlots - 32 || (nth > th && ge < kmax)) {  // no room / unverified theta: exact fallback
    me.ovf = 1;
    me.theta = __int_as_float(0x7f800000);
  }
  return me;
}

// Append pass of one 32-column chunk (scores via s_of(j), positions pos0 + j; columns >= mi are
// padding), called by the whole warp; g4[8] are the 4-column group maxima.  Groups are skipped
// warp-uniformly; inside a group the 4 slots come from a prefix of predicates.
template <typename ScoreFn>
__device__ __forceinline__ void hrow_append_chunk(ScoreFn s_of, const float (&g4)[8], float E, int pos0, int mi,
                                                  HRow& me, HBuf sb, int rr) {
  sb.assume_shared();
  uint32_t* b = sb.buf + rr;
  const int R = sb.R;
  const float thr = fmaxf(__fsub_rd(me.theta, E), -3.402823466e38f);  // padding (-inf) never passes
  int c = me.cnt;
  float vmax = me.vmax;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const bool gp = g4[g] >= thr;
    if (__any_sync(0xffffffffu, gp)) {
      bool p[4];
      uint32_t e[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float sj = s_of(4 * g + j);
        p[j] = sj >= thr && pos0 + 4 * g + j < mi;
        e[j] = bf16_down_bits(__fsub_rd(sj, E)) | (uint32_t)(pos0 + 4 * g + j);
      }
      const int o1 = c + p[0], o2 = o1 + p[1], o3 = o2 + p[2];
      if (p[0]) b[c * R] = e[0];
      if (p[1]) b[o1 * R] = e[1];
      if (p[2]) b[o2 * R] = e[2];
      if (p[3]) b[o3 * R] = e[3];
      c = o3 + p[3];
      if (gp) vmax = fmaxf(vmax, __fsub_rd(g4[g], E));
    }
  }
  me.cnt = c;
  me.vmax = vmax;
}

__device__ __forceinline__ void hrow_maybe_refresh(HRow& me, HBuf sb, int rr, float e0x2, int kmax) {
  if (__any_sync(0xffffffffu, me.cnt > kHSlots - 32)) me = hrow_refresh(me, sb, rr, e0x2, kmax);
}

// Final compaction, then the candidate positions (or the overflow mark) are written out.
__device__ __forceinline__ void hrow_finish(HRow& me, HBuf sb, int rr, float e0x2, int kmax, int64_t row, int64_t n,
                                            int32_t* __restrict__ cand, int32_t* __restrict__ ccount,
                                            int32_t* __restrict__ ovf_list, int* __restrict__ ovf_count) {
  me = hrow_refresh(me, sb, rr, e0x2, kmax);
  if (row < n) {
    if (me.ovf) {
      ccount[row] = -1;
      const int slot = atomicAdd(ovf_count, 1);
      ovf_list[slot] = (int32_t)row;
    } else {
      ccount[row] = me.cnt;
      const uint32_t* b = sb.buf + rr;
      for (int i = 0; i < me.cnt; ++i) cand[row * kCand + i] = (int32_t)(b[i * sb.R] & 0xffffu);
    }
  }
}

}  // namespace rmips
