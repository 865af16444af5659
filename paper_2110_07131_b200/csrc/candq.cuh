// candq.cuh -- per-user-row top-k_max CANDIDATE filter of the tensor-core build (k_build_tc):
// the same invariant as cand.cuh (the SIMT build's filter), with 4-byte entries so that a CTA can
// keep 256 rows (two user tiles, eight epilogue warps) or 128 rows next to d = 256 operand tiles.
//
// Alg. 1 lines 7-9: every user's k_max largest inner products over P.  Scores s~ are
// reduced-precision (fp16 operands, fp32 accumulation) with a per-item error bound E
// (common.cuh).  Each epilogue thread owns one user row and keeps
//   theta : a valid lower bound of the k_max-th largest TRUE score seen so far;
//   a slot-major shared-memory buffer of packed entries (q << 20) | position, where q is a
//           12-bit QUANTISED LOWER BOUND of the item's score:
//              deq(q) = base + q * w  (rounded down, w a power of two)  <=  lo = s~ - E  <=  s,
//           and lo < deq(q) + qe, qe = w (1 + 2^-10).  The row's quantiser (base = -smax, w) is
//           fixed for its whole scan, so every entry is quantised exactly once and the bound qe
//           holds for all of them (re-quantising on a rebased grid would add up to one quantum per
//           rebase to that bound; measured, it also kept more candidates).
// An item is appended iff s~ >= theta - E; an entry is dropped only when its upper bound
// (< deq(q) + qe + 2 E, rounded up; E0 = the largest E during the scan, the entry's own group bound
// at the end) is below theta.  Every true top-k_max item has s >= tau_kmax >= theta, so it is never
// rejected or dropped.
// Refresh (when a row of the warp may not have room for another 32-column chunk): a quaternary
// search over q (integer compares on the packed words) for the largest qt with #{q >= qt} >= k_max;
// theta <- max(theta, deq(qt)); then one compaction pass that drops entries below
// theta - 2 E0 - qe.
// Positions must be < 2^PB (PB = 20: m <= 1,048,576 with 12-bit bounds; PB = 21: m <= 2^21 with
// 11-bit bounds; larger item sets use the 8-byte entries of cand.cuh, FPol in candpol.cuh).  SLOTS (128 or 256) entries per row: 256 for k_max above ~80 (a refresh must leave
// room for another 32-column chunk above the k_max kept entries).
#pragma once
#include "common.cuh"
#include "sm100.cuh"

namespace rmips {

// Entry format: (q << PB) | position, PB position bits (20: m <= 2^20 with a 12-bit bound; 21: m <= 2^21
// with an 11-bit bound).
template <int PB>
struct QFmt {
  static constexpr int kPosBits = PB;
  static constexpr uint32_t kPosMask = (1u << PB) - 1u;
  static constexpr int kQMax = (1 << (32 - PB)) - 1;  // largest quantised bound
};
constexpr int kQPosBits = 20;  // (the default format)
constexpr uint32_t kQPosMask = QFmt<20>::kPosMask;
constexpr int kQMax = QFmt<20>::kQMax;

struct QRow {
  float theta;  // valid lower bound of the k_max-th largest true score (scaled units)
  float base;   // quantisation origin
  float w;      // quantum (power of two): (smax - base) / w <= 4095, so q never saturates
  float inv;    // 1 / w (exact)
  float smax;   // bound on every score: |s~| <= smax
  float vmax;   // largest appended lower bound (unquantised)
  int cnt;      // entries in the buffer
  int ovf;      // overflowed: exact fallback
};

__device__ __forceinline__ float pow2_ceil(float x) {  // smallest power of two >= x (x > 0, finite)
  int e;
  const float f = frexpf(x, &e);  // x = f * 2^e, f in [0.5, 1)
  return ldexpf(1.f, f == 0.5f ? e - 1 : e);
}

// Buffer of R rows: entry i of row r at buf[i * R + r].
// perr (optional): the per-item error table, entry j appended with E = perr[j & ~(kPerrGroup - 1)].
struct QBuf {
  uint32_t* buf;
  int R;
  const float* perr;
  __device__ __forceinline__ void assume_shared() const { __builtin_assume(__isShared(buf)); }
};

// Quantised lower bound of x (base <= x <= smax): floor((x - base) / w) <= 4095.  The quantum
// covers [base, smax], never only [base, vmax]: a saturated q would no longer bound lo from above
// (lo < deq(q) + w), and the drop test relies on that.
template <int PB = 20>
__device__ __forceinline__ uint32_t q_of(float x, const QRow& me) {
  const float dd = __fsub_rd(x, me.base) * me.inv;  // exact power-of-two scaling of a rounded-down gap
  return dd >= (float)QFmt<PB>::kQMax ? (uint32_t)QFmt<PB>::kQMax : (uint32_t)dd;
}
__device__ __forceinline__ float deq(uint32_t q, const QRow& me) { return __fadd_rd(me.base, (float)q * me.w); }
// lo - deq(q) < qe = w (1 + 2^-10): the quantum plus the rounding of deq.  Entries are quantised once
// (the quantiser of a row never changes), so this bounds every entry of the buffer.
__device__ __forceinline__ float qrow_qe(const QRow& me) { return __fmul_ru(me.w, 1.0009765625f); }

// The build kernels bound the scores of a group of kPerrGroup = 4 item tiles of 128 by the error
// bound of the group's first item (perr is non-increasing along the norm-sorted items).
constexpr uint32_t kPerrGroup = 512;
// Upper bound of the true score of an entry with dequantised value x at item position j.
__device__ __forceinline__ float entry_ub(float x, float qe, const float* __restrict__ perr, uint32_t j) {
  return __fadd_ru(__fadd_ru(x, qe), __fmul_ru(2.f, __ldg(perr + (j & ~(kPerrGroup - 1u)))));
}

// smax bounds |s~| for every item (scores are in [-smax, smax]).
template <int PB = 20>
__device__ __forceinline__ QRow qrow_init(bool live, float smax) {
  const float inf = __int_as_float(0x7f800000);
  QRow r;
  r.theta = live ? -inf : inf;
  r.base = -smax;
  r.w = pow2_ceil(fmaxf(2.f * smax, 1e-30f) / (float)QFmt<PB>::kQMax);
  r.inv = 1.f / r.w;
  r.smax = smax;
  r.vmax = -inf;
  r.cnt = 0;
  r.ovf = 0;
  return r;
}

// Refresh of this thread's row (all 32 lanes of the warp call it together).  Not inlined: one
// copy per kernel keeps the hot loops in the instruction cache.
// theta_only (the build kernels' stale-theta checkpoints): the search starts at the current theta and
// only theta moves (no compaction, no re-quantisation: the entries stay valid under the old quantiser).
template <int SLOTS, int PB = 20>
static __device__ __noinline__ QRow qrow_refresh(QRow me, QBuf sb, int rr, float e0x2, int kmax,
                                                 bool theta_only = false, bool final_pass = false) {
  constexpr int kQPosBits = PB;  // (this function's entry format)
  constexpr uint32_t kQPosMask = QFmt<PB>::kPosMask;
  constexpr int kQMax = QFmt<PB>::kQMax;
  if (me.ovf) return me;
  sb.assume_shared();
  uint32_t* b = sb.buf + rr;
  const int R = sb.R;
  const int cn = me.cnt;
  const float th = me.theta;
  float nth = th;
  if (cn >= kmax) {
    // #{q >= 0} = cn >= kmax; the search keeps #{q >= qL} >= kmax (verified counts only), so the
    // resulting deq(qL) is a valid theta whatever the history of re-quantisation
    int qL = 0;
    int qU = (int)q_of<PB>(me.vmax, me) + 1;  // exclusive upper end
    // (theta_only: deq(q_of<PB>(theta)) <= theta, and #{q >= q_of<PB>(theta)} >= #{lo >= theta} >= k_max holds
    // since the last full refresh verified it; the search below keeps its own counts anyway)
    if (theta_only && th > me.base) qL = min((int)q_of<PB>(th, me), qU - 1);
#pragma unroll 1
    for (int pass = 0; pass < 6 && qU - qL > 1; ++pass) {
      const int span = qU - qL;
      const uint32_t t1 = (uint32_t)(qL + (span >> 2)) << kQPosBits, t2 = (uint32_t)(qL + (span >> 1)) << kQPosBits,
                     t3 = (uint32_t)(qL + ((3 * span) >> 2)) << kQPosBits;
      int a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0}, a3[4] = {0, 0, 0, 0};
      int i = 0;
      for (; i + 8 <= cn; i += 8) {
        uint32_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = b[(i + u) * R];
#pragma unroll
        for (int u = 0; u < 8; ++u) a1[u & 3] += v[u] >= t1, a2[u & 3] += v[u] >= t2, a3[u & 3] += v[u] >= t3;
      }
      for (; i < cn; ++i) {
        const uint32_t v0 = b[i * R];
        a1[0] += v0 >= t1, a2[0] += v0 >= t2, a3[0] += v0 >= t3;
      }
      const int c1 = (a1[0] + a1[1]) + (a1[2] + a1[3]), c2 = (a2[0] + a2[1]) + (a2[2] + a2[3]),
                c3 = (a3[0] + a3[1]) + (a3[2] + a3[3]);
      const int m1 = qL + (span >> 2), m2 = qL + (span >> 1), m3 = qL + ((3 * span) >> 2);
      if (c3 >= kmax) qL = m3;
      else if (c2 >= kmax) qL = m2, qU = m3;
      else if (c1 >= kmax) qL = m1, qU = m2;
      else qU = m1;
    }
    nth = fmaxf(th, deq((uint32_t)qL, me));
  }
  if (theta_only) {
    me.theta = nth;
    return me;
  }
  // compaction: an entry's true score s < deq(q) + qe + 2 E (E the bound its score was appended
  // with, see the file header), so an entry whose bound, rounded up, is below theta is dropped.  The
  // scan's refreshes test E = E0 (the largest bound, no table loads); the final one, and a refresh
  // that would otherwise leave no room (exact fallback), test each entry's own group bound
  // perr[j & ~(kPerrGroup - 1)] (sb.perr, when the kernel supplies it).  The quantiser never changes,
  // so every entry was quantised once.
  QRow nw = me;
  nw.theta = nth;
  const float qe = qrow_qe(me);
  const float keep0 = __fsub_rd(__fsub_rd(nth, e0x2), qe);  // x >= keep0 stays
  int wpos = 0, ge = 0, i = 0;
  for (; i + 8 <= cn; i += 8) {
    uint32_t v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = b[(i + u) * R];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float x = deq(v[u] >> kQPosBits, me);
      ge += x >= nth;
      if (x >= keep0) b[wpos++ * R] = v[u];
    }
  }
  for (; i < cn; ++i) {
    const uint32_t v0 = b[i * R];
    const float x = deq(v0 >> kQPosBits, me);
    ge += x >= nth;
    if (x >= keep0) b[wpos++ * R] = v0;
  }
  const float* __restrict__ perr = sb.perr;
  if (perr && (final_pass || wpos > SLOTS - 32) && nth > -3.402823466e38f) {
    const int c0 = wpos;
    wpos = 0;
    for (i = 0; i < c0; ++i) {
      const uint32_t v0 = b[i * R];
      if (!(entry_ub(deq(v0 >> kQPosBits, me), qe, perr, v0 & kQPosMask) < nth)) b[wpos++ * R] = v0;
    }
  }
  nw.cnt = wpos;
  if (wpos > SLOTS - 32 || (nth > th && ge < kmax)) {  // no room / unverified theta: exact fallback
    nw.ovf = 1;
    nw.theta = __int_as_float(0x7f800000);
  }
  return nw;
}

// Seed threshold (build_tc2cta.cu's seed pass): slots [0, cnt) of row rr hold, as float bits, lower bounds of
// the maxima of disjoint item groups (group max of s~ minus E, rounded down: <= the true score of a distinct
// item), so the k_max-th largest of them is a valid lower bound of tau_kmax.  Returns the largest level of a
// 5-pass quaternary search over [min, vmax] that keeps at least k_max of them (-inf if cnt < k_max).
static __device__ __noinline__ float qrow_seed(QBuf sb, int rr, int cnt, float vmax, int kmax) {
  if (cnt < kmax) return -__int_as_float(0x7f800000);
  sb.assume_shared();
  const uint32_t* b = sb.buf + rr;
  const int R = sb.R;
  float m0 = vmax, m1 = vmax;
  int i = 0;
  for (; i + 2 <= cnt; i += 2) m0 = fminf(m0, __uint_as_float(b[i * R])), m1 = fminf(m1, __uint_as_float(b[(i + 1) * R]));
  for (; i < cnt; ++i) m0 = fminf(m0, __uint_as_float(b[i * R]));
  float L = fminf(m0, m1), U2 = vmax;
#pragma unroll 1
  for (int pass = 0; pass < 5; ++pass) {
    const float w = U2 - L;
    const float t1 = fmaf(w, 0.25f, L), t2 = fmaf(w, 0.5f, L), t3 = fmaf(w, 0.75f, L);
    int a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0}, a3[4] = {0, 0, 0, 0};
    int j = 0;
    for (; j + 8 <= cnt; j += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __uint_as_float(b[(j + u) * R]);
#pragma unroll
      for (int u = 0; u < 8; ++u) a1[u & 3] += v[u] >= t1, a2[u & 3] += v[u] >= t2, a3[u & 3] += v[u] >= t3;
    }
    for (; j < cnt; ++j) {
      const float v0 = __uint_as_float(b[j * R]);
      a1[0] += v0 >= t1, a2[0] += v0 >= t2, a3[0] += v0 >= t3;
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

// Append pass of one 32-column chunk (scores via s_of(j), positions pos0 + j; columns >= mi are
// padding), called by the whole warp; g4[8] are the 4-column group maxima.  Groups are skipped
// warp-uniformly; inside a group the 4 slots come from a prefix of predicates.
template <int PB = 20, typename ScoreFn>
__device__ __forceinline__ void qrow_append_chunk(ScoreFn s_of, const float (&g4)[8], float E, int pos0, int mi,
                                                  QRow& me, QBuf sb, int rr) {
  constexpr int kQPosBits = PB;  // (this function's entry format)
  sb.assume_shared();
  uint32_t* b = sb.buf + rr;
  const int R = sb.R;
  // padding columns (>= mi) hold -inf (epiq_slow) and never pass.  The quantisable-bound condition
  // lo = rd(s~ - E) >= base is folded into the threshold: it holds iff s~ >= base + E (base is a float),
  // iff s~ >= ru(base + E) -- the same appends as testing it per column
  const float thr = fmaxf(fmaxf(__fsub_rd(me.theta, E), __fadd_ru(me.base, E)), -3.402823466e38f);
  int c = me.cnt;
  float vmax = me.vmax;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    const bool gp = g4[g] >= thr;
    if (__any_sync(0xffffffffu, gp)) {
      float lo[4];
      bool p[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float sj = s_of(4 * g + j);
        lo[j] = __fsub_rd(sj, E);
        p[j] = sj >= thr;
      }
      const int o1 = c + p[0], o2 = o1 + p[1], o3 = o2 + p[2];
      if (p[0]) b[c * R] = (q_of<PB>(lo[0], me) << kQPosBits) | (uint32_t)(pos0 + 4 * g);
      if (p[1]) b[o1 * R] = (q_of<PB>(lo[1], me) << kQPosBits) | (uint32_t)(pos0 + 4 * g + 1);
      if (p[2]) b[o2 * R] = (q_of<PB>(lo[2], me) << kQPosBits) | (uint32_t)(pos0 + 4 * g + 2);
      if (p[3]) b[o3 * R] = (q_of<PB>(lo[3], me) << kQPosBits) | (uint32_t)(pos0 + 4 * g + 3);
      c = o3 + p[3];
      if (p[0] | p[1] | p[2] | p[3]) vmax = fmaxf(vmax, __fsub_rd(g4[g], E));
    }
  }
  me.cnt = c;
  me.vmax = vmax;
}

template <int SLOTS, int PB = 20>
__device__ __forceinline__ void qrow_maybe_refresh(QRow& me, QBuf sb, int rr, float e0x2, int kmax) {
  if (__any_sync(0xffffffffu, me.cnt > SLOTS - 32)) me = qrow_refresh<SLOTS, PB>(me, sb, rr, e0x2, kmax);
}

// Final compaction, then the candidate positions (or the overflow mark) are written out.  A live row
// always holds at least min(k_max, m) entries (every finite score passes while theta = -inf, and a
// refresh keeps every entry with lo >= theta, of which there are >= k_max); fewer means scores that
// never compare (NaN: a user whose norm exceeds FLT_MAX, build.cu) and the row takes the exact
// fallback.
template <int SLOTS, int PB = 20>
__device__ __forceinline__ void qrow_finish(QRow& me, QBuf sb, int rr, float e0x2, int kmax, int64_t m, int64_t row,
                                            int64_t n, int32_t* __restrict__ cand, int cstride,
                                            int32_t* __restrict__ ccount, int32_t* __restrict__ ovf_list,
                                            int* __restrict__ ovf_count) {
  me = qrow_refresh<SLOTS, PB>(me, sb, rr, e0x2, kmax, false, true);
  if (row < n) {
    if (me.ovf || (int64_t)me.cnt < (m < kmax ? m : (int64_t)kmax)) {
      ccount[row] = -1;
      const int slot = atomicAdd(ovf_count, 1);
      ovf_list[slot] = (int32_t)row;
    } else {
      ccount[row] = me.cnt;
      const uint32_t* b = sb.buf + rr;
      for (int i = 0; i < me.cnt; ++i) cand[row * cstride + i] = (int32_t)(b[i * sb.R] & QFmt<PB>::kPosMask);
    }
  }
}

}  // namespace rmips
