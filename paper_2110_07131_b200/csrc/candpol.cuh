// candpol.cuh -- the 4-byte candidate-entry policy of the tensor-core build kernel build_tcq.cu
// behind a small interface:
//   QPol  candq.cuh: 12-bit quantised lower bound | 20-bit position (m <= 2^20)
// It keeps cand.cuh's invariant: theta is a valid lower bound of the row's
// k_max-th largest true score, an item is appended iff s~ >= theta - E, and an entry is dropped
// only when its upper bound is below theta.
#pragma once
#include "candq.cuh"
#include "common.cuh"

namespace rmips {

struct QPol {
  using Row = QRow;
  using Buf = QBuf;
  static constexpr int kSlots = kQSlots;
  __device__ static Row init(bool live, float smax) { return qrow_init(live, smax); }
  // theta <- max(theta, s) for a valid lower bound s, on an EMPTY buffer: the quantiser is rebased
  // to [s - 2 E0 - 2 w, smax] (as a refresh would), so appended entries keep lo >= base
  __device__ static void seed(Row& me, float s, float e0x2) {
    if (!(s > me.theta) || me.cnt != 0 || me.ovf) return;
    me.theta = s;
    me.base = __fsub_rd(__fsub_rd(s, e0x2), __fmul_ru(2.f, me.w));
    const float span = __fsub_ru(me.smax, me.base);
    me.w = pow2_ceil(fmaxf(span, fabsf(me.base) * 1e-6f + 1e-30f) / (float)kQMax);
    me.inv = 1.f / me.w;
  }
  template <typename F>
  __device__ static void append(F f, const float (&g4)[8], float E, int pos0, int mi, Row& me, Buf sb, int rr) {
    qrow_append_chunk(f, g4, E, pos0, mi, me, sb, rr);
  }
  __device__ static Row refresh(Row me, Buf sb, int rr, float e0x2, int kmax) {
    return qrow_refresh(me, sb, rr, e0x2, kmax);
  }
  __device__ static void maybe_refresh(Row& me, Buf sb, int rr, float e0x2, int kmax) {
    qrow_maybe_refresh(me, sb, rr, e0x2, kmax);
  }
  __device__ static void finish(Row& me, Buf sb, int rr, float e0x2, int kmax, int64_t m, int64_t row, int64_t n,
                                int32_t* cand,
                                int32_t* ccount, int32_t* ovf_list, int* ovf_count) {
    qrow_finish(me, sb, rr, e0x2, kmax, m, row, n, cand, ccount, ovf_list, ovf_count);
  }
  __device__ static int32_t pos(uint32_t e) { return (int32_t)(e & kQPosMask); }
};

}  // namespace rmips
