// candpol.cuh -- the candidate-entry policies of the tensor-core build kernel build_tcq.cu behind one
// small interface:
//   QPolT<SLOTS, PB>  candq.cuh: 4-byte entries, quantised lower bound | PB-bit position (PB = 20 or 21)
//                 (m <= 2^20); SLOTS = 128 (k_max <= 80) or 256 (larger k_max)
//   FPol          cand.cuh: 8-byte entries {lo, position} (any m < 2^31), 128 slots
// Every policy keeps cand.cuh's invariant: theta is a valid lower bound of the row's
// k_max-th largest true score, an item is appended iff s~ >= theta - E, and an entry is dropped only
// when its upper bound is below theta.
#pragma once
#include "cand.cuh"
#include "candq.cuh"
#include "common.cuh"

namespace rmips {

template <int SLOTS, int PB = 20>  // PB position bits (20: m <= 2^20; 21: m <= 2^21, an 11-bit bound)
struct QPolT {
  using Row = QRow;
  using Buf = QBuf;
  static constexpr int kSlots = SLOTS;
  static constexpr int kBufBytes = 128 * SLOTS * 4;  // 128 rows
  static constexpr int64_t kMaxItems = (int64_t)QFmt<PB>::kPosMask + 1;
  // perr: the per-item error table (the final drop tests each entry's own bound, candq.cuh)
  __device__ static Buf buf(uint8_t* p, const float* perr) { return QBuf{reinterpret_cast<uint32_t*>(p), 128, perr}; }
  __device__ static Row init(bool live, float smax) { return qrow_init<PB>(live, smax); }
  template <typename F>
  __device__ static void append(F f, const float (&g4)[8], float E, int pos0, int mi, Row& me, Buf sb, int rr) {
    qrow_append_chunk<PB>(f, g4, E, pos0, mi, me, sb, rr);
  }
  __device__ static void maybe_refresh(Row& me, Buf sb, int rr, float e0x2, int kmax) {
    qrow_maybe_refresh<SLOTS, PB>(me, sb, rr, e0x2, kmax);
  }
  __device__ static void refresh_theta(Row& me, Buf sb, int rr, float e0x2, int kmax) {  // (whole warp)
    me = qrow_refresh<SLOTS, PB>(me, sb, rr, e0x2, kmax, true);
  }
  __device__ static void compact(Row& me, Buf sb, int rr, float e0x2, int kmax) {  // (whole warp)
    me = qrow_refresh<SLOTS, PB>(me, sb, rr, e0x2, kmax);
  }
  static constexpr int kEntWords = SLOTS;  // 32-bit words of a row's saved entries
  // seed pass: value i of the row (float bits) in slot i; the k_max-th largest of cnt values
  __device__ static void seed_store(Buf sb, int rr, int i, float v) { sb.buf[i * sb.R + rr] = __float_as_uint(v); }
  __device__ static float seed_theta(Buf sb, int rr, int cnt, float vmax, int kmax) {
    return qrow_seed(sb, rr, cnt, vmax, kmax);
  }
  // Row state of a two-pass (regrouped) build: entries row-major at ent[row * SLOTS ..], {theta, vmax,
  // cnt, ovf} at meta[row]; the quantiser (base, w) depends on smax only, the same in both passes
  __device__ static void save(const Row& me, Buf sb, int rr, uint32_t* ent, uint4* meta, int64_t row) {
    sb.assume_shared();
    const uint32_t* b = sb.buf + rr;
    uint32_t* o = ent + row * SLOTS;
    for (int i = 0; i < me.cnt; ++i) o[i] = b[i * sb.R];
    meta[row] = make_uint4(__float_as_uint(me.theta), __float_as_uint(me.vmax), (uint32_t)me.cnt, (uint32_t)me.ovf);
  }
  __device__ static void load(Row& me, Buf sb, int rr, const uint32_t* ent, const uint4* meta, int64_t row) {
    const uint4 mt = __ldg(meta + row);
    me.theta = __uint_as_float(mt.x);
    me.vmax = __uint_as_float(mt.y);
    me.cnt = (int)mt.z;
    me.ovf = (int)mt.w;
    sb.assume_shared();
    uint32_t* b = sb.buf + rr;
    const uint32_t* s = ent + row * SLOTS;
    for (int i = 0; i < me.cnt; ++i) b[i * sb.R] = __ldg(s + i);
  }
  __device__ static void finish(Row& me, Buf sb, int rr, float e0x2, int kmax, int64_t m, int64_t row, int64_t n,
                                int32_t* cand, int32_t* ccount, int32_t* ovf_list, int* ovf_count) {
    qrow_finish<SLOTS, PB>(me, sb, rr, e0x2, kmax, m, row, n, cand, SLOTS, ccount, ovf_list, ovf_count);
  }
};

struct FPol {
  using Row = CandRow;
  using Buf = CandSmem;
  static constexpr int kSlots = kCand;
  static constexpr int kBufBytes = kCandSmemBytes;
  static constexpr int64_t kMaxItems = (int64_t)1 << 31;
  __device__ static Buf buf(uint8_t* p, const float*) { return CandSmem::at(p); }
  __device__ static Row init(bool live, float) { return cand_init(live); }
  template <typename F>
  __device__ static void append(F f, const float (&g4)[8], float E, int pos0, int, Row& me, Buf sb, int rr) {
    cand_append_chunk(f, g4, E, pos0, me, sb, rr);  // columns >= m hold -inf (epiq_slow): never appended
  }
  __device__ static void maybe_refresh(Row& me, Buf sb, int rr, float e0x2, int kmax) {
    cand_maybe_refresh(me, sb, rr, e0x2, kmax);
  }
  __device__ static void refresh_theta(Row& me, Buf sb, int rr, float e0x2, int kmax) {  // (whole warp)
    me = cand_refresh(me, sb, rr, e0x2, kmax, true);
  }
  __device__ static void finish(Row& me, Buf sb, int rr, float e0x2, int kmax, int64_t m, int64_t row, int64_t n,
                                int32_t* cand, int32_t* ccount, int32_t* ovf_list, int* ovf_count) {
    cand_finish(me, sb, rr, e0x2, kmax, m, row, n, cand, kCand, ccount, ovf_list, ovf_count);
  }
  __device__ static void compact(Row& me, Buf sb, int rr, float e0x2, int kmax) {  // (whole warp)
    me = cand_refresh(me, sb, rr, e0x2, kmax);
  }
  static constexpr int kEntWords = 2 * kCand;  // 8-byte entries
  __device__ static void save(const Row& me, Buf sb, int rr, uint32_t* ent, uint4* meta, int64_t row) {
    cand_save(me, sb, rr, reinterpret_cast<uint2*>(ent), meta, row);
  }
  __device__ static void load(Row& me, Buf sb, int rr, const uint32_t* ent, const uint4* meta, int64_t row) {
    cand_load(me, sb, rr, reinterpret_cast<const uint2*>(ent), meta, row);
  }
  // seed pass: two values per 8-byte slot (as k_build_tc's seed), the k_max-th largest via cand_seed
  __device__ static void seed_store(Buf sb, int rr, int i, float v) {
    uint32_t* w = reinterpret_cast<uint32_t*>(sb.buf + (i >> 1) * kCandRows + rr);
    w[i & 1] = __float_as_uint(v);
  }
  __device__ static float seed_theta(Buf sb, int rr, int cnt, float vmax, int kmax) {
    CandRow t = cand_init(true);
    t.cnt = cnt >> 1;
    t.vmax = vmax;
    return cand_seed(t, sb, rr, kmax);
  }
};

// FPol with the branch-free append of k_build_tc's slow path (every column's slot from a running count; no
// per-group votes): the CTA-pair kernel at d_pad = 64 (development switch RMIPS_2CTA_FPOL=2)
struct FPolFlat : FPol {
  template <typename F>
  __device__ static void append(F f, const float (&g4)[8], float E, int pos0, int, Row& me, Buf sb, int rr) {
    const float mx = fmaxf(fmaxf(fmaxf(g4[0], g4[1]), fmaxf(g4[2], g4[3])), fmaxf(fmaxf(g4[4], g4[5]), fmaxf(g4[6], g4[7])));
    cand_append_flat(f, mx, E, pos0, me, sb, rr);  // columns >= m hold -inf (epiq_slow): never appended
  }
};

}  // namespace rmips
