// build_tc2.cu -- B4 on the 5th-generation tensor cores for d <= 64 (the default d <= 64 kernel;
// build_tc.cu keeps the 4-warp variant with 8-byte entries for m > 2^20): the |Q| x |P| x d
// contraction of Alg. 1 lines 7-9 (over ALL of P per BASELINE north star) fused with
// the per-row top-k_max candidate epilogue, so the score matrix never reaches HBM.
//
// One persistent CTA per SM over 128-user tiles, 10 warps:
//   warp 0      TMA producer: user tile A (128 x 64 fp16, once per tile), item tiles B (128 x 64)
//               through a kStages-deep ring (SWIZZLE_128B)
//   warp 1      TMEM allocator + MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M = N = 128,
//               K = 4 x 16, fp32 accumulators in TMEM, kAcc = 4 stages of 128 columns
//   warps 2-9   epilogue, two warps per TMEM lane quadrant: warp w reads lanes 32 (w % 4) ..
//               of column half h = (w - 2) / 4 of every accumulator tile.  A thread owns (user
//               row, column half): its own candidate buffer (4-byte entries, candpol.cuh) and its
//               own theta, shared with the partner thread of the other half (any theta either
//               half holds is a valid lower bound of the row's tau_kmax, so the larger is used).
//   Two epilogue warps per SM sub-partition hide each other's dependency latencies; the
//   4-warp kernel (build_tc.cu) issues from one warp per sub-partition.
// Seed pass: the first seed_tiles item tiles are contracted twice.  The first time only the
// 32-column chunk maxima minus E are kept (lower bounds of distinct items' true scores); the
// k_max-th largest of the row's 4 seed_tiles maxima is a valid starting theta, which spares the
// filter the dense phase in which theta would otherwise climb from -inf.
// Early termination (Cauchy-Schwarz on the norm-sorted items) as in build_tc.cu, with 8 epilogue
// warps reporting per user tile.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "candpol.cuh"
#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace rmips {

namespace {

constexpr int kBM = 128;                  // users per tile (TMEM lanes)
constexpr int kBN = 128;                  // items per tile (accumulator columns)
constexpr int kStages = 4;                // smem ring depth for item tiles
constexpr int kAcc = 4;                   // TMEM accumulator stages (kAcc * kBN = 512 columns)
constexpr int kTileBytes = kBM * 64 * 2;  // one 128 x 64 fp16 tile = 16 KB
constexpr int kThreads = 320;
constexpr int kEpiWarps = 8;
constexpr int kRows2 = 2 * kBM;           // candidate-buffer rows: (column half, user row)

struct Smem2 {
  static constexpr int A = 0;
  static constexpr int B = kTileBytes;
  static constexpr int CAND = B + kStages * kTileBytes;            // [128 slots][256 rows] u32
  static constexpr int PUB = CAND + 128 * kRows2 * 4;              // [5][256] half-row exchange
  static constexpr int BAR = PUB + 5 * kRows2 * 4;
  static constexpr int TOTAL = BAR + 256 + 1024;                   // + alignment slack
  static_assert(TOTAL <= 232448, "shared memory");
};

// max of a 32-column chunk (3-input max trees).  The fast path is one compare of it per chunk;
// padding columns of a ragged last tile are TMA zero fill: at worst they flag a chunk, and the
// slow path masks them before appending.
__device__ __forceinline__ float chunk_max32(const uint32_t (&h)[32]) {
  float g[8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
    g[i] = fmaxf(fmaxf(__uint_as_float(h[4 * i]), __uint_as_float(h[4 * i + 1])),
                 fmaxf(__uint_as_float(h[4 * i + 2]), __uint_as_float(h[4 * i + 3])));
  return fmaxf(fmaxf(fmaxf(g[0], g[1]), fmaxf(g[2], g[3])), fmaxf(fmaxf(g[4], g[5]), fmaxf(g[6], g[7])));
}

// Slow path (one copy per kernel): re-read each flagged chunk from TMEM, append, and refresh when
// a row of the warp may not have room for another chunk.  Before a refresh theta is raised to the
// partner half's published theta; after it, this half's theta is published.
template <class Pol>
__device__ __noinline__ typename Pol::Row epi2_slow(uint32_t bits, uint32_t taddr, int base0, int mi, float E0,
                                                    float E1, typename Pol::Row me, typename Pol::Buf sb, int rr,
                                                    float e0x2, int kmax, volatile float* pub_me,
                                                    volatile float* pub_pt) {
  sb.assume_shared();
#pragma unroll 1
  while (bits) {
    const int c = __ffs(bits) - 1;
    bits &= bits - 1;
    uint32_t r[32];
    sm100::tmem_ld32(taddr + 32 * c, r);
    sm100::tmem_ld_wait(r);
    const int pos0 = base0 + 32 * c;
    if (pos0 + 32 > mi) {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (pos0 + j >= mi) r[j] = 0xff800000u;  // -inf
    }
    float g4[8];
#pragma unroll
    for (int g = 0; g < 8; ++g)
      g4[g] = fmaxf(fmaxf(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1])),
                    fmaxf(__uint_as_float(r[4 * g + 2]), __uint_as_float(r[4 * g + 3])));
    Pol::append([&](int j) { return __uint_as_float(r[j]); }, g4, c ? E1 : E0, pos0, mi, me, sb, rr);
    if (__any_sync(0xffffffffu, me.cnt > Pol::kSlots - 32)) {
      if (!me.ovf) me.theta = fmaxf(me.theta, *pub_pt);
      me = Pol::refresh(me, sb, rr, e0x2, kmax);
      *pub_me = me.ovf ? -__int_as_float(0x7f800000) : me.theta;
    }
  }
  return me;
}

// k_max-th largest of cn lower bounds f[i * kBM] (i < cn >= kmax): the largest level of a 5-pass
// quaternary search over [min, max] keeping at least kmax values (-inf if cn < kmax).
__device__ __noinline__ float seed_theta(const float* f, int cn, int kmax) {
  if (cn < kmax) return -__int_as_float(0x7f800000);
  __builtin_assume(__isShared(f));
  float lo0 = f[0], lo1 = f[0], hi0 = f[0], hi1 = f[0];
  int i = 1;
  for (; i + 2 <= cn; i += 2) {
    const float a = f[i * kBM], b = f[(i + 1) * kBM];
    lo0 = fminf(lo0, a), hi0 = fmaxf(hi0, a), lo1 = fminf(lo1, b), hi1 = fmaxf(hi1, b);
  }
  if (i < cn) lo0 = fminf(lo0, f[i * kBM]), hi0 = fmaxf(hi0, f[i * kBM]);
  float L = fminf(lo0, lo1), U = fmaxf(hi0, hi1);
#pragma unroll 1
  for (int pass = 0; pass < 5; ++pass) {
    const float w = U - L;
    const float t1 = fmaf(w, 0.25f, L), t2 = fmaf(w, 0.5f, L), t3 = fmaf(w, 0.75f, L);
    int a1[4] = {0, 0, 0, 0}, a2[4] = {0, 0, 0, 0}, a3[4] = {0, 0, 0, 0};
    i = 0;
    for (; i + 8 <= cn; i += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = f[(i + u) * kBM];
#pragma unroll
      for (int u = 0; u < 8; ++u) a1[u & 3] += v[u] >= t1, a2[u & 3] += v[u] >= t2, a3[u & 3] += v[u] >= t3;
    }
    for (; i < cn; ++i) {
      const float v0 = f[i * kBM];
      a1[0] += v0 >= t1, a2[0] += v0 >= t2, a3[0] += v0 >= t3;
    }
    const int c1 = (a1[0] + a1[1]) + (a1[2] + a1[3]), c2 = (a2[0] + a2[1]) + (a2[2] + a2[3]),
              c3 = (a3[0] + a3[1]) + (a3[2] + a3[3]);
    if (c3 >= kmax) L = t3;
    else if (c2 >= kmax) L = t2, U = t3;
    else if (c1 >= kmax) L = t1, U = t2;
    else U = t1;
  }
  return L;
}

// Joint threshold of a row's two halves (finish of a user tile, both halves synchronised): the
// largest level of a 5-pass quaternary search over [L, U] with #{own lo >= t} + #{partner lo >= t}
// >= kmax (L itself is a valid theta; the counts are exact for the fp32 levels, so the result is
// valid by construction).  Entries are candq.cuh words, dequantised with each half's (base, w).
__device__ __noinline__ float joint_theta(const uint32_t* own, int cn, float base, float w, const uint32_t* pt, int cp,
                                          float base_p, float w_p, float L, float U, int kmax) {
  __builtin_assume(__isShared(own));
  __builtin_assume(__isShared(pt));
#pragma unroll 1
  for (int pass = 0; pass < 5; ++pass) {
    const float wd = U - L;
    const float t1 = fmaf(wd, 0.25f, L), t2 = fmaf(wd, 0.5f, L), t3 = fmaf(wd, 0.75f, L);
    int a1 = 0, a2 = 0, a3 = 0, b1 = 0, b2 = 0, b3 = 0;
    int i = 0;
    for (; i + 4 <= cn; i += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float x = __fadd_rd(base, (float)(own[(i + u) * kRows2] >> kQPosBits) * w);
        a1 += x >= t1, a2 += x >= t2, a3 += x >= t3;
      }
    }
    for (; i < cn; ++i) {
      const float x = __fadd_rd(base, (float)(own[i * kRows2] >> kQPosBits) * w);
      a1 += x >= t1, a2 += x >= t2, a3 += x >= t3;
    }
    i = 0;
    for (; i + 4 <= cp; i += 4) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float x = __fadd_rd(base_p, (float)(pt[(i + u) * kRows2] >> kQPosBits) * w_p);
        b1 += x >= t1, b2 += x >= t2, b3 += x >= t3;
      }
    }
    for (; i < cp; ++i) {
      const float x = __fadd_rd(base_p, (float)(pt[i * kRows2] >> kQPosBits) * w_p);
      b1 += x >= t1, b2 += x >= t2, b3 += x >= t3;
    }
    if (a3 + b3 >= kmax) L = t3;
    else if (a2 + b2 >= kmax) L = t2, U = t3;
    else if (a1 + b1 >= kmax) L = t1, U = t2;
    else U = t1;
  }
  return L;
}

}  // namespace

template <class Pol>
__global__ void __launch_bounds__(kThreads, 1)
k_build_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
            const float* __restrict__ perr, const double* __restrict__ pnorm, const float* __restrict__ pscale,
            int cs_enable, int64_t n, int64_t m, int kmax, int seed_tiles, int32_t* __restrict__ cand,
            int32_t* __restrict__ ccount, int32_t* __restrict__ ovf_list, int* __restrict__ ovf_count,
            unsigned long long* __restrict__ tiles_done) {
  using namespace sm100;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sA = sbase + Smem2::A;
  const uint32_t sB = sbase + Smem2::B;
  const typename Pol::Buf sb{reinterpret_cast<uint32_t*>(smem + Smem2::CAND), kRows2};
  // half-row exchange, each [2 halves][128 rows]: theta (valid; -inf if overflowed), entry count
  // (-1: overflowed), and the quantiser base / quantum / largest bound of the final buffer
  float* thpub = reinterpret_cast<float*>(smem + Smem2::PUB);
  int* cntpub = reinterpret_cast<int*>(thpub + kRows2);
  float* basepub = reinterpret_cast<float*>(cntpub + kRows2);
  float* wpub = basepub + kRows2;
  float* vmaxpub = wpub + kRows2;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Smem2::BAR);
  const uint32_t bar0 = smem_u32(bars);
  auto BAR = [&](int i) { return bar0 + 8u * i; };
  const int A_FULL = 0, A_EMPTY = 1, B_FULL = 2, B_EMPTY = 2 + kStages, ACC_FULL = 2 + 2 * kStages,
            ACC_EMPTY = 2 + 2 * kStages + kAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 + 2 * kStages + 2 * kAcc);
  volatile int* done_cum = reinterpret_cast<volatile int*>(tmem_slot + 1);
  volatile int* stage_end = done_cum + 1;
  volatile int* acc_end = stage_end + kStages;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_utiles = (int)((n + kBM - 1) / kBM);
  const int nit = (int)((m + kBN - 1) / kBN);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    mbar_init(BAR(A_FULL), 1);
    mbar_init(BAR(A_EMPTY), 1);
    for (int s = 0; s < kStages; ++s) mbar_init(BAR(B_FULL + s), 1), mbar_init(BAR(B_EMPTY + s), 1);
    for (int a = 0; a < kAcc; ++a) mbar_init(BAR(ACC_FULL + a), 1), mbar_init(BAR(ACC_EMPTY + a), kEpiWarps);
    *done_cum = 0;
    for (int s = 0; s < kStages; ++s) stage_end[s] = 0;
    for (int a = 0; a < kAcc; ++a) acc_end[a] = 0;
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(smem_u32(tmem_slot), kAcc * kBN);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0;
      int t = 0;
      for (int ut = blockIdx.x; ut < num_utiles; ut += gridDim.x, ++t) {
        if (t > 0) mbar_wait_sleep(BAR(A_EMPTY), (t - 1) & 1);
        mbar_arrive_expect_tx(BAR(A_FULL), kTileBytes);
        tma_load_2d(sA, &tmA, 0, ut * kBM, BAR(A_FULL));
        for (int j = 0; j < seed_tiles + nit; ++j) {  // seed pass, then all item tiles
          const int it = j < seed_tiles ? j : j - seed_tiles;
          mbar_wait_sleep(BAR(B_EMPTY + stage), ph ^ 1);
          if (*done_cum >= kEpiWarps * (t + 1)) {  // every epilogue warp is done with this user tile
            stage_end[stage] = t + 1;
            mbar_arrive(BAR(B_FULL + stage));  // release: the marker is visible to the MMA warp
            if (++stage == kStages) stage = 0, ph ^= 1;
            break;
          }
          mbar_arrive_expect_tx(BAR(B_FULL + stage), kTileBytes);
          tma_load_2d(sB + stage * kTileBytes, &tmB, 0, it * kBN, BAR(B_FULL + stage));
          if (++stage == kStages) stage = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16_f32(kBM, kBN);
      unsigned long long tiles_issued = 0;  // distinct (user tile, item tile) contractions
      int stage = 0, as = 0;
      uint32_t ph = 0, aph = 0;
      int t = 0;
      for (int ut = blockIdx.x; ut < num_utiles; ut += gridDim.x, ++t) {
        mbar_wait_sleep(BAR(A_FULL), t & 1);
        tc_fence_after();
        for (int j = 0; j < seed_tiles + nit; ++j) {
          mbar_wait_sleep(BAR(ACC_EMPTY + as), aph ^ 1);
          mbar_wait_sleep(BAR(B_FULL + stage), ph);
          tc_fence_after();
          if (stage_end[stage] == t + 1) {  // the producer ended this user tile: forward the marker
            mbar_arrive(BAR(B_EMPTY + stage));
            acc_end[as] = t + 1;
            mbar_arrive(BAR(ACC_FULL + as));
            if (++stage == kStages) stage = 0, ph ^= 1;
            if (++as == kAcc) as = 0, aph ^= 1;
            break;
          }
          const uint32_t d = tmem + as * kBN;
          const uint32_t b0 = sB + stage * kTileBytes;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_f16(d, sdesc_sw128(sA + kk * 32), sdesc_sw128(b0 + kk * 32), idesc, kk != 0);
          mma_commit(BAR(B_EMPTY + stage));
          mma_commit(BAR(ACC_FULL + as));
          tiles_issued += j >= seed_tiles;  // the seed pass repeats tiles: not counted
          if (++stage == kStages) stage = 0, ph ^= 1;
          if (++as == kAcc) as = 0, aph ^= 1;
        }
        mma_commit(BAR(A_EMPTY));
      }
      atomicAdd(tiles_done, (unsigned long long)tiles_issued);
    }
  } else {
    // ------------------------------------------------ epilogue: one thread per (user row, half)
    const int h = (warp - 2) >> 2;             // column half of every accumulator tile
    const int q = warp & 3;                    // TMEM lane quadrant
    const int rloc = q * 32 + lane;            // user row within the tile
    const int rr = h * kBM + rloc;             // candidate-buffer row
    const int mi = (int)m;
    const float e0x2 = __fadd_ru(__ldg(perr), __ldg(perr));
    const float pscl = __ldg(pscale);
    // |s~| <= smax for every score (candq.cuh's quantiser range; generous margins)
    const float smax = __fadd_ru(__fmul_ru((float)(__ldg(pnorm) * (double)pscl), 1.02f), __fmul_ru(2.f, e0x2));
    volatile float* pub_me = thpub + h * kBM + rloc;
    volatile float* pub_pt = thpub + (1 - h) * kBM + rloc;
    const float ninf = -__int_as_float(0x7f800000);
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(1 + q) : "memory"); };
    int as = 0;
    uint32_t aph = 0;
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + h * 64;
    constexpr int kCsEvery = 4;
    // 32-column chunks are double-buffered (r0: chunk 0 of the current tile's half, r1: chunk 1);
    // 10 warps leave 168 registers per thread (3 warps on two of the SM sub-partitions)
    uint32_t r0[32], r1[32];
    int t = 0;
    for (int ut = blockIdx.x; ut < num_utiles; ut += gridDim.x, ++t) {
      const int64_t row = (int64_t)ut * kBM + rloc;
      typename Pol::Row me = Pol::init(row < n, smax);  // dead rows: theta = +inf, never pass
      *pub_me = ninf;
      mbar_wait(BAR(ACC_FULL + as), aph);
      tc_fence_after();
      tmem_ld32(tq + as * kBN, r0);
      tmem_ld_wait(r0);
      if (seed_tiles > 0) {
        // seed pass: chunk maxima of this half into the row's float slots 4 j + 2 h + c
        float* fs = reinterpret_cast<float*>(sb.buf) + rloc;  // float view [slot][128 rows]
        for (int j = 0; j < seed_tiles; ++j) {
          const int b0 = j * kBN + 64 * h;
          tmem_ld32(tq + as * kBN + 32, r1);
          const float l0 = __fsub_rd(chunk_max32(r0), __ldg(perr + b0));
          tmem_ld_wait(r1);
          const float l1 = __fsub_rd(chunk_max32(r1), __ldg(perr + b0 + 32));
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(BAR(ACC_EMPTY + as));
          if (++as == kAcc) as = 0, aph ^= 1;
          mbar_wait(BAR(ACC_FULL + as), aph);  // the main pass follows: always a next stage
          tc_fence_after();
          tmem_ld32(tq + as * kBN, r0);
          fs[(4 * j + 2 * h) * kBM] = l0;
          fs[(4 * j + 2 * h + 1) * kBM] = l1;
          tmem_ld_wait(r0);
        }
        pair_sync();  // both halves' maxima are in
        const float s = seed_theta(fs, 4 * seed_tiles, kmax);
        pair_sync();  // both halves have read them: the slots become candidate entries
        Pol::seed(me, s, e0x2);
      }
      float En0 = (64 * h < mi) ? __ldg(perr + 64 * h) : 0.f, En1 = (64 * h + 32 < mi) ? __ldg(perr + 64 * h + 32) : 0.f;
      double pnr = nit > kCsEvery ? __ldg(pnorm + kCsEvery * kBN) : 0.0;  // raw norm, scaled at use
      int it = 0;
      bool done = false;  // warp-uniform: this warp's rows cannot gain any more
      // one item tile: r0 holds chunk 0 of this half of tile it (loaded); chunk 1 is loaded into
      // r1 while chunk 0 is checked, and chunk 0 of the next tile into r0 while the slow path runs
      auto step = [&]() -> bool {
        const int base0 = it * kBN + 64 * h;
        const float E0 = En0, E1 = En1;
        const bool more = it + 1 < nit;
        En0 = (base0 + kBN < mi) ? __ldg(perr + base0 + kBN) : 0.f;
        En1 = (base0 + kBN + 32 < mi) ? __ldg(perr + base0 + kBN + 32) : 0.f;
        const int as_next = as + 1 == kAcc ? 0 : as + 1;
        const uint32_t aph_next = as + 1 == kAcc ? aph ^ 1 : aph;
        tmem_ld32(tq + as * kBN + 32, r1);
        const bool p0 = __fadd_ru(chunk_max32(r0), E0) >= me.theta;
        tmem_ld_wait(r1);
        const bool p1 = __fadd_ru(chunk_max32(r1), E1) >= me.theta;
        if (more) {
          mbar_wait(BAR(ACC_FULL + as_next), aph_next);
          tc_fence_after();
          tmem_ld32(tq + as_next * kBN, r0);
        }
        const uint32_t bits = (uint32_t)__any_sync(0xffffffffu, p0) | ((uint32_t)__any_sync(0xffffffffu, p1) << 1);
        if (bits) me = epi2_slow<Pol>(bits, tq + as * kBN, base0, mi, E0, E1, me, sb, rr, e0x2, kmax, pub_me, pub_pt);
        tc_fence_before();  // this stage is no longer read: release it
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(ACC_EMPTY + as));
        as = as_next;
        aph = aph_next;
        if (!more) return true;
        tmem_ld_wait(r0);
        ++it;
        if (it % kCsEvery == 0) {
          // every item from tile it on has scaled true score <= |p_first(it)| 2^e (1 + 2^-16)
          const float pnn = cs_enable ? __double2float_ru(pnr * (double)pscl) : __int_as_float(0x7f800000);
          const uint32_t mk = __reduce_min_sync(0xffffffffu, f2key(me.theta));
          if (__fmul_ru(pnn, 1.0000153f) < key2f(mk)) {
            done = true;
            return true;
          }
          if ((it + kCsEvery) * kBN < mi) pnr = __ldg(pnorm + (it + kCsEvery) * kBN);
        }
        return false;
      };
      while (!step()) {
      }
      if (lane == 0) atomicAdd(const_cast<int*>(done_cum), 1);  // one event per warp and user tile
      if (done) {  // drain: release the remaining stages unread; stage `as` (tile it) is full
        for (; it < nit; ++it) {
          const bool end = acc_end[as] == t + 1;
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(BAR(ACC_EMPTY + as));
          if (++as == kAcc) as = 0, aph ^= 1;
          if (end || it + 1 == nit) break;
          mbar_wait(BAR(ACC_FULL + as), aph);
          tc_fence_after();
        }
      }
      // finish: the joint theta of both halves (k_max-th largest bound over the row's two buffers),
      // then each half compacts with it and one candidate list per row is written
      const int mine = h * kBM + rloc, other = (1 - h) * kBM + rloc;
      *pub_me = me.ovf ? ninf : me.theta;
      cntpub[mine] = me.ovf ? -1 : me.cnt;
      basepub[mine] = me.base;
      wpub[mine] = me.w;
      vmaxpub[mine] = me.vmax;
      pair_sync();
      if (!me.ovf && row < n && cntpub[other] >= 0) {
        const int cp = cntpub[other];
        const float L = fmaxf(me.theta, *pub_pt), U = fmaxf(me.vmax, vmaxpub[other]);
        if (me.cnt + cp >= kmax && U > L)
          me.theta = joint_theta(sb.buf + rr, me.cnt, me.base, me.w, sb.buf + other, cp, basepub[other], wpub[other],
                                 L, U, kmax);
        else
          me.theta = L;
      }
      pair_sync();  // both halves are done reading each other's buffer
      me = Pol::refresh(me, sb, rr, e0x2, kmax);
      cntpub[h * kBM + rloc] = me.ovf ? -1 : me.cnt;
      pair_sync();
      const int pc = cntpub[(1 - h) * kBM + rloc];
      if (row < n) {
        if (me.ovf || pc < 0 || me.cnt + pc > kCand) {
          if (h == 0) {
            ccount[row] = -1;
            const int slot = atomicAdd(ovf_count, 1);
            ovf_list[slot] = (int32_t)row;
          }
        } else {
          if (h == 0) ccount[row] = me.cnt + pc;
          const uint32_t* b = sb.buf + rr;
          int32_t* dst = cand + row * kCand + (h ? pc : 0);
          for (int i = 0; i < me.cnt; ++i) dst[i] = Pol::pos(b[i * kRows2]);
        }
      }
      pair_sync();  // the buffer is reused by the next user tile's seed pass
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kAcc * kBN);
}

// ------------------------------------------------------------------------------ host side
namespace {
int sm_count2() {
  static int c = 0;
  if (!c) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
  }
  return c;
}
}  // namespace

template <class Pol>
static cudaError_t launch_tc2(const BuildCtx& c, cudaStream_t st) {
  rmips_index_s* x = c.idx;
  CUtensorMap ta, tb;
  if (!make_tmap_f16_box(&ta, x->U16, (uint64_t)x->n, (uint64_t)x->dpad, kBM)) return cudaErrorNotSupported;
  if (!make_tmap_f16_box(&tb, x->P16, (uint64_t)c.mb, (uint64_t)x->dpad, kBN)) return cudaErrorNotSupported;
  cudaError_t e = cudaFuncSetAttribute(k_build_tc2<Pol>, cudaFuncAttributeMaxDynamicSharedMemorySize, Smem2::TOTAL);
  if (e != cudaSuccess) return e;
  const int tiles = (int)((x->n + kBM - 1) / kBM);
  const int grid = tiles < sm_count2() ? tiles : sm_count2();
  const int cs = getenv("RMIPS_NO_CS") ? 0 : 1;  // dev A/B switch for the C-S exit
  // seed pass: at most 32 full tiles (128 maxima fill the float view of the buffer), >= k_max maxima
  const int nit = (int)((c.mb + kBN - 1) / kBN);
  int seed = nit >= 16 ? (nit / 4 < 32 ? nit / 4 : 32) : 0;
  if (const char* s = getenv("RMIPS_SEED_TILES")) seed = atoi(s) < seed ? atoi(s) : seed;  // dev switch
  if (4 * seed < x->kmax) seed = 0;
  k_build_tc2<Pol><<<grid, kThreads, Smem2::TOTAL, st>>>(ta, tb, x->perr, x->pnorm, c.scale_dev, cs, x->n, c.mb,
                                                          x->kmax, seed, c.cand, c.ccount, c.ovf_list, c.ovf_count,
                                                          c.tiles_done);
  count_launch();
  return cudaGetLastError();
}

// d_pad = 64, k_max <= 64 (each half-row buffer must be able to hold k_max entries below its
// refresh trigger) and m <= 2^20 (20-bit positions); otherwise cudaErrorNotSupported
// (build_tc.cu's 8-byte-entry kernel).
cudaError_t build_tc2(const BuildCtx& c, cudaStream_t st) {
  if (c.idx->dpad != 64 || c.idx->kmax > 64) return cudaErrorNotSupported;
  if (c.mb <= (int64_t)kQPosMask + 1) return launch_tc2<QPol>(c, st);
  return cudaErrorNotSupported;
}

}  // namespace rmips
