// build_tcq.cu -- B4 on the 5th-generation tensor cores for any d (build_tc.cu has the faster d <= 64
// kernel for k_max <= 80): the |Q| x |P| x d contraction of Alg. 1 lines 7-9 (over ALL of
// P per BASELINE north star) fused with the per-row top-k_max candidate epilogue (candpol.cuh), so the
// score matrix never reaches HBM.
//
// k_build_tcq<KB, Pol>: K = 64*KB columns (d_pad), 128-user tiles, 128-item tiles.  One persistent CTA
// per SM; per user tile:
//   warp 0      TMA producer: one ring of 16 KB K-block units (128 rows x 64 fp16, SWIZZLE_128B); the
//               last K block of a row is trimmed to the columns that hold data (a 16-, 32- or 64-column
//               box, tail_cols(d): d = 200 streams 416 instead of 512 bytes per row)
//   warp 1      MMA warp (all lanes run the loop, one elected lane issues):
//                 KB = 1..4  the user tile A is copied into TENSOR memory with tcgen05.cp (8 columns per
//                            K step, in issue order after the previous tile's MMAs); every item tile is
//                            then one tcgen05.mma.cta_group::1.kind::f16 chain, M = N = 128,
//                            K = 16 x ksteps, A from TMEM, only B from shared memory (an MMA that also
//                            re-read A from shared memory needs more than the SM's 128 B/clk)
//                 KB = 0     d_pad > 256 (A does not fit next to the accumulators): the K loop streams
//                            the user tile's K blocks next to the item tile's (A and B from shared
//                            memory; A re-read from L2 per item tile), kbn = d_pad / 64 at run time
//   warps 2-5   epilogue: warp w reads TMEM lane quadrant w % 4; every thread owns one user row and
//               filters its 128 scores per item tile (3-input max trees, one compare per 32-column
//               chunk), with one out-of-line slow path that re-reads flagged chunks.
// Pol: the candidate entries (candpol.cuh): 4-byte quantised (m <= 2^20; 128 or 256 slots) or 8-byte.
// Early termination (Cauchy-Schwarz on the norm-sorted items) as in build_tc.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "candpol.cuh"
#include "common.cuh"
#include "epiq.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace rmips {

namespace {

// development-only experiment switches (librmips_dev.so reads them from the environment)
constexpr int kDevNoFeed = 1;   // RMIPS_NOFEED: item units after the first ring round are not reloaded
constexpr int kDevEpiSkip = 2;  // RMIPS_EPI_SKIP: the epilogue releases every stage unread
constexpr int kDevEpiLoad = 4;  // RMIPS_EPI_LOAD: ... after reading it from TMEM (no filter work)

constexpr int kBM = 128;                 // users per tile (TMEM lanes)
constexpr int kUTile = kBM * 64 * 2;     // one 128 x 64 fp16 K-block unit = 16 KB

template <int KB, class Pol>
struct Cfg {
  static constexpr int BN = 128;                              // items per tile (= kBM: A and B units alike)
  // ring of K-block units: every unit the shared memory left next to the candidate buffers holds
  static constexpr int NST_FIT = (232448 - 2048 - Pol::kBufBytes) / kUTile;
  static constexpr int NST = NST_FIT < 10 ? NST_FIT : 10;
  static constexpr int ACC_COLS = BN;                         // TMEM columns per accumulator stage
  static constexpr int NACC = KB == 0 ? 4 : 3;
  static constexpr int A_TMEM = NACC * ACC_COLS;              // column of the A tile in TMEM (KB > 0)
  static constexpr int TMEM_COLS = 512;
  static_assert(KB == 0 || A_TMEM + 32 * KB <= TMEM_COLS, "tensor memory");
  static constexpr int THREADS = 192;
  static constexpr int RING = 0;
  static constexpr int CAND = RING + NST * kUTile;
  static constexpr int BAR = CAND + Pol::kBufBytes;
  static constexpr int TOTAL = BAR + 512 + 1024;    // barriers + control words, alignment slack
  static_assert(NST >= 6 && TOTAL <= 232448, "shared memory");
};

}  // namespace

// tmA / tmB: 64-column boxes; tmAt / tmBt: the last K block's tail box (tail columns, tail_cols(d)).
template <int KB, class Pol>
__global__ void __launch_bounds__(Cfg<KB, Pol>::THREADS, 1)
k_build_tcq(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAt,
            const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBt,
            const float* __restrict__ perr, const double* __restrict__ pnorm, const float* __restrict__ pscale,
            int64_t n, int64_t m, int kmax, int ksteps, int kb_rt, int tail, int dev, int32_t* __restrict__ cand,
            int32_t* __restrict__ ccount, int32_t* __restrict__ ovf_list, int* __restrict__ ovf_count,
            unsigned long long* __restrict__ tiles_done, int stale_every) {
  using namespace sm100;
  using C = Cfg<KB, Pol>;
  constexpr int NST = C::NST, NACC = C::NACC, BN = C::BN;
  constexpr bool kStreamA = KB == 0;
  const int kbn = kStreamA ? kb_rt : KB;          // K blocks per row
  // ring slots in use: NST (dev: RMIPS_NST=k limits it, for the feed-latency experiments)
  const int nst = ((dev >> 8) & 0xff) ? min(NST, (dev >> 8) & 0xff) : NST;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte aligned base, derived from smem_raw by pointer arithmetic so that the compiler
  // keeps the shared state space (LDS/STS rather than generic loads/stores)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sR = sbase + C::RING;
  const typename Pol::Buf sb = Pol::buf(smem + C::CAND, perr);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR);
  const uint32_t bar0 = smem_u32(bars);
  auto BAR = [&](int i) { return bar0 + 8u * i; };
  const int R_FULL = 0, R_EMPTY = NST, ACC_FULL = 2 * NST, ACC_EMPTY = 2 * NST + NACC;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NST + 2 * NACC);
  // early-termination control words (Cauchy-Schwarz, as in build_tc.cu): epilogue warps done
  // with a user tile (cumulative, 4 per tile), and the producer -> MMA -> epilogue end markers
  volatile int* done_cum = reinterpret_cast<volatile int*>(tmem_slot + 1);
  volatile int* stage_end = done_cum + 1;
  volatile int* acc_end = stage_end + NST;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_utiles = (int)((n + kBM - 1) / kBM);
  const int nit = (int)((m + BN - 1) / BN);
  const uint32_t tail_bytes = (uint32_t)(kBM * tail * 2);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmAt);
    tma_prefetch(&tmBt);
    for (int s = 0; s < NST; ++s) mbar_init(BAR(R_FULL + s), 1), mbar_init(BAR(R_EMPTY + s), 1);
    for (int a = 0; a < NACC; ++a) mbar_init(BAR(ACC_FULL + a), 1), mbar_init(BAR(ACC_EMPTY + a), 4);
    *done_cum = 0;
    for (int s = 0; s < NST; ++s) stage_end[s] = 0;
    for (int a = 0; a < NACC; ++a) acc_end[a] = 0;
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(smem_u32(tmem_slot), C::TMEM_COLS);
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
      // one K-block unit (rows r0.., K block kb) of map m / tail map mt into the next ring slot
      int nloads = 0;
      auto load_unit = [&](const CUtensorMap* mfull, const CUtensorMap* mtail, int kb, int r0) {
        const bool last = kb == kbn - 1;
        mbar_wait_sleep(BAR(R_EMPTY + stage), ph ^ 1);
        if ((dev & kDevNoFeed) && mfull == &tmB && nloads >= 2 * NST) {
          mbar_arrive(BAR(R_FULL + stage));  // dev: the MMA re-reads the stale slot (no L2 feed)
        } else {
          mbar_arrive_expect_tx(BAR(R_FULL + stage), last ? tail_bytes : (uint32_t)kUTile);
          tma_load_2d(sR + stage * kUTile, last ? mtail : mfull, kb * 64, r0, BAR(R_FULL + stage));
        }
        ++nloads;
        if (++stage == nst) stage = 0, ph ^= 1;
      };
      for (int ut = blockIdx.x; ut < num_utiles; ut += gridDim.x, ++t) {
        if (!kStreamA)
          for (int kb = 0; kb < kbn; ++kb) load_unit(&tmA, &tmAt, kb, ut * kBM);  // the user tile A
        for (int it = 0; it < nit; ++it) {
          mbar_wait_sleep(BAR(R_EMPTY + stage), ph ^ 1);
          if (*done_cum >= 4 * (t + 1)) {  // every epilogue warp is done with this user tile
            stage_end[stage] = t + 1;
            mbar_arrive(BAR(R_FULL + stage));  // release: the marker is visible to the MMA warp
            if (++stage == nst) stage = 0, ph ^= 1;
            break;
          }
          for (int kb = 0; kb < kbn; ++kb) {
            if (kStreamA) load_unit(&tmA, &tmAt, kb, ut * kBM);  // K block kb of the user tile ...
            load_unit(&tmB, &tmBt, kb, it * BN);                 // ... and of the item tile
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA warp
    // All lanes run the loop (warp-uniform state, descriptors in uniform registers); the elected
    // lane issues.  Descriptors: the unit's base plus a constant per K step (16 fp16 = 32 bytes =
    // 2 in the 16-byte address field); the tail unit has its own swizzle.
    constexpr uint32_t idesc = idesc_f16_f32(kBM, BN);
    unsigned long long tiles_issued = 0;  // (user tile, item tile) contractions issued
    int stage = 0, as = 0;
    uint32_t ph = 0, aph = 0;
    int t = 0;
    auto unit_desc = [&](int st_, int kb) {
      const uint32_t a = sR + st_ * kUTile;
      return kb == kbn - 1 ? sdesc_swz(a, 2 * tail) : sdesc_sw128(a);
    };
    auto next = [&]() {
      if (++stage == nst) stage = 0, ph ^= 1;
    };
    for (int ut = blockIdx.x; ut < num_utiles; ut += gridDim.x, ++t) {
      if (!kStreamA) {
        for (int kb = 0; kb < kbn; ++kb) {  // the user tile: into tensor memory, unit by unit
          mbar_wait_sleep(BAR(R_FULL + stage), ph);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t adesc = unit_desc(stage, kb);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              if (4 * kb + kk < ksteps)
                tmem_cp_128x256b(tmem + C::A_TMEM + 8 * (4 * kb + kk), adesc + (uint64_t)(2 * kk));
            mma_commit(BAR(R_EMPTY + stage));  // the unit is free once the copy has completed
          }
          __syncwarp();
          next();
        }
      }
      for (int it = 0; it < nit; ++it) {
        mbar_wait_sleep(BAR(ACC_EMPTY + as), aph ^ 1);
        mbar_wait_sleep(BAR(R_FULL + stage), ph);
        tc_fence_after();
        if (stage_end[stage] == t + 1) {  // the producer ended this user tile: forward the marker
          if (elect_one()) {
            mbar_arrive(BAR(R_EMPTY + stage));
            acc_end[as] = t + 1;
            mbar_arrive(BAR(ACC_FULL + as));
          }
          __syncwarp();
          next();
          if (++as == NACC) as = 0, aph ^= 1;
          break;
        }
        const uint32_t d = tmem + as * C::ACC_COLS;
        for (int kb = 0; kb < kbn; ++kb) {
          if (kb > 0) {  // (the first unit of the tile was awaited above)
            mbar_wait_sleep(BAR(R_FULL + stage), ph);
            tc_fence_after();
          }
          if (kStreamA) {
            // unit `stage` = K block kb of the user tile, the next unit = of the item tile
            const int sa = stage;
            next();
            mbar_wait_sleep(BAR(R_FULL + stage), ph);
            tc_fence_after();
            if (elect_one()) {
              const uint64_t adesc = unit_desc(sa, kb), bdesc = unit_desc(stage, kb);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                if (4 * kb + kk < ksteps)
                  mma_f16(d, adesc + (uint64_t)(2 * kk), bdesc + (uint64_t)(2 * kk), idesc, (kb | kk) != 0);
              mma_commit(BAR(R_EMPTY + sa));
              mma_commit(BAR(R_EMPTY + stage));
            }
          } else if (elect_one()) {
            const uint64_t bdesc = unit_desc(stage, kb);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // K steps of 16 (zero padding beyond d skipped)
              if (4 * kb + kk < ksteps)
                mma_f16_ts(d, tmem + C::A_TMEM + 8 * (4 * kb + kk), bdesc + (uint64_t)(2 * kk), idesc, (kb | kk) != 0);
            mma_commit(BAR(R_EMPTY + stage));
          }
          __syncwarp();
          next();
        }
        if (elect_one()) mma_commit(BAR(ACC_FULL + as));
        __syncwarp();
        ++tiles_issued;
        if (++as == NACC) as = 0, aph ^= 1;
      }
    }
    if (lane == 0) atomicAdd(tiles_done, tiles_issued);
  } else {
    // ------------------------------------------------ epilogue: one thread per user row
    // The 64-column halves of an item tile are software-pipelined: the TMEM load of the next half
    // (of this tile or the next one) is in flight while the current half is filtered.
    const int q = warp & 3;                   // TMEM lane quadrant of this warp
    const int rr = q * 32 + lane;             // row in the candidate buffer
    const int mi = (int)m;
    const float e0x2 = __fadd_ru(__ldg(perr), __ldg(perr));
    // |s~| <= |u^| |p^| + E with |u^| <= 1 + 2^-10, |p^| <= |p| 2^e (1 + 2^-11): every score is
    // in [-smax, smax] (generous margins: the quantiser of candq.cuh must never saturate)
    const float smax = __fadd_ru(__fmul_ru((float)(__ldg(pnorm) * (double)__ldg(pscale)), 1.02f), __fmul_ru(2.f, e0x2));
    const float pscl = __ldg(pscale);
    int as = 0;
    uint32_t aph = 0;
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    constexpr int kCsEvery = 4;   // Cauchy-Schwarz check period (item tiles)
    static_assert(kCsEvery * C::BN == (int)kPerrGroup, "candq.cuh drops on perr[j & ~(kPerrGroup - 1)]");
    uint32_t hA[64], hB[64];
    int t = 0;
    for (int ut = blockIdx.x; ut < num_utiles; ut += gridDim.x, ++t) {
      const int64_t row = (int64_t)ut * kBM + q * 32 + lane;
      typename Pol::Row me = Pol::init(row < n, smax);  // dead rows (user >= n): theta = +inf, never pass
      int lastc = 0;  // the row's entry count at its last checkpoint refresh
      // error bound of every chunk of a group of kCsEvery item tiles: perr of the group's first item
      // (perr is non-increasing along the norm-sorted items, so it bounds every later item's);
      // the next group's is prefetched a whole group ahead
      float Eg = __ldg(perr), EgN = (kCsEvery * BN < mi) ? __ldg(perr + kCsEvery * BN) : 0.f;
      double pnr = nit > kCsEvery ? __ldg(pnorm + kCsEvery * BN) : 0.0;  // raw norm, scaled at the check
      mbar_wait(BAR(ACC_FULL + as), aph);
      tc_fence_after();
      tmem_ld64(tq + as * C::ACC_COLS, hA);
      tmem_ld_wait64(hA);
      int it = 0;
      bool done = false;  // warp-uniform: this warp's rows cannot gain any more
      if (dev & (kDevEpiSkip | kDevEpiLoad)) {  // dev: release every accumulator stage (MMA + feed alone)
        uint32_t sink = 0;
        for (; it < nit; ++it) {
          if (dev & kDevEpiLoad) {
            const uint32_t tcur = tq + as * C::ACC_COLS;
            tmem_ld64(tcur, hA);
            tmem_ld64(tcur + 64, hB);
            tmem_ld_wait64(hA);
            tmem_ld_wait64(hB);
            sink ^= hA[0] ^ hB[63];  // (constant indices: the arrays stay in registers)
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(BAR(ACC_EMPTY + as));
          if (++as == NACC) as = 0, aph ^= 1;
          if (it + 1 < nit) {
            mbar_wait(BAR(ACC_FULL + as), aph);
            tc_fence_after();
          }
        }
        if (sink == 0x12345678u) ccount[0] = 0;  // keeps the loads
      }
      for (; it < nit; ++it) {
        const int base0 = it * BN;
        const float E[4] = {Eg, Eg, Eg, Eg};
        const uint32_t tcur = tq + as * C::ACC_COLS;
        tmem_ld64(tcur + 64, hB);                 // second half of this tile
        uint32_t bits = epiq_fast(hA, E[0], E[1], me.theta);
        const bool more = it + 1 < nit;
        const int as_next = as + 1 == NACC ? 0 : as + 1;
        const uint32_t aph_next = as + 1 == NACC ? aph ^ 1 : aph;
        // the stage is released as soon as this tile is done, before the next tile's accumulator is
        // awaited (build_tc.cu: the MMA may then run NACC tiles ahead)
        tmem_ld_wait64(hB);
        bits |= epiq_fast(hB, E[2], E[3], me.theta) << 2;
        if (bits) me = epiq_slow<Pol>(bits, tcur, base0, mi, make_float4(E[0], E[1], E[2], E[3]), me, sb, rr, e0x2, kmax);
        tc_fence_before();                        // this stage is no longer read: release it
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(ACC_EMPTY + as));
        if (more) {                               // first half of the next tile
          mbar_wait(BAR(ACC_FULL + as_next), aph_next);
          tc_fence_after();
          tmem_ld64(tq + as_next * C::ACC_COLS, hA);
          tmem_ld_wait64(hA);
        }
        as = as_next;
        aph = aph_next;
        if ((it + 1) % kCsEvery == 0 && more) {
          // every item from tile it + 1 on has scaled true score <= pnn (1 + 2^-16)
          const uint32_t mk = __reduce_min_sync(0xffffffffu, f2key(me.theta));
          const float pnn = __double2float_ru(pnr * (double)pscl);
          if (__fmul_ru(pnn, 1.0000153f) < key2f(mk)) {
            done = true;
            break;
          }
          // stale-theta checkpoint refresh, as build_tc2cta.cu: rows that appended since their last refresh
          if (stale_every > 0 && (it + 1) % stale_every == 0 && __fmul_ru(pnn, 1.0000153f) < 1.5f * key2f(mk) &&
              __any_sync(0xffffffffu, me.cnt != lastc)) {  // (only near the exit: within 1.5x of the stale one)
            Pol::refresh_theta(me, sb, rr, e0x2, kmax);
            lastc = me.cnt;
            if (__fmul_ru(pnn, 1.0000153f) < key2f(__reduce_min_sync(0xffffffffu, f2key(me.theta)))) {
              done = true;
              break;
            }
          }
          Eg = EgN;
          if (base0 + (kCsEvery + 1) * BN < mi) {
            pnr = __ldg(pnorm + base0 + (kCsEvery + 1) * BN);
            EgN = __ldg(perr + base0 + (kCsEvery + 1) * BN);
          }
        }
      }
      if (lane == 0) atomicAdd(const_cast<int*>(done_cum), 1);  // one event per warp and user tile
      if (done) {                                 // drain: release the remaining stages unread
        for (++it; it < nit; ++it) {              // stage `as` (tile it) is already full
          const bool end = acc_end[as] == t + 1;
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(BAR(ACC_EMPTY + as));
          if (++as == NACC) as = 0, aph ^= 1;
          if (end || it + 1 == nit) break;
          mbar_wait(BAR(ACC_FULL + as), aph);
          tc_fence_after();
        }
      }
      if (dev & (kDevEpiSkip | kDevEpiLoad)) {
        if (row < n) ccount[row] = 0;  // dev: empty lists, no fallback
      } else {
        Pol::finish(me, sb, rr, e0x2, kmax, m, row, n, cand, ccount, ovf_list, ovf_count);
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
}

// ------------------------------------------------------------------------------ host side
static int sm_count_q() {
  static int c = 0;
  if (!c) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev);
  }
  return c;
}

template <int KB, class Pol>
static cudaError_t launch_tcq(const BuildCtx& c, cudaStream_t st) {
  using C = Cfg<KB, Pol>;
  rmips_index_s* x = c.idx;
  const int tail = tail_cols(x->d);
  CUtensorMap ta, tat, tb, tbt;
  if (!make_tmap_f16_box(&ta, x->U16, (uint64_t)x->n, (uint64_t)x->ldh, kBM) ||
      !make_tmap_f16_box(&tat, x->U16, (uint64_t)x->n, (uint64_t)x->ldh, kBM, tail) ||
      !make_tmap_f16_box(&tb, x->P16, (uint64_t)c.mb, (uint64_t)x->ldh, C::BN) ||
      !make_tmap_f16_box(&tbt, x->P16, (uint64_t)c.mb, (uint64_t)x->ldh, C::BN, tail))
    return cudaErrorNotSupported;
  cudaError_t e = set_smem_attr((const void*)k_build_tcq<KB, Pol>, C::TOTAL);
  if (e != cudaSuccess) return e;
  const int tiles = (int)((x->n + kBM - 1) / kBM);
  const int grid = tiles < sm_count_q() ? tiles : sm_count_q();
  const int ksteps = (x->d + 15) / 16;  // K steps of 16 that touch real (non-padding) columns
  int dev = 0;
#ifdef RMIPS_DEV
  dev = (getenv("RMIPS_NOFEED") ? kDevNoFeed : 0) | (getenv("RMIPS_EPI_SKIP") ? kDevEpiSkip : 0) |
        (getenv("RMIPS_EPI_LOAD") ? kDevEpiLoad : 0);
  if (const char* v = getenv("RMIPS_NST")) dev |= (atoi(v) & 0xff) << 8;
#endif
  x->build_kernel = KB == 0 ? 3 : 2;
  x->cand_slots = Pol::kSlots;
  int stale_every = 16;  // stale-theta checkpoint refresh period (item tiles), as build_tc2cta.cu
#ifdef RMIPS_DEV
  if (const char* e = getenv("RMIPS_STALE_EVERY")) stale_every = atoi(e);  // 0: off
#endif
  k_build_tcq<KB, Pol><<<grid, C::THREADS, C::TOTAL, st>>>(ta, tat, tb, tbt, x->perr, x->pnorm, c.scale_dev, x->n,
                                                          c.mb, x->kmax, ksteps, x->dpad / 64, tail, dev, c.cand,
                                                          c.ccount, c.ovf_list, c.ovf_count, c.tiles_done, stale_every);
  count_launch();
  return cudaGetLastError();
}

template <class Pol>
static cudaError_t launch_tcq_kb(const BuildCtx& c, cudaStream_t st) {
  switch (c.idx->dpad) {
    case 64: return launch_tcq<1, Pol>(c, st);
    case 128: return launch_tcq<2, Pol>(c, st);
    case 192: return launch_tcq<3, Pol>(c, st);
    case 256: return launch_tcq<4, Pol>(c, st);
    default: return launch_tcq<0, Pol>(c, st);  // d_pad > 256: A streamed with B
  }
}

// 256 slots also for d > 240: there the scores crowd near the k_max-th largest, and more than 96 entries
// often fall inside the error band a refresh must keep, which sent rows to the exact fallback
// (configs[4] recipe, 148,000 users x 1 M items, 128 slots: d = 256 10 rows (+210 ms), d = 513 1,115
// rows (8.8 s); d = 240: none).  These shapes take build_tcq (the CTA-pair kernel has no room for them).
// m in (2^20, 2^21]: 256 slots of 21-bit positions (QPolT<256, 21>) whatever k_max and d -- the 8-byte
// entries (128 slots) overflowed rows there (m = 1.3 M: k_max = 80 at d = 256, or d >= 513).
int build_cand_stride(int kmax, int64_t mb, int build_flags, int d) {
  if (build_flags & RMIPS_BUILD_SIMT) return kCand;
  if (mb <= QPolT<256>::kMaxItems) return (kmax > kQ128MaxKmax || d > 240) ? 256 : kCand;
  return mb <= QPolT<256, 21>::kMaxItems ? 256 : kCand;
}

// Any d_pad: the candidate policy by (m, k_max, d): 4-byte entries while positions fit 20 bits (256
// slots above k_max = 80 or d = 240) or 21 bits (256 slots, an 11-bit bound), else 8-byte entries (128
// slots: crowded rows then overflow to the exact fallback, R11).
cudaError_t build_tcq(const BuildCtx& c, cudaStream_t st) {
  if (c.cstride == 256 && c.mb > QPolT<256>::kMaxItems) return launch_tcq_kb<QPolT<256, 21>>(c, st);
  if (c.cstride == 256) return launch_tcq_kb<QPolT<256>>(c, st);
  if (c.mb <= QPolT<128>::kMaxItems) return launch_tcq_kb<QPolT<128>>(c, st);
  return launch_tcq_kb<FPol>(c, st);
}

}  // namespace rmips
