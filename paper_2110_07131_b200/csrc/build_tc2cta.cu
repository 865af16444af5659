// build_tc2cta.cu -- B4 over CTA PAIRS: the |Q| x |P| x d contraction of Alg. 1 lines 7-9 (
// over ALL of P per BASELINE north star) on tcgen05.mma.cta_group::2 (M = 256 users of two SMs,
// N = 128 items), fused with the per-row top-k_max candidate epilogue (candpol.cuh / epiq.cuh).
//
// Why pairs: with one SM per 128-user tile (build_tcq.cu) every byte of an item tile is written into
// shared memory by TMA and read once by the MMA, 2 x 64 B/clk at the tensor rate -- the SM's whole
// shared-memory bandwidth.  In a pair each SM holds and feeds HALF of every item tile (64 of its 128
// rows) and the 2-SM MMA reads both halves, so each SM's shared-memory traffic per flop halves.
//
// Cluster of 2 CTAs (rank 0 = leader L, rank 1 = follower F), persistent over user-tile PAIRS: the pair
// processes user tiles 2 tp + rank against the same item tiles.  Per CTA:
//   warp 0   TMA producer: the CTA's user tile A (KB K-block units of 128 x 64, last one trimmed to
//            tail_cols(d)) into its A buffer, and its half of every item tile (KB units of 64 x 64) into
//            a ring of 8 KB slots; every load completes its bytes on the LEADER's barriers (.cta_group::2)
//   warp 1   leader only: tcgen05.cp.cta_group::2 of the A tiles into both TMEMs, then one
//            tcgen05.mma.cta_group::2 chain per item tile (A from TMEM, B halves from both shared
//            memories), tcgen05.commit multicast to both CTAs' barriers
//   warps 2-5 epilogue of the CTA's own 128 rows, exactly as build_tcq.cu
// Early termination (Cauchy-Schwarz) is decided per PAIR: all 8 epilogue warps report to the leader's
// done counter; the leader's producer decides for every group of kGroup item tiles, one group ahead, and
// tells the follower's producer (DEC barriers), so both halves of a tile are either loaded or both
// skipped; the leader ends the user-tile pair with a marker.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cub/cub.cuh>

#include "candpol.cuh"
#include "common.cuh"
#include "epiq.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace rmips {
namespace {

constexpr int kBM = 128;                 // users per CTA (TMEM lanes)
constexpr int kAUnit = 128 * 64 * 2;     // one K block of a user tile: 16 KB
constexpr int kBUnit = 64 * 64 * 2;      // one K block of this CTA's half item tile: 8 KB
constexpr int kGroup = 4;                // item tiles per end-of-pair decision (the C-S check period)

// The ring holds whole item tiles: a slot is this CTA's KB K-block units of one item tile (one full
// barrier, one 13-MMA chain, one commit per tile: the MMA warp's per-tile overhead does not scale with
// the K blocks).
template <int KB, class Pol>
struct Cfg2 {
  static constexpr int BN = 128;                 // items per pair MMA tile (64 rows in each CTA)
  static constexpr int TS = KB * kBUnit;         // bytes of a tile slot
  static constexpr int RING = KB * kAUnit;       // after the A buffer
  static constexpr int NSB_FIT = (232448 - 3072 - RING - Pol::kBufBytes) / TS;
  static constexpr int NSB = NSB_FIT < 8 ? NSB_FIT : 8;  // tile slots
  static constexpr int NDEC = 8;                 // end-of-pair decision barriers (see the producer)
  static constexpr int CAND = RING + NSB * TS;
  static constexpr int BAR = CAND + Pol::kBufBytes;
  static constexpr int NACC = 3, ACC_COLS = 128, A_TMEM = NACC * ACC_COLS, TMEM_COLS = 512;
  static constexpr int THREADS = 192;
  // barriers R_FULL[NSB] R_EMPTY[NSB] DEC[NDEC] ACC_FULL[NACC] ACC_EMPTY[NACC] A_FULL A_EMPTY, then words
  static constexpr int NBARS = 2 * NSB + NDEC + 2 * NACC + 2;
  static constexpr int TOTAL = BAR + NBARS * 8 + (4 + NSB + NDEC + NACC) * 4 + 1024;
  static_assert(KB >= 1 && KB <= 4 && A_TMEM + 32 * KB <= TMEM_COLS, "tensor memory");
  static_assert(NSB >= 2 && TOTAL <= 232448, "shared memory");
};

}  // namespace

template <int KB, class Pol>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg2<KB, Pol>::THREADS, 1)
k_build_tc2cta(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmAt,
               const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmBt,
               const float* __restrict__ perr, const double* __restrict__ pnorm, const float* __restrict__ pscale,
               int64_t n, int64_t m, int kmax, int ksteps, int tail, int32_t* __restrict__ cand,
               int32_t* __restrict__ ccount, int32_t* __restrict__ ovf_list, int* __restrict__ ovf_count,
               unsigned long long* __restrict__ tiles_done, int stale_every, int seed, int it0, int nit_cap,
               float* __restrict__ theta_out, uint32_t* __restrict__ st_ent, uint4* __restrict__ st_meta,  // (entries: Pol's format)
               const int32_t* __restrict__ row_map) {
  using namespace sm100;
  using C = Cfg2<KB, Pol>;
  constexpr int NSB = C::NSB, NDEC = C::NDEC, NACC = C::NACC, BN = C::BN, TS = C::TS;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sA = sbase, sR = sbase + C::RING;
  const typename Pol::Buf sb = Pol::buf(smem + C::CAND, perr);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::BAR);
  const uint32_t bar0 = smem_u32(bars);
  auto BAR = [&](int i) { return bar0 + 8u * i; };
  const int R_FULL = 0, R_EMPTY = NSB, DEC = 2 * NSB, ACC_FULL = 2 * NSB + NDEC, ACC_EMPTY = ACC_FULL + NACC,
            A_FULL = ACC_EMPTY + NACC, A_EMPTY = A_FULL + 1;
  uint32_t* words = reinterpret_cast<uint32_t*>(bars + C::NBARS);
  uint32_t* tmem_slot = words;
  volatile uint32_t* done_cum = words + 1;   // leader: epilogue warps of the pair done with a tile pair (8 each)
  volatile uint32_t* stage_end = words + 2;  // [NSB] leader: producer -> MMA end marker (t + 1)
  volatile uint32_t* acc_end = stage_end + NSB;  // [NACC] both: MMA -> epilogue end marker
  volatile uint32_t* dec = acc_end + NACC;   // [NDEC] follower: the leader's decision for a group of tiles
  const uint32_t w_done = smem_u32(words + 1), w_acc_end = smem_u32(words + 2 + NSB),
                 w_dec = smem_u32(words + 2 + NSB + NACC);

  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_utiles = (int)((n + kBM - 1) / kBM);
  const int num_tp = (num_utiles + 1) / 2;
  const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
  // head pass (nit_cap > 0): only the first nit_cap item tiles; regrouped pass: item tiles it0 .. (see
  // the host side; it0 is a multiple of kGroup)
  const int nit = nit_cap > 0 && (int64_t)nit_cap * BN < m ? nit_cap : (int)((m + BN - 1) / BN);
  const uint32_t a_tail_bytes = (uint32_t)(kBM * tail * 2), b_tail_bytes = (uint32_t)(64 * tail * 2);
  const uint32_t a_bytes = (uint32_t)((KB - 1) * kAUnit) + a_tail_bytes;
  const uint32_t b_bytes = (uint32_t)((KB - 1) * kBUnit) + b_tail_bytes;  // this CTA's half of an item tile

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmAt);
    tma_prefetch(&tmBt);
    for (int s = 0; s < NSB; ++s) mbar_init(BAR(R_FULL + s), 1), mbar_init(BAR(R_EMPTY + s), 1);
    for (int s = 0; s < NDEC; ++s) mbar_init(BAR(DEC + s), 1);
    for (int a = 0; a < NACC; ++a) mbar_init(BAR(ACC_FULL + a), 1), mbar_init(BAR(ACC_EMPTY + a), 8);
    mbar_init(BAR(A_FULL), 1);
    mbar_init(BAR(A_EMPTY), 1);
    *done_cum = 0;
    for (int s = 0; s < NSB; ++s) stage_end[s] = 0;
    for (int s = 0; s < NDEC; ++s) dec[s] = 0;
    for (int a = 0; a < NACC; ++a) acc_end[a] = 0;
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc_cg2(smem_u32(tmem_slot), C::TMEM_COLS);
    tmem_relinquish_cg2();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // both CTAs' barriers exist before any remote arrive or TMA completion
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto L = [&](uint32_t a) { return mapa_shared(a, 0); };  // the leader's copy of a shared address
  auto F = [&](uint32_t a) { return mapa_shared(a, 1); };  // the follower's

  if (warp == 0) {
    // ------------------------------------------------ TMA producer (both CTAs)
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0, decph = 0;  // ring phase; per-slot DEC phase bits
      int t = 0;
      auto next = [&]() {
        if (++stage == NSB) stage = 0, ph ^= 1;
      };
      for (int tp = pair; tp < num_tp; tp += npairs, ++t) {
        const int ut = 2 * tp + (int)rank;  // (the follower of an odd last pair reads rows >= n: zero fill)
        mbar_wait_sleep(BAR(A_EMPTY), (t & 1) ^ 1);
        if (leader) mbar_arrive_expect_tx(BAR(A_FULL), 2 * a_bytes);
        for (int kb = 0; kb < KB; ++kb)
          tma_load_2d_cg2(sA + kb * kAUnit, kb == KB - 1 ? &tmAt : &tmA, kb * 64, ut * kBM, L(BAR(A_FULL)));
        // Item tiles go in groups of kGroup.  At the start of group g the leader decides whether group
        // g + 1 is issued (every epilogue warp of the pair done -> the pair ends there) and sends that
        // decision to the follower a whole group AHEAD, so the follower's wait for it is off the feed's
        // critical path; group 0 is always issued.  (At most two groups of tiles follow the last
        // report; the epilogue drains them unread.)
        // (seed pass: item tiles 0 .. seed-1 are issued first, then the pass's tiles it0 ..; groups are
        // counted over that whole sequence)
        bool end_next = false;
        const int ntot = seed + nit - it0;
        for (int jj = 0; jj < ntot; ++jj) {
          const int it = jj < seed ? jj : it0 + jj - seed;
          if (jj % kGroup == 0) {
            const int g = jj / kGroup;
            bool end = false;
            if (leader) {
              end = end_next;
              if (end) {
                mbar_wait_sleep(BAR(R_EMPTY + stage), ph ^ 1);
                stage_end[stage] = t + 1;
                mbar_arrive(BAR(R_FULL + stage));  // the marker (no bytes) for the MMA warp
              } else if ((g + 1) * kGroup < ntot) {
                end_next = *done_cum >= 8u * (uint32_t)(t + 1);  // every epilogue warp of the pair is done
                st_cluster_u32(F(w_dec + 4 * ((g + 1) & 7)), end_next ? 1u : 0u);
                mbar_arrive_cluster(F(BAR(DEC + ((g + 1) & 7))));
              }
            } else if (g > 0) {
              // (NDEC = 8 decision barriers: the leader runs at most NSB <= 8 tiles, i.e. fewer than 8
              // groups, ahead of the follower, so a barrier never advances twice before its wait)
              mbar_wait_cluster(BAR(DEC + (g & 7)), (decph >> (g & 7)) & 1u);
              decph ^= 1u << (g & 7);
              end = dec[g & 7] != 0;
            }
            if (end) {
              next();
              break;
            }
          }
          mbar_wait_sleep(BAR(R_EMPTY + stage), ph ^ 1);
          if (leader) mbar_arrive_expect_tx(BAR(R_FULL + stage), 2 * b_bytes);
          for (int kb = 0; kb < KB; ++kb)
            tma_load_2d_cg2(sR + stage * TS + kb * kBUnit, kb == KB - 1 ? &tmBt : &tmB, kb * 64,
                            it * BN + 64 * (int)rank, L(BAR(R_FULL + stage)));
          next();
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA warp (leader only)
    if (leader) {
      constexpr uint32_t idesc = idesc_f16_f32(2 * kBM, BN);
      unsigned long long tiles_issued = 0;
      int stage = 0, as = 0;
      uint32_t ph = 0, aph = 0;
      int t = 0;
      auto next = [&]() {
        if (++stage == NSB) stage = 0, ph ^= 1;
      };
      auto bdesc_of = [&](int kb) {
        const uint32_t a = sR + stage * TS + kb * kBUnit;
        return kb == KB - 1 ? sdesc_swz(a, 2 * tail) : sdesc_sw128(a);
      };
      for (int tp = pair; tp < num_tp; tp += npairs, ++t) {
        mbar_wait_sleep(BAR(A_FULL), t & 1);
        tc_fence_after();
        if (elect_one()) {
#pragma unroll
          for (int kb = 0; kb < KB; ++kb) {
            const uint32_t a = sA + kb * kAUnit;
            const uint64_t adesc = kb == KB - 1 ? sdesc_swz(a, 2 * tail) : sdesc_sw128(a);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              if (4 * kb + kk < ksteps)
                tmem_cp_128x256b_cg2(tmem + C::A_TMEM + 8 * (4 * kb + kk), adesc + (uint64_t)(2 * kk));
          }
          mma_commit_cg2(BAR(A_EMPTY), 3);  // both A buffers are free once the copies completed
        }
        __syncwarp();
        for (int jj = 0; jj < seed + nit - it0; ++jj) {
          mbar_wait_sleep(BAR(ACC_EMPTY + as), aph ^ 1);
          mbar_wait_sleep(BAR(R_FULL + stage), ph);
          tc_fence_after();
          if (stage_end[stage] == (uint32_t)(t + 1)) {  // the producer ended this tile pair: forward
            if (elect_one()) {
              mbar_arrive(BAR(R_EMPTY + stage));
              mbar_arrive_cluster(F(BAR(R_EMPTY + stage)));
              acc_end[as] = t + 1;
              st_cluster_u32(F(w_acc_end + 4 * as), (uint32_t)(t + 1));
              mbar_arrive(BAR(ACC_FULL + as));
              mbar_arrive_cluster(F(BAR(ACC_FULL + as)));
            }
            __syncwarp();
            next();
            if (++as == NACC) as = 0, aph ^= 1;
            break;
          }
          const uint32_t d = tmem + as * C::ACC_COLS;
          if (elect_one()) {
#pragma unroll
            for (int kb = 0; kb < KB; ++kb) {
              const uint64_t bdesc = bdesc_of(kb);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                if (4 * kb + kk < ksteps)
                  mma_f16_ts_cg2(d, tmem + C::A_TMEM + 8 * (4 * kb + kk), bdesc + (uint64_t)(2 * kk), idesc,
                                 (kb | kk) != 0);
            }
            mma_commit_cg2(BAR(R_EMPTY + stage), 3);
          }
          __syncwarp();
          next();
          if (elect_one()) mma_commit_cg2(BAR(ACC_FULL + as), 3);
          __syncwarp();
          tiles_issued += jj >= seed ? 2 : 0;  // two 128 x 128 (user tile, item tile) contractions (the seed
                                               // pass repeats tiles: not counted)
          if (++as == NACC) as = 0, aph ^= 1;
        }
      }
      if (lane == 0) atomicAdd(tiles_done, tiles_issued);
    }
  } else {
    // ------------------------------------------------ epilogue: one thread per user row (both CTAs)
    const int q = warp & 3;
    const int rr = q * 32 + lane;
    const int mi = (int)m;
    const float e0x2 = __fadd_ru(__ldg(perr), __ldg(perr));
    const float smax = __fadd_ru(__fmul_ru((float)(__ldg(pnorm) * (double)__ldg(pscale)), 1.02f), __fmul_ru(2.f, e0x2));
    const float pscl = __ldg(pscale);
    int as = 0;
    uint32_t aph = 0;
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    constexpr int kCsEvery = 4;
    static_assert(kCsEvery * C::BN == (int)kPerrGroup, "candq.cuh drops on perr[j & ~(kPerrGroup - 1)]");
    uint32_t hA[64], hB[64];
    int t = 0;
    auto release = [&](int a) {  // this warp is done reading accumulator stage a (the leader's barrier)
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(BAR(ACC_EMPTY + a));
        else mbar_arrive_remote(L(BAR(ACC_EMPTY + a)));
      }
    };
    for (int tp = pair; tp < num_tp; tp += npairs, ++t) {
      const int ut = 2 * tp + (int)rank;
      const int64_t row = (int64_t)ut * kBM + rr;
      typename Pol::Row me = Pol::init(row < n, smax);
      // regrouped pass: the row continues from its head-pass state (theta, entries), saved at the row's
      // index place
      const int64_t orow = row_map && row < n ? (int64_t)__ldg(row_map + row) : row;
      if (row_map && row < n) Pol::load(me, sb, rr, st_ent, st_meta, orow);
      int lastc = me.cnt;  // the row's entry count at its last checkpoint refresh (below)
      const int b0 = it0 * BN;
      float Eg = __ldg(perr + b0), EgN = (b0 + kCsEvery * BN < mi) ? __ldg(perr + b0 + kCsEvery * BN) : 0.f;
      double pnr = nit > it0 + kCsEvery ? __ldg(pnorm + b0 + kCsEvery * BN) : 0.0;
      if (seed > 0) {
        // Seed pass over item tiles 0 .. seed-1 (contracted again below): the maxima of the 16 groups of 8
        // items of each tile, minus the tile's error bound (rounded down), are lower bounds of distinct items'
        // true scores, so the k_max-th largest of them is a valid starting theta (Pol::seed_theta).  They sit in the
        // row's (still empty) candidate slots, 16 per tile.
        float vmx = -__int_as_float(0x7f800000);
        for (int j = 0; j < seed; ++j) {
          mbar_wait(BAR(ACC_FULL + as), aph);
          tc_fence_after();
          tmem_ld64(tq + as * C::ACC_COLS, hA);
          tmem_ld64(tq + as * C::ACC_COLS + 64, hB);
          const float Ej = __ldg(perr + j * BN);  // bounds every item of tile j (perr is non-increasing)
          tmem_ld_wait64(hA);
          tmem_ld_wait64(hB);
          release(as);
          if (++as == NACC) as = 0, aph ^= 1;
#pragma unroll
          for (int g = 0; g < 16; ++g) {
            const uint32_t* h = g < 8 ? hA + 8 * g : hB + 8 * (g - 8);
            const auto f = [](uint32_t u) { return __uint_as_float(u); };
            const float gm = fmaxf(fmaxf(fmaxf(f(h[0]), f(h[1])), fmaxf(f(h[2]), f(h[3]))),
                                   fmaxf(fmaxf(f(h[4]), f(h[5])), fmaxf(f(h[6]), f(h[7]))));
            const float lo = __fsub_rd(gm, Ej);
            Pol::seed_store(sb, rr, 16 * j + g, lo);
            vmx = fmaxf(vmx, lo);
          }
        }
        me.theta = fmaxf(me.theta, Pol::seed_theta(sb, rr, 16 * seed, vmx, kmax));  // dead rows keep +inf
      }
      mbar_wait(BAR(ACC_FULL + as), aph);
      tc_fence_after();
      tmem_ld64(tq + as * C::ACC_COLS, hA);
      tmem_ld_wait64(hA);
      int it = it0;
      bool done = false;
      for (; it < nit; ++it) {
        const int base0 = it * BN;
        const float E[4] = {Eg, Eg, Eg, Eg};
        const uint32_t tcur = tq + as * C::ACC_COLS;
        tmem_ld64(tcur + 64, hB);
        uint32_t bits = epiq_fast(hA, E[0], E[1], me.theta);
        const bool more = it + 1 < nit;
        const int as_next = as + 1 == NACC ? 0 : as + 1;
        const uint32_t aph_next = as + 1 == NACC ? aph ^ 1 : aph;
        tmem_ld_wait64(hB);
        bits |= epiq_fast(hB, E[2], E[3], me.theta) << 2;
        if (bits) me = epiq_slow<Pol>(bits, tcur, base0, mi, make_float4(E[0], E[1], E[2], E[3]), me, sb, rr, e0x2, kmax);
        release(as);
        if (more) {
          mbar_wait(BAR(ACC_FULL + as_next), aph_next);
          tc_fence_after();
          tmem_ld64(tq + as_next * C::ACC_COLS, hA);
          tmem_ld_wait64(hA);
        }
        as = as_next;
        aph = aph_next;
        if ((it + 1) % kCsEvery == 0 && more) {
          uint32_t mk = __reduce_min_sync(0xffffffffu, f2key(me.theta));
          const float pnn = __double2float_ru(pnr * (double)pscl);
          if (__fmul_ru(pnn, 1.0000153f) < key2f(mk)) {
            done = true;
            break;
          }
          // Late in the scan appends are rare, so a row's buffer seldom reaches the refresh mark and its
          // theta (last set at a refresh) lags the k_max-th largest lower bound it already holds, which
          // delays this exit: every stale_every tiles the warp refreshes rows that appended since their
          // last refresh (theta stays a valid lower bound: the same refresh) and tests the exit again.
          // (An always-current theta exits where the final thresholds do: 2,330 of 7,813 item tiles per
          // user tile of configs[4] against 2,577 with the refresh mark alone.)
          if (stale_every > 0 && (it + 1) % stale_every == 0 && __fmul_ru(pnn, 1.0000153f) < 1.5f * key2f(mk) &&
              __any_sync(0xffffffffu, me.cnt != lastc)) {  // (only near the exit: within 1.5x of the stale one)
            Pol::refresh_theta(me, sb, rr, e0x2, kmax);
            lastc = me.cnt;
            mk = __reduce_min_sync(0xffffffffu, f2key(me.theta));
            if (__fmul_ru(pnn, 1.0000153f) < key2f(mk)) {
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
      if (lane == 0) {  // one event per warp and tile pair, on the leader's counter
        if (leader) atomicAdd(const_cast<uint32_t*>(done_cum), 1u);
        else red_add_cluster_u32(L(w_done), 1u);
      }
      // a warp that is not done never meets an end marker: the leader ends a tile pair only after all 8
      // epilogue warps (this one included) reported
      if (done) {  // drain: release the remaining stages unread up to the end marker
        for (++it; it < nit; ++it) {
          mbar_wait_cluster(BAR(ACC_FULL + as), aph);  // (complete: acquires the leader's marker write)
          const bool end = acc_end[as] == (uint32_t)(t + 1);
          release(as);
          if (++as == NACC) as = 0, aph ^= 1;
          if (end || it + 1 == nit) break;
          mbar_wait(BAR(ACC_FULL + as), aph);
          tc_fence_after();
        }
      }
      if (theta_out) {  // head pass: compact, save the row's state, and its theta as the regrouping key
        Pol::compact(me, sb, rr, e0x2, kmax);
        if (row < n) {
          Pol::save(me, sb, rr, st_ent, st_meta, row);
          theta_out[row] = me.ovf ? -__int_as_float(0x7f800000) : me.theta;
        }
      } else {  // lists go to the row's place in the index order (row_map: regrouped pass)
        Pol::finish(me, sb, rr, e0x2, kmax, m, orow, n, cand, ccount, ovf_list, ovf_count);
      }
      __syncwarp();
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no remote barrier / shared-memory access of the peer is outstanding
  if (warp == 1) tmem_dealloc_cg2(tmem, C::TMEM_COLS);
}

// ------------------------------------------------------------------------------ host side
// Regrouping (two passes).  A tile pair ends at the Cauchy-Schwarz exit of its LAST row, i.e. at the
// largest exit point over 256 users, and norm-sorted users have unrelated exit points (the exit of row u
// is where ||p|| 2^e drops below theta_u ~ tau_kmax(u) / ||u||, a function of u's direction).  So:
//   head pass   the first `head` item tiles of every user tile; each row is compacted and its state
//               (theta, entries) saved at its index place, its theta (a valid lower bound of tau_kmax)
//               written as the regrouping key;
//   sort        rows by that theta, descending (CUB radix sort of n float keys), and gather a copy of
//               U16 in that order;
//   main pass   item tiles head .. over the regrouped rows, each row continuing from its saved state,
//               the lists written to the rows' index places (row_map).
// Offline (configs[4] recipe, 4,096 users, exact taus): random 256-row groups exit at 2,318 item tiles
// on average, groups sorted by the theta of the first 32 item tiles at 2,076 (by the exact exit: 2,058).
// The head items are paid once (the dense phase, where theta climbs from -inf, costs ~10x a steady-state
// tile: ncu, configs[4], 16 head tiles = 8.3 ms of the build).
__global__ void k_iota32(int32_t* __restrict__ v, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}

// out row i = in row perm[i]; rows of ldh halves (ldh a multiple of 16: 32-byte rows), 16-byte copies
__global__ void k_gather_rows16(const uint4* __restrict__ in, const int32_t* __restrict__ perm, int64_t n,
                                int vec_per_row, uint4* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t r = i / vec_per_row;
  if (r >= n) return;
  const int v = (int)(i - r * vec_per_row);
  out[i] = __ldg(in + (int64_t)__ldg(perm + r) * vec_per_row + v);
}

// Scratch of a regrouped build (one allocation, freed stream-ordered by regroup_free).
cudaError_t regroup_alloc(Regroup& g, int64_t n, int ldh, int slots, cudaStream_t st) {
  g.cub_bytes = 0;
  cub::DeviceRadixSort::SortPairsDescending(nullptr, g.cub_bytes, (const float*)nullptr, (float*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, (int)n);
  auto up = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const size_t o_th = 0, o_ths = o_th + up(n * 4), o_io = o_ths + up(n * 4), o_pm = o_io + up(n * 4),
               o_cub = o_pm + up(n * 4), o_u = o_cub + up(g.cub_bytes), o_me = o_u + up((size_t)n * ldh * 2),
               o_en = o_me + up((size_t)n * 16), total = o_en + up((size_t)n * slots * 4);
  const cudaError_t e = cudaMallocAsync(&g.buf, total, st);
  if (e != cudaSuccess) return e;
  char* B = static_cast<char*>(g.buf);
  g.th = reinterpret_cast<float*>(B + o_th);
  g.ths = reinterpret_cast<float*>(B + o_ths);
  g.io = reinterpret_cast<int32_t*>(B + o_io);
  g.pm = reinterpret_cast<int32_t*>(B + o_pm);
  g.cub = B + o_cub;
  g.U16b = reinterpret_cast<__half*>(B + o_u);
  g.meta = reinterpret_cast<uint4*>(B + o_me);
  g.ent = reinterpret_cast<uint32_t*>(B + o_en);
  return cudaSuccess;
}

void regroup_free(Regroup& g, cudaStream_t st) {
  if (g.buf) cudaFreeAsync(g.buf, st);
  g.buf = nullptr;
}

// rows sorted by their head theta (descending; ties by row: the sort is stable), U16 gathered in that
// order; g.ths = the sorted thetas (the regrouped pass's theta_in), g.pm = regrouped row -> index row
cudaError_t regroup_rows(Regroup& g, const __half* U16, int64_t n, int ldh, cudaStream_t st) {
  k_iota32<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g.io, n);
  count_launch();
  cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(g.cub, g.cub_bytes, g.th, g.ths, g.io, g.pm, (int)n, 0, 32, st);
  count_launch(6);  // (CUB: histogram, exclusive sum, 4 onesweep passes)
  if (e != cudaSuccess) return e;
  const int vpr = ldh / 8;
  const int64_t tot = n * vpr;
  k_gather_rows16<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(reinterpret_cast<const uint4*>(U16), g.pm, n, vpr,
                                                                 reinterpret_cast<uint4*>(g.U16b));
  count_launch();
  return cudaGetLastError();
}

template <int KB, class Pol>
static cudaError_t launch_tc2cta(const BuildCtx& c, cudaStream_t st) {
  using C = Cfg2<KB, Pol>;
  rmips_index_s* x = c.idx;
  const int tail = tail_cols(x->d);
  CUtensorMap ta, tat, tb, tbt;
  if (!make_tmap_f16_box(&ta, x->U16, (uint64_t)x->n, (uint64_t)x->ldh, kBM) ||
      !make_tmap_f16_box(&tat, x->U16, (uint64_t)x->n, (uint64_t)x->ldh, kBM, tail) ||
      !make_tmap_f16_box(&tb, x->P16, (uint64_t)c.mb, (uint64_t)x->ldh, 64) ||
      !make_tmap_f16_box(&tbt, x->P16, (uint64_t)c.mb, (uint64_t)x->ldh, 64, tail))
    return cudaErrorNotSupported;
  cudaError_t e = set_smem_attr((const void*)k_build_tc2cta<KB, Pol>, C::TOTAL);
  if (e != cudaSuccess) return e;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, x->device);
  const int tiles = (int)((x->n + kBM - 1) / kBM);
  const int pairs_needed = (tiles + 1) / 2, pairs_max = sms / 2;
  const int grid = 2 * (pairs_needed < pairs_max ? pairs_needed : pairs_max);
  x->build_kernel = 4;
  x->cand_slots = Pol::kSlots;
  int stale_every = 16;  // checkpoint refresh period in item tiles (a multiple of the C-S check period 4)
  // head pass length in item tiles (a multiple of the C-S check period); regrouping pays when the item
  // set is long against the head and there are several waves of tile pairs to regroup
  int head = 32;
#ifdef RMIPS_DEV
  if (const char* e = getenv("RMIPS_HEAD_TILES")) head = atoi(e) & ~3;    // 0: no regrouping
#endif
  const int64_t nit = (c.mb + 127) / 128;
  const bool regroup = head > 0 && nit >= 16 * (int64_t)head && tiles >= 4 * sms && (int64_t)head * 128 >= x->kmax;
  // the stale-theta refresh no longer cuts tiles once the rows are regrouped and continue from their head
  // state (configs[4]: 16,723,224 item tiles with it, 16,723,392 without, 0.7-1 ms faster without)
  if (regroup) stale_every = 0;
#ifdef RMIPS_DEV
  if (const char* e = getenv("RMIPS_STALE_EVERY")) stale_every = atoi(e);  // 0: off
#endif
  const int kmax = x->kmax, ksteps = (x->d + 15) / 16;
  // seed pass (the single pass and the head pass): 8 item tiles, 128 group maxima in the row's 128 slots
  int seed = nit >= 32 && Pol::kSlots >= 128 && 128 >= kmax ? 8 : 0;
#ifdef RMIPS_DEV
  if (const char* e = getenv("RMIPS_SEED_TILES")) seed = atoi(e) > 0 ? seed : 0;  // 0: no seed pass
#endif
  const int64_t n = x->n;
  // the two-pass scratch (~n (0.5 KB + 2 ldh) bytes); when it cannot be had the build takes the single pass
  Regroup g;
  CUtensorMap ga, gat;
  bool two = regroup;
  if (two && regroup_alloc(g, n, x->ldh, Pol::kEntWords, st) != cudaSuccess) {
    cudaGetLastError();
    g.buf = nullptr;
    two = false;
  }
  if (two && (!make_tmap_f16_box(&ga, g.U16b, (uint64_t)n, (uint64_t)x->ldh, kBM) ||
              !make_tmap_f16_box(&gat, g.U16b, (uint64_t)n, (uint64_t)x->ldh, kBM, tail))) {
    regroup_free(g, st);
    two = false;
  }
  if (!two) {
    if (regroup) stale_every = 16;  // (the single pass's period)
    k_build_tc2cta<KB, Pol><<<grid, C::THREADS, C::TOTAL, st>>>(ta, tat, tb, tbt, x->perr, x->pnorm, c.scale_dev, n,
                                                                c.mb, kmax, ksteps, tail, c.cand, c.ccount, c.ovf_list,
                                                                c.ovf_count, c.tiles_done, stale_every, seed, 0, 0,
                                                                nullptr, nullptr, nullptr, nullptr);
    count_launch();
    return cudaGetLastError();
  }
  k_build_tc2cta<KB, Pol><<<grid, C::THREADS, C::TOTAL, st>>>(ta, tat, tb, tbt, x->perr, x->pnorm, c.scale_dev, n, c.mb,
                                                              kmax, ksteps, tail, c.cand, c.ccount, c.ovf_list,
                                                              c.ovf_count, c.tiles_done, stale_every, seed, 0, head,
                                                              g.th, g.ent, g.meta, nullptr);
  count_launch();
  e = regroup_rows(g, x->U16, n, x->ldh, st);
  if (e == cudaSuccess) {
    k_build_tc2cta<KB, Pol><<<grid, C::THREADS, C::TOTAL, st>>>(ga, gat, tb, tbt, x->perr, x->pnorm, c.scale_dev, n,
                                                                c.mb, kmax, ksteps, tail, c.cand, c.ccount,
                                                                c.ovf_list, c.ovf_count, c.tiles_done, stale_every, 0,
                                                                head, 0, nullptr, g.ent, g.meta, g.pm);
    count_launch();
    e = cudaGetLastError();
  }
  regroup_free(g, st);
  return e;
}

// CTA-pair build for d_pad <= 256 with 128-slot 4-byte candidate lists (m <= 2^20, k_max <= 80);
// cudaErrorNotSupported otherwise (the caller then takes build_tcq).
cudaError_t build_tc2cta(const BuildCtx& c, cudaStream_t st) {
  if (c.cstride != kCand || c.mb > QPolT<128>::kMaxItems) return cudaErrorNotSupported;
  switch (c.idx->dpad) {
    case 64:
#ifdef RMIPS_DEV
      if (const char* e = getenv("RMIPS_2CTA_FPOL"))  // 8-byte entries (cand.cuh); 2: branch-free appends
        return atoi(e) == 2 ? launch_tc2cta<1, FPolFlat>(c, st) : launch_tc2cta<1, FPol>(c, st);
#endif
      return launch_tc2cta<1, QPolT<128>>(c, st);
    case 128: return launch_tc2cta<2, QPolT<128>>(c, st);
    case 192: return launch_tc2cta<3, QPolT<128>>(c, st);
    case 256: return launch_tc2cta<4, QPolT<128>>(c, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace rmips
