// query_tc.cu -- Q2 + Q3 on the 5th-generation tensor cores: Lemma 3 block pruning
// and the fused query x user contraction with the O(1) Lemma 1 classify epilogue (
// Alg. 3 lines 4-9).  The |B| x |Q| score block never leaves TMEM.
//
// Work item = (query sub-batch s of <= 256 norm-sorted queries, user tile t of 128 norm-sorted
// users).  One persistent CTA per SM walks the work items, 6 warps:
//   warp 0      TMA producer: the sub-batch's queries Q16 (256 x 64 fp16 per K block, kept in
//               shared memory while the CTA stays on that sub-batch) and the stream of user tiles
//               through a ring of K-block units (128 x 64 fp16 each, SWIZZLE_128B); d_pad <= 256
//   warp 1      TMEM allocator + MMA issuer: tcgen05.mma.cta_group::1.kind::f16, M = 128 users,
//               N = the Lemma 3 prefix of the sub-batch rounded up to 16 (<= 256 queries),
//               K = 16 x 4 per K block, fp32 accumulators in TMEM, 2 stages x 256 columns
//   warps 2-5   epilogue: one thread per user row (TMEM lane); 32 query columns per tcgen05.ld;
//               a chunk whose max score is below the row's threshold minus the chunk's error
//               bound is rejected wholesale (the common case), otherwise each pair is classified
//               exactly like the SIMT kernel (classify(), query.cu) and accepted / undecided
//               pairs are compacted per warp (one atomic per list per chunk).
// Every role evaluates the Lemma 3 prefix of a work item itself (same inputs, same answer), so a
// pruned item costs neither HBM traffic nor MMA nor epilogue time.
#include <cuda.h>

#include "common.cuh"
#include "internal.h"
#include "sm100.cuh"

namespace rmips {

#ifdef RMIPS_EPI_PROFILE
__device__ unsigned long long g_qprof[8];  // development-only wait-time counters (tools/query_profile.py)
#define QPROF_T0() const long long _t0 = clock64()
#define QPROF_ADD(slot) atomicAdd(&g_qprof[slot], (unsigned long long)(clock64() - _t0))
#else
#define QPROF_T0()
#define QPROF_ADD(slot)
#endif

namespace {

constexpr int kBM = 128;                  // users per tile (TMEM lanes)
constexpr int kUTileBytes = kBM * 64 * 2; // one K block of a user tile: 128 x 64 fp16 = 16 KB
constexpr int kQTileBytes = kQB * 64 * 2; // 256 x 64 fp16 = 32 KB
constexpr int kThreads = 320;           // producer, MMA, 8 epilogue warps (2 per TMEM lane quadrant)
// development-only switch bits OR-ed into `flags` by librmips_dev.so (never set in the product)
constexpr int kDevQEpiSkip = 1 << 28;  // RMIPS_Q_EPI_SKIP: the epilogue releases every stage unread
constexpr int kDevQNoSlow = 1 << 27;   // RMIPS_Q_NO_SLOW: flagged chunks are not classified (timing only)
constexpr int kDevQCount = 1 << 26;    // RMIPS_Q_COUNT: count flagged / examined warp-chunks (g_qdev)
constexpr int kDevQNoFeed = 1 << 25;   // RMIPS_Q_NOFEED: ring units after the first round are not reloaded
#ifdef RMIPS_DEV
__device__ unsigned long long g_qdev[4];  // dev: [0] flagged warp-chunks, [1] examined warp-chunks
#endif
constexpr int kAccCols = 256;             // TMEM columns per accumulator stage
constexpr int kAcc = 2;

// The user stream is a ring of K-block units (16 KB each): a user tile of d_pad = 64*KB columns
// takes KB consecutive units, and the MMA on K block kb starts as soon as that unit has landed.
// KB = 0 (d_pad > 256: the queries do not fit in shared memory next to the ring): every ring unit holds
// K block kb of the user tile (16 KB) AND of the sub-batch's queries (32 KB, re-read from L2 per tile).
// KB = 1..4: the resident queries take (KB - 1) 32 KB units plus the trimmed tail unit (256 x tail
// columns), and the ring gets every 16 KB unit left (at most kMaxNU): d = 200 keeps 104 KB of queries and
// 7 ring units.  The layout is computed at run time (QLayout) from KB and the tail width.
constexpr int kMaxNU = 8;
struct QLayout {
  int nu, unit, a, bar, total;  // ring units, unit bytes, ring offset, barrier offset, dynamic smem bytes
  __host__ __device__ static QLayout make(int KB, int tail) {
    QLayout l;
    if (KB == 0) {
      l.unit = kUTileBytes + kQTileBytes;
      l.a = 0;
      l.nu = 4;
    } else {
      l.unit = kUTileBytes;
      l.a = ((KB - 1) * kQTileBytes + kQB * tail * 2 + 1023) / 1024 * 1024;
      l.nu = (232448 - 1024 - 512 - l.a) / l.unit;
      if (l.nu > kMaxNU) l.nu = kMaxNU;
    }
    l.bar = l.a + l.nu * l.unit;
    l.total = l.bar + 512 + 1024;  // barriers (<= 2 + 2 kMaxNU + 4) + TMEM slot, alignment slack
    return l;
  }
};

__device__ __forceinline__ int lemma3_len(const float* __restrict__ qn_sub, int cnt, float tbv) {
  int lo = 0, hi = cnt;  // queries are norm-sorted: the kept ones are a prefix (#{qn >= tbv})
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(qn_sub + mid) >= tbv) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Same decision rule as classify() in query.cu: 0 reject, 1 accept, 2 undecided.
__device__ __forceinline__ int classify_tc(float acc, float thr_s, float qe) {
  float E = __fadd_ru(qe, fabsf(thr_s) * 2.384185791015625e-07f);
  if (__fadd_ru(acc, E) < thr_s) return 0;
  if (__fsub_rd(acc, E) >= thr_s) return 1;
  return 2;
}

// Per-warp slot pools: a warp reserves list slots kPoolChunk at a time (one returning atomic per
// reservation instead of one per chunk); slots it does not fill are padded with kSentinel at the
// end of the kernel, which sorts last and is skipped by the exact path.
constexpr int kPoolChunk = 128;
struct QPool {
  unsigned long long abase, ubase;  // next free slot of the accepted / undecided pool
  int aleft, uleft;                 // slots left in it
};

// Position of this lane's first record among `tot` records of the warp (prefix p, count c):
// records beyond the pool continue in a freshly reserved block.
__device__ __forceinline__ void pool_take(unsigned long long& base, int& left, int tot, unsigned long long* counter,
                                          unsigned long long& nbase) {
  nbase = 0;
  if (tot > left) {  // warp-uniform
    const int need = tot - left;
    const int res = (need + kPoolChunk - 1) / kPoolChunk * kPoolChunk;
    if ((threadIdx.x & 31) == 0) nbase = atomicAdd(counter, (unsigned long long)res);
    nbase = __shfl_sync(0xffffffffu, nbase, 0);
  }
}
__device__ __forceinline__ unsigned long long pool_slot(unsigned long long base, int left, unsigned long long nbase,
                                                        int p) {
  return p < left ? base + p : nbase + (p - left);
}
__device__ __forceinline__ void pool_advance(unsigned long long& base, int& left, int tot, unsigned long long nbase) {
  if (tot > left) {
    const int need = tot - left;
    const int res = (need + kPoolChunk - 1) / kPoolChunk * kPoolChunk;
    base = nbase + need;
    left = res - need;
  } else {
    base += tot;
    left -= tot;
  }
}

struct QSlowOut {
  QPool pool;
  uint32_t na, nu;
};

// Classify every pair of the flagged 32-column chunks (re-read from TMEM), then compact the
// accepted and undecided pairs of the warp: one atomic per list per chunk.  Returns this
// thread's (accepted, undecided) counts.  The stage stays held until this returns, so the chain
// is kept short: the chunk's 32 error bounds are one coalesced load issued with the TMEM read and
// broadcast by shuffles, and every pair is classified branch-free (as classify_tc).
__device__ __noinline__ QSlowOut q_slow(QPool pool, uint32_t flag, uint32_t tbase, int len, bool live, float thr_s,
                                        const float* __restrict__ qe_sub, const int32_t* __restrict__ qp_sub,
                                        uint64_t uo, int64_t row, bool force, unsigned long long* __restrict__ ctr,
                                        AccSink acc_list, uint64_t* __restrict__ und_list,
                                        int64_t cap) {
  using namespace sm100;
  const int lane = threadIdx.x & 31;
  const float thr_abs = fabsf(thr_s) * 2.384185791015625e-07f;
  uint32_t n_acc = 0, n_und = 0;
#pragma unroll 1
  while (flag) {
    const int ci = __ffs(flag) - 1;
    flag &= flag - 1;
    const int col0 = 32 * ci;
    uint32_t r[32];
    tmem_ld32(tbase + col0, r);
    const float qv = __ldg(qe_sub + col0 + lane);  // qerr of slot col0 + lane (broadcast below)
    tmem_ld_wait(r);
    const int lim = live ? min(32, len - col0) : 0;  // columns of this chunk that are scored
    uint32_t am = 0, um = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float E = __fadd_ru(__shfl_sync(0xffffffffu, qv, j), thr_abs);
      const float a = __uint_as_float(r[j]);
      const bool keep = j < lim && !(__fadd_ru(a, E) < thr_s);  // not rejected (classify_tc: 0)
      const bool acc = keep && __fsub_rd(a, E) >= thr_s;          // accepted (1); else undecided (2)
      am |= (uint32_t)acc << j;
      um |= (uint32_t)(keep && !acc) << j;
    }
    if (force) um |= am, am = 0;
    if (!__any_sync(0xffffffffu, (am | um) != 0)) continue;
    const int na = __popc(am), nu = __popc(um);
    n_acc += na;
    n_und += nu;
    // warp-inclusive prefix sums; slots come from the warp's pools (rarely an atomic)
    int pa = na, pu = nu;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int xa = __shfl_up_sync(0xffffffffu, pa, o), xu = __shfl_up_sync(0xffffffffu, pu, o);
      if (lane >= o) pa += xa, pu += xu;
    }
    const int ta = __shfl_sync(0xffffffffu, pa, 31), tu = __shfl_sync(0xffffffffu, pu, 31);
    unsigned long long na_base, nu_base;
    if (!acc_list.bits) pool_take(pool.abase, pool.aleft, ta, ctr + C_ACCEPTED_TOTAL, na_base);
    pool_take(pool.ubase, pool.uleft, tu, ctr + C_UND_TOTAL, nu_base);
    int p = pa - na;
    while (am) {
      const int j = __ffs(am) - 1;
      am &= am - 1;
      const uint64_t key = ((uint64_t)(uint32_t)__ldg(qp_sub + col0 + j) << 32) | uo;
      if (acc_list.bits) {
        acc_list.set(key);
      } else {
        const unsigned long long slot = pool_slot(pool.abase, pool.aleft, na_base, p++);
        if ((int64_t)slot < cap) acc_list.list[slot] = key;
      }
    }
    p = pu - nu;
    while (um) {
      const int j = __ffs(um) - 1;
      um &= um - 1;
      const unsigned long long slot = pool_slot(pool.ubase, pool.uleft, nu_base, p++);
      if ((int64_t)slot < cap) und_list[slot] = ((uint64_t)(uint32_t)__ldg(qp_sub + col0 + j) << 32) | (uint64_t)row;
    }
    if (!acc_list.bits) pool_advance(pool.abase, pool.aleft, ta, na_base);
    pool_advance(pool.ubase, pool.uleft, tu, nu_base);
  }
  QSlowOut out;
  out.pool = pool;
  out.na = n_acc;
  out.nu = n_und;
  return out;
}

}  // namespace

// Lemma 3 for every work item (sub-batch s, user tile t): the number of leading
// norm-sorted queries with ||q|| >= tb_k(t) (0 prunes the item whole), plus the block counters.
__global__ void __launch_bounds__(256)
k_lemma3_lens(const float* __restrict__ tbk, const float* __restrict__ qn, const int32_t* __restrict__ qcount,
              int nblocks, int bsz, int64_t nlb, int64_t nwork, int flags, int32_t* __restrict__ wlen,
              unsigned long long* __restrict__ ctr) {
  pdl_enter();  // (PDL: see launch_pdl)
  // the norms of the (at most kStage) sub-batches this CTA's items fall in are staged in shared memory, so
  // each binary search is a chain of shared loads instead of ~8 dependent L2 round trips
  constexpr int kStage = 4;
  __shared__ float sq[kStage * kQB];
  const int64_t w0 = blockIdx.x * (int64_t)blockDim.x;
  const int64_t wl = min(w0 + (int64_t)blockDim.x, nwork) - 1;
  const int s0 = (int)(w0 / nblocks), ns = wl >= w0 ? (int)(wl / nblocks) - s0 + 1 : 0;
  const bool staged = ns <= kStage;
  if (staged)
    for (int i = threadIdx.x; i < ns * kQB; i += blockDim.x) sq[i] = __ldg(qn + (int64_t)s0 * kQB + i);
  __syncthreads();
  const int64_t w = w0 + threadIdx.x;
  unsigned long long pairs = 0, pruned = 0, scored = 0;
  if (w < nwork) {
    const int s = (int)(w / nblocks), t = (int)(w - (int64_t)s * nblocks);
    const int cnt = qcount[s];
    const float* qs = qn + (int64_t)s * kQB;
    const float* ss = sq + (s - s0) * kQB;
    const int len = tile_lemma3(t, bsz, nlb, cnt, (flags & RMIPS_FLAG_NO_BLOCKS) != 0, tbk,
                                [&](float tbv) {
                                  if (!staged) return lemma3_len(qs, cnt, tbv);
                                  int lo = 0, hi = cnt;  // as lemma3_len, on the staged copy
                                  while (lo < hi) {
                                    const int mid = (lo + hi) >> 1;
                                    if (ss[mid] >= tbv) lo = mid + 1; else hi = mid;
                                  }
                                  return lo;
                                },
                                pairs, pruned);
    wlen[w] = len;
    scored = len > 0;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    pairs += __shfl_xor_sync(0xffffffffu, pairs, o);
    pruned += __shfl_xor_sync(0xffffffffu, pruned, o);
    scored += __shfl_xor_sync(0xffffffffu, scored, o);
  }
  if ((threadIdx.x & 31) == 0 && pairs) {
    atomicAdd(ctr + C_BLOCK_PAIRS, pairs);
    atomicAdd(ctr + C_BLOCK_PRUNED, pruned);
    atomicAdd(ctr + C_TILES_SCORED, scored);
  }
}

template <int KB>
__global__ void __launch_bounds__(kThreads, 1)
k_query_tc(const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmUt,
           const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmQt, int kb_rt, int tail,
           const float* __restrict__ thrk, const float* __restrict__ tbk, const int32_t* __restrict__ perm_u,
           int64_t n, int nblocks, const float* __restrict__ qn, const float* __restrict__ qerr,
           const float* __restrict__ qscale, const int32_t* __restrict__ qperm, const int32_t* __restrict__ qcount,
           int nsub, int flags, int ksteps, const int32_t* __restrict__ wlen, unsigned long long* __restrict__ ctr,
           AccSink acc_list, uint64_t* __restrict__ und_list, int64_t cap) {
  pdl_enter();  // (PDL: see launch_pdl)
  using namespace sm100;
  const QLayout lay = QLayout::make(KB, tail);
  const int kStages = lay.nu;  // ring units
  const int kUnit = lay.unit;
  constexpr bool kStreamQ = KB == 0;
  const int kbn = kStreamQ ? kb_rt : KB;  // K blocks per row; the last one is `tail` columns wide
  const uint32_t utail = (uint32_t)(kBM * tail * 2), qtail = (uint32_t)(kQB * tail * 2);
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t sQ = sbase;
  const uint32_t sA = sbase + lay.a;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + lay.bar);
  const uint32_t bar0 = smem_u32(bars);
  auto BAR = [&](int i) { return bar0 + 8u * i; };
  const int Q_FULL = 0, Q_EMPTY = 1, A_FULL = 2, A_EMPTY = 2 + kStages, ACC_FULL = 2 + 2 * kStages,
            ACC_EMPTY = 2 + 2 * kStages + kAcc;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 + 2 * kStages + 2 * kAcc);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t nwork = (int64_t)nsub * nblocks;
  const bool use_blocks = !(flags & RMIPS_FLAG_NO_BLOCKS);

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmU);
    tma_prefetch(&tmQ);
    tma_prefetch(&tmUt);
    tma_prefetch(&tmQt);
    mbar_init(BAR(Q_FULL), 1);
    mbar_init(BAR(Q_EMPTY), 1);
    for (int s = 0; s < kStages; ++s) mbar_init(BAR(A_FULL + s), 1), mbar_init(BAR(A_EMPTY + s), 1);
    for (int a = 0; a < kAcc; ++a) mbar_init(BAR(ACC_FULL + a), 1), mbar_init(BAR(ACC_EMPTY + a), 8);
    fence_mbar_init();
  }
  if (warp == 1) {
    tmem_alloc(smem_u32(tmem_slot), kAcc * kAccCols);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Work items w = blockIdx.x + i * gridDim.x; (sub-batch s, user tile t) advanced without
  // divisions; the Lemma 3 prefix of every item comes from k_lemma3_lens (one load).
  auto first_item = [&](int& s, int& t) {
    s = (int)((int64_t)blockIdx.x / nblocks);
    t = (int)((int64_t)blockIdx.x - (int64_t)s * nblocks);
  };
  auto next_item = [&](int& s, int& t) {
    t += gridDim.x;
    while (t >= nblocks) t -= nblocks, ++s;
  };
  // Lemma 3 prefix lengths of this CTA's items, loaded four items ahead (the producer and MMA warps
  // otherwise start every item with a dependent global load)
  struct LenQ {
    int v0, v1, v2, v3;
  };
  auto lenq_init = [&]() {
    LenQ q;
    const int64_t g = gridDim.x, w0 = blockIdx.x;
    q.v0 = w0 < nwork ? __ldg(wlen + w0) : 0;
    q.v1 = w0 + g < nwork ? __ldg(wlen + w0 + g) : 0;
    q.v2 = w0 + 2 * g < nwork ? __ldg(wlen + w0 + 2 * g) : 0;
    q.v3 = w0 + 3 * g < nwork ? __ldg(wlen + w0 + 3 * g) : 0;
    return q;
  };
  auto lenq_pop = [&](LenQ& q, int64_t w) {  // the length of item w; item w + 4 g is requested
    const int len = q.v0;
    q.v0 = q.v1, q.v1 = q.v2, q.v2 = q.v3;
    const int64_t w4 = w + 4 * (int64_t)gridDim.x;
    q.v3 = w4 < nwork ? __ldg(wlen + w4) : 0;
    return len;
  };

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      int stage = 0, cur_s = -1, nq = 0, nloads = 0;
      uint32_t ph = 0;
      int s, t;
      first_item(s, t);
      LenQ lq = lenq_init();
      for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x, next_item(s, t)) {
        const int len = lenq_pop(lq, w);
        if (len == 0) continue;
        if (!kStreamQ && s != cur_s) {
          if (nq > 0) mbar_wait(BAR(Q_EMPTY), (nq - 1) & 1);
          mbar_arrive_expect_tx(BAR(Q_FULL), (uint32_t)((kbn - 1) * kQTileBytes) + qtail);
          for (int kb = 0; kb < kbn; ++kb)
            tma_load_2d(sQ + kb * kQTileBytes, kb == kbn - 1 ? &tmQt : &tmQ, kb * 64, s * kQB, BAR(Q_FULL));
          ++nq;
          cur_s = s;
        }
        for (int kb = 0; kb < kbn; ++kb) {
          {
            QPROF_T0();
            mbar_wait(BAR(A_EMPTY + stage), ph ^ 1);
            QPROF_ADD(4);
          }
          const bool last = kb == kbn - 1;
          if ((flags & kDevQNoFeed) && nloads >= kStages) {  // dev: stale unit, no HBM traffic
            mbar_arrive(BAR(A_FULL + stage));
            if (++stage == kStages) stage = 0, ph ^= 1;
            continue;
          }
          ++nloads;
          mbar_arrive_expect_tx(BAR(A_FULL + stage), (last ? utail : (uint32_t)kUTileBytes) +
                                                         (kStreamQ ? (last ? qtail : (uint32_t)kQTileBytes) : 0u));
          tma_load_2d(sA + stage * kUnit, last ? &tmUt : &tmU, kb * 64, t * kBM, BAR(A_FULL + stage));
          if (kStreamQ)
            tma_load_2d(sA + stage * kUnit + kUTileBytes, last ? &tmQt : &tmQ, kb * 64, s * kQB, BAR(A_FULL + stage));
          if (++stage == kStages) stage = 0, ph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // The whole warp walks the work (warp-uniform state: descriptors in uniform registers); the
    // elected lane issues the tcgen05 instructions (as in build_tcq.cu).
    int stage = 0, as = 0, cur_s = -1, nq = 0;
    uint32_t ph = 0, aph = 0;
    int s, t;
    first_item(s, t);
    LenQ lq = lenq_init();
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x, next_item(s, t)) {
      const int len = lenq_pop(lq, w);
      if (len == 0) continue;
      if (!kStreamQ && s != cur_s) {
        if (nq > 0) {
          if (elect_one()) mma_commit(BAR(Q_EMPTY));  // all MMAs on the previous sub-batch's queries
          __syncwarp();
        }
        QPROF_T0();
        mbar_wait(BAR(Q_FULL), nq & 1);
        QPROF_ADD(0);
        ++nq;
        cur_s = s;
      }
      {
        QPROF_T0();
        mbar_wait(BAR(ACC_EMPTY + as), aph ^ 1);
        QPROF_ADD(1);
      }
      const int N = (len + 15) & ~15;
      const uint32_t idesc = idesc_f16_f32(kBM, N);
      const uint32_t d = tmem + as * kAccCols;
      if (!kStreamQ) {
        // the work item's KB units are all awaited first, then one elected MMA chain (13 MMAs at
        // d = 200) with one commit per unit: the MMA warp's per-item overhead does not scale with KB
        int st_ = stage;
        uint32_t ph_ = ph;
        for (int kb = 0; kb < kbn; ++kb) {
          QPROF_T0();
          mbar_wait(BAR(A_FULL + st_), ph_);
          QPROF_ADD(2);
          if (++st_ == kStages) st_ = 0, ph_ ^= 1;
        }
        tc_fence_after();
        if (elect_one()) {
          int su = stage;
#pragma unroll
          for (int kb = 0; kb < KB; ++kb) {
            const bool last = kb == KB - 1;  // the tail K block has its own swizzle (tail_cols)
            const uint32_t ua = sA + su * kUnit, qa = sQ + kb * kQTileBytes;
            const uint64_t adesc = last ? sdesc_swz(ua, 2 * tail) : sdesc_sw128(ua);
            const uint64_t bdesc = last ? sdesc_swz(qa, 2 * tail) : sdesc_sw128(qa);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // K advance: 32 bytes = 2 in the 16-byte address field
              if (4 * kb + kk < ksteps)
                mma_f16(d, adesc + (uint64_t)(2 * kk), bdesc + (uint64_t)(2 * kk), idesc, (kb | kk) != 0);
            mma_commit(BAR(A_EMPTY + su));
            if (++su == kStages) su = 0;
          }
        }
        __syncwarp();
        stage = st_;
        ph = ph_;
      } else {  // KB = 0: per unit (the queries' K blocks stream with the users')
        for (int kb = 0; kb < kbn; ++kb) {
          {
            QPROF_T0();
            mbar_wait(BAR(A_FULL + stage), ph);
            QPROF_ADD(2);
          }
          tc_fence_after();
          const bool last = kb == kbn - 1;  // the tail K block has its own swizzle (tail_cols)
          const uint32_t ua = sA + stage * kUnit, qa = kStreamQ ? ua + kUTileBytes : sQ + kb * kQTileBytes;
          const uint64_t adesc = last ? sdesc_swz(ua, 2 * tail) : sdesc_sw128(ua);
          const uint64_t bdesc = last ? sdesc_swz(qa, 2 * tail) : sdesc_sw128(qa);
          const int kk_end = min(4, ksteps - 4 * kb);  // zero-padding K steps are skipped
          if (elect_one()) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // K advance: 32 bytes = 2 in the 16-byte address field
              if (kk < kk_end) mma_f16(d, adesc + (uint64_t)(2 * kk), bdesc + (uint64_t)(2 * kk), idesc, (kb | kk) != 0);
            mma_commit(BAR(A_EMPTY + stage));
          }
          __syncwarp();
          if (++stage == kStages) stage = 0, ph ^= 1;
        }
      }
      if (elect_one()) mma_commit(BAR(ACC_FULL + as));
      __syncwarp();
      if (++as == kAcc) as = 0, aph ^= 1;
    }
  } else {
    // ------------------------------------------------ epilogue: one thread per user row
    // Fast pass over the len scored columns (two halves of 4 chunks): chunk max vs the row's
    // threshold.  Chunks where some pair may be accepted / undecided are flagged and classified
    // by q_slow (one out-of-line copy: the hot loop stays inside the instruction cache), which
    // re-reads them from TMEM before the stage is released.
    // Eight epilogue warps: warp w reads TMEM lane quadrant w % 4 and the query-column half
    // (w - 2) / 4 (pairs are independent, so the two warps of a quadrant share nothing).
    const int q = warp & 3;  // TMEM lane quadrant of this warp
    const int hsel = (warp - 2) >> 2;
    const int rloc = q * 32 + lane;
    const bool force = (flags & RMIPS_FLAG_FORCE_VERIFY) != 0;
    unsigned long long n_scored = 0, n_fast = 0, n_und = 0;
    QPool pool{0ull, 0ull, 0, 0};
    int as = 0;
    uint32_t aph = 0;
    int s, t;
    first_item(s, t);
    // the per-item inputs (Lemma 3 prefix, the row's threshold, the sub-batch scale and error
    // bounds) are loaded one work item ahead, so their latency hides behind the current item
    int p_len = 0;
    float p_sc = 0.f, p_thr = 0.f, p_qe[8];
    auto preload = [&](int64_t w_, int s_, int t_) {
      if (w_ >= nwork) return;
      p_len = __ldg(wlen + w_);
      p_sc = __ldg(qscale + s_);
      const int64_t r_ = (int64_t)t_ * kBM + rloc;
      p_thr = r_ < n ? __ldg(thrk + r_) : 0.f;
      const float* qs_ = qerr + (int64_t)s_ * kQB;
#pragma unroll
      for (int c = 0; c < 8; ++c) p_qe[c] = __ldg(qs_ + 32 * c);
    };
    preload(blockIdx.x, s, t);
    for (int64_t w = blockIdx.x; w < nwork; w += gridDim.x, next_item(s, t)) {
      const int len = p_len;
      const float sc = p_sc, thr_raw = p_thr;
      float qe[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) qe[c] = p_qe[c];
      {
        int s2 = s, t2 = t;
        next_item(s2, t2);
        preload(w + gridDim.x, s2, t2);
      }
      if (len == 0) continue;
      const int64_t row = (int64_t)t * kBM + rloc;
      const bool live = row < n;
      const float thr_s = live ? thr_raw * sc : CUDART_INF_F;  // dead rows reject everything
      const float thr_abs = fabsf(thr_s) * 2.384185791015625e-07f;
      const float* qe_sub = qerr + (int64_t)s * kQB;
      const int hlen = min(128, max(0, len - 128 * hsel));  // scored columns of this warp's half
      if (flags & kDevQEpiSkip) {  // dev: MMA + feed alone
        mbar_wait(BAR(ACC_FULL + as), aph);
        tc_fence_after();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR(ACC_EMPTY + as));
        if (++as == kAcc) as = 0, aph ^= 1;
        continue;
      }
      if (live) n_scored += hlen;
      // qerr is non-increasing along the norm-sorted slots: a chunk's first slot bounds it
      // (chunks at or beyond len are masked below, so their entries never matter)
      float Emax[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) Emax[c] = __fadd_ru(qe[c], thr_abs);
      {
        QPROF_T0();
        mbar_wait(BAR(ACC_FULL + as), aph);
        if (lane == 0) QPROF_ADD(3);
      }
      tc_fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + as * kAccCols;
      uint32_t flag = 0;  // warp-uniform: chunks that need the slow path
      if (hsel * 128 < len) {
        const int h = hsel;
        uint32_t r[4][32];
        tmem_ld32(tbase + h * 128, r[0]);
        tmem_ld32(tbase + h * 128 + 32, r[1]);
        tmem_ld32(tbase + h * 128 + 64, r[2]);
        tmem_ld32(tbase + h * 128 + 96, r[3]);
        tmem_ld_wait(r[0]);
        reg_fence(r[1]);
        reg_fence(r[2]);
        reg_fence(r[3]);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          // columns >= len hold stale or zero values: a spurious flag only costs a slow-path
          // visit, which masks them
          const float mx = sm100::max32_bits(r[c]);
          const float em = h ? Emax[4 + c] : Emax[c];
          const bool all_rej = !live || (__fadd_ru(mx, em) < thr_s);
          flag |= (uint32_t)(!__all_sync(0xffffffffu, all_rej)) << (4 * h + c);
        }
      }
      // chunks at or beyond len are never classified
      flag &= len >= 256 ? 0xffu : ((1u << ((len + 31) >> 5)) - 1u);
#ifdef RMIPS_DEV
      if (lane == 0 && (flags & kDevQCount) && hsel * 128 < len) {
        atomicAdd(&g_qdev[0], (unsigned long long)__popc(flag));
        atomicAdd(&g_qdev[1], (unsigned long long)((min(len, 128 * hsel + 128) - 128 * hsel + 31) / 32));
      }
#endif
      if (flag && !(flags & kDevQNoSlow)) {
        const uint64_t uo = live ? (uint64_t)(uint32_t)__ldg(perm_u + row) : 0;
        const QSlowOut o = q_slow(pool, flag, tbase, len, live, thr_s, qe_sub, qperm + (int64_t)s * kQB, uo, row,
                                  force, ctr, acc_list, und_list, cap);
        pool = o.pool;
        n_fast += o.na;
        n_und += o.nu;
      }
      tc_fence_before();  // this accumulator stage is fully read: hand it back to the MMA warp
      __syncwarp();
      if (lane == 0) mbar_arrive(BAR(ACC_EMPTY + as));
      if (++as == kAcc) as = 0, aph ^= 1;
    }
    // pad the unused pool slots (warp-uniform pools; lanes share the work)
    for (int i = lane; i < pool.aleft; i += 32)
      if ((int64_t)(pool.abase + i) < cap) acc_list.list[pool.abase + i] = kSentinel;
    for (int i = lane; i < pool.uleft; i += 32)
      if ((int64_t)(pool.ubase + i) < cap) und_list[pool.ubase + i] = kSentinel;
    // counters: one atomic per warp
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      n_scored += __shfl_xor_sync(0xffffffffu, n_scored, o);
      n_fast += __shfl_xor_sync(0xffffffffu, n_fast, o);
      n_und += __shfl_xor_sync(0xffffffffu, n_und, o);
    }
    if (lane == 0 && n_scored) {
      atomicAdd(ctr + C_SCORED, n_scored);
      atomicAdd(ctr + C_ACCEPT_FAST, n_fast);
      atomicAdd(ctr + C_ACC_REAL, n_fast);
      atomicAdd(ctr + C_REJECTED, n_scored - n_fast - n_und);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kAcc * kAccCols);
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

template <int KB>
static cudaError_t launch_query_tc(QueryCtx& c, cudaStream_t st) {
  rmips_index_s* x = c.idx;
  const int tail = tail_cols(x->d);
  CUtensorMap tu, tut, tq, tqt;
  if (!make_tmap_f16_box(&tu, x->U16, (uint64_t)x->n, (uint64_t)x->ldh, kBM) ||
      !make_tmap_f16_box(&tut, x->U16, (uint64_t)x->n, (uint64_t)x->ldh, kBM, tail) ||
      !make_tmap_f16_box(&tq, c.Q16, (uint64_t)c.nsub * kQB, (uint64_t)x->ldh, kQB) ||
      !make_tmap_f16_box(&tqt, c.Q16, (uint64_t)c.nsub * kQB, (uint64_t)x->ldh, kQB, tail))
    return cudaErrorNotSupported;
  const int smem = QLayout::make(KB, tail).total;
  cudaError_t e = set_smem_attr((const void*)k_query_tc<KB>, smem);
  if (e != cudaSuccess) return e;
  const int64_t nwork = (int64_t)c.nsub * x->nblocks;
  const int grid = (int)(nwork < sm_count_q() ? nwork : sm_count_q());
  int kflags = c.flags & 0xffff;  // bits 16.. carry the dev switches only
#ifdef RMIPS_DEV
  if (getenv("RMIPS_Q_EPI_SKIP")) kflags |= kDevQEpiSkip;
  if (getenv("RMIPS_Q_NO_SLOW")) kflags |= kDevQNoSlow;
  if (getenv("RMIPS_Q_COUNT")) kflags |= kDevQCount;
  if (getenv("RMIPS_Q_NOFEED")) kflags |= kDevQNoFeed;
#endif
  CK_PDL(launch_pdl(k_lemma3_lens, dim3((unsigned)((nwork + 255) / 256)), dim3(256), 0, st, x->tb + (int64_t)(c.k - 1) * x->nlb, c.qn,
                                                                 c.qcount, (int)x->nblocks, x->bsz, x->nlb, nwork,
                                                                 c.flags, c.wlen,
                                                                 c.counters));
  count_launch();
  if (c.ev_k[0]) cudaEventRecord(c.ev_k[0], st);
  CK_PDL(launch_pdl(k_query_tc<KB>, dim3(grid), dim3(kThreads), smem, st, tu, tut, tq, tqt, x->dpad / 64, tail, x->thr + (int64_t)(c.k - 1) * x->n,
                                               x->tb + (int64_t)(c.k - 1) * x->nlb, x->perm_u, x->n,
                                               (int)x->nblocks, c.qn, c.qerr, c.qscale, c.qperm, c.qcount, c.nsub,
                                               kflags, (x->d + 15) / 16, c.wlen, c.counters, AccSink{c.acc, c.bits, c.nw, c.dirty, c.nbr}, c.und, c.cap));
  count_launch();
  if (c.ev_k[1]) cudaEventRecord(c.ev_k[1], st);
  return cudaGetLastError();
}

cudaError_t query_filter_tc(QueryCtx& c, cudaStream_t st) {
#ifdef RMIPS_DEV
  if (getenv("RMIPS_DISABLE_TC")) return cudaErrorNotSupported;
#endif
  if (c.idx->n == 0) return cudaSuccess;
  switch (c.idx->dpad) {
    case 64: return launch_query_tc<1>(c, st);
    case 128: return launch_query_tc<2>(c, st);
    case 192: return launch_query_tc<3>(c, st);
    case 256: return launch_query_tc<4>(c, st);
    default: return launch_query_tc<0>(c, st);  // d_pad > 256: queries streamed with the users
  }
}

}  // namespace rmips

#ifdef RMIPS_EPI_PROFILE
extern "C" RMIPS_API int rmips_debug_query_profile(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, rmips::g_qprof, sizeof(rmips::g_qprof));
  if (reset) {
    static unsigned long long z[8] = {};
    cudaMemcpyToSymbol(rmips::g_qprof, z, sizeof z);
  }
  return 0;
}
#endif

#ifdef RMIPS_DEV
extern "C" RMIPS_API int rmips_debug_qdev(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, rmips::g_qdev, sizeof(rmips::g_qdev));
  if (reset) {
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(rmips::g_qdev, z, sizeof z);
  }
  return 0;
}
#endif
