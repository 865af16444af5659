// common.cuh -- internal definitions shared by the rmips CUDA sources (sm_100a only).
//
// Citations: P:n = PAPER.md line n (arXiv 2110.07131), SV = SURVEY.md, DESIGN.md §n.
#pragma once
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <math_constants.h>
#include <stdint.h>
#include <cmath>
#include <string>

#include "../../include/rmips.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "rmips is written for sm_100a (B200) only"
#endif

namespace rmips {

// Programmatic dependent launch (the query chain, internal.h launch_pdl): a kernel lets its dependent start
// launching at once and waits for its own predecessor (complete, memory flushed) before touching any of its
// outputs.  Both are no-ops when the kernel was launched without the attribute.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

// ---------------------------------------------------------------------------------------
// Fixed geometry.
constexpr int kTileU = 128;        // users per tile == Lemma 3 block size (reading R5)
constexpr int kCand = 128;         // candidate slots per user row in the build epilogue
constexpr int kCandPitch = kCand + 1;  // smem row pitch (bank-conflict-free appends)
constexpr int kQB = 256;           // queries per kernel batch (tcgen05 N <= 256)
constexpr int kMaxDim = 1024;      // largest d (the exact select stages fp64 user rows in shared memory)

// Device status flags (bitwise OR into Index::d_flags[0]).
constexpr int kFlagNonfinite = 1;
constexpr int kFlagPairOverflow = 2;

// Counter slots (Index::d_counters), mirrored into rmips_stats_t.
enum Counter {
  C_BLOCK_PAIRS = 0, C_BLOCK_PRUNED, C_SCORED, C_REJECTED, C_ACCEPT_FAST, C_UNDECIDED,
  C_EXACT_ACCEPT, C_SCANS, C_ITEMS_SCANNED, C_ACCEPTED_TOTAL, C_UND_TOTAL, C_TILES_SCORED, C_ACC_REAL,
  C_SCAN_EXACT,
  kNumCounters
};
// C_ACCEPTED_TOTAL / C_UND_TOTAL count RESERVED list slots (the tcgen05 filter reserves in blocks and
// pads unused slots with kSentinel); C_ACC_REAL counts the accepted records themselves.
constexpr uint64_t kSentinel = ~0ull;

// ---------------------------------------------------------------------------------------
// The exact inner product (R7).  Left-to-right fp64 sum of the products of the
// fp32 inputs.  Each product of two fp32 values is exact in fp64, so fma(a, b, s) rounds
// exactly once, like s + a*b: the result is bit-identical to the oracle's orc_dot and,
// crucially, the SAME routine evaluates q.u and p.u, so a query equal to an item gives
// bitwise-equal values (the identity ties of DESIGN.md R9).
__device__ __forceinline__ double dot64(const float* __restrict__ a, const float* __restrict__ b, int d) {
  double s = 0.0;
  for (int j = 0; j < d; ++j) s = __fma_rn((double)__ldg(a + j), (double)__ldg(b + j), s);
  return s;
}

// Order-preserving float <-> uint32 key (for radix selection).
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Warp-aggregated append of one 64-bit record per active predicate into a global list.
__device__ __forceinline__ void warp_append_u64(bool pred, uint64_t rec, unsigned long long* count,
                                                uint64_t* list, int64_t cap) {
  uint32_t bal = __ballot_sync(0xffffffffu, pred);
  if (!bal) return;
  int lane = threadIdx.x & 31;
  int leader = __ffs(bal) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(count, (unsigned long long)__popc(bal));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (pred) {
    unsigned long long pos = base + __popc(bal & lanemask_lt());
    if ((int64_t)pos < cap) list[pos] = rec;
  }
}

// Where accepted (query, user) pairs go: appended to a key list (sorted afterwards), or, when
// the batch's b x n bit matrix fits the workspace, set as bit (q, u) of that matrix (row stride
// nw words), which the output kernels read back in (q, u) order without a sort.
struct AccSink {
  uint64_t* list;
  uint32_t* bits;
  int64_t nw;
  uint8_t* dirty;  // bits path: one byte per 32-word block (1024 users) of a query row, set with its bits
  int64_t nbr;     // blocks per row
  // warp-collective: every lane calls it (bits is warp-uniform)
  __device__ __forceinline__ void put(bool pred, uint64_t key, unsigned long long* count, int64_t cap) const {
    if (bits) {
      if (pred) set(key);
    } else {
      warp_append_u64(pred, key, count, list, cap);
    }
  }
  __device__ __forceinline__ void put_one(uint64_t key, unsigned long long* count, int64_t cap) const {
    if (bits) {
      set(key);
    } else {
      const unsigned long long pos = atomicAdd(count, 1ull);
      if ((int64_t)pos < cap) list[pos] = key;
    }
  }
  __device__ __forceinline__ void set(uint64_t key) const {
    const uint32_t u = (uint32_t)key;
    const int64_t q = (int64_t)(key >> 32);
    atomicOr(bits + q * nw + (u >> 5), 1u << (u & 31));
    dirty[q * nbr + (u >> 10)] = 1;  // (every writer stores 1: no race to resolve)
  }
};

// Lemma 3 over the blocks of bsz users that overlap the 128-user tile t: len = the longest
// norm-sorted query prefix any of them keeps (the tile's MMA N; the rows of blocks with shorter
// prefixes reject the extra pairs exactly by Lemma 1), and the (block, query) pair counts of the blocks
// whose first user lies in the tile (every block is counted once).  len_of(tb) = #{queries : ||q|| >= tb}.
template <class LenFn>
__device__ __forceinline__ int tile_lemma3(int64_t t, int bsz, int64_t nlb, int cnt, bool no_blocks,
                                           const float* __restrict__ tbk, LenFn len_of,
                                           unsigned long long& pairs, unsigned long long& pruned) {
  const int64_t r0 = t * kTileU, r1 = r0 + kTileU;
  const int64_t b_first = r0 / bsz, b_last = min(nlb - 1, (r1 - 1) / bsz);
  int len = 0;
  for (int64_t bl = b_first; bl <= b_last; ++bl) {
    const int l = len_of(no_blocks ? -CUDART_INF_F : tbk[bl]);
    len = max(len, l);
    if (bl * bsz >= r0) pairs += cnt, pruned += cnt - l;
  }
  return len;
}

__device__ __forceinline__ void warp_count(bool pred, unsigned long long* ctr) {
  uint32_t bal = __ballot_sync(0xffffffffu, pred);
  if ((threadIdx.x & 31) == __ffs(bal | 0x80000000u) - 1 && bal) atomicAdd(ctr, (unsigned long long)__popc(bal));
}

// ---------------------------------------------------------------------------------------
// Filter error bound (SV Appendix D).  Users are scaled by 1/nu (nu ~ |u|),
// items and queries by a power of two, both rounded to fp16; products are exact in fp32;
// accumulation in fp32 (tensor core or FFMA).  For a = u/nu, b = p*2^e:
//   |fl(a_hat . b_hat) - a.b| <= c1 * |b| + c2
// c1 = 2^-10 (1 + 2^-9)            two fp16 roundings (2^-11 each) + fp32 pre-rounding of u/nu
//    + (dpad + 4) * 2^-22          fp32 accumulation (4x the sequential fp32 bound)
//    + 2^-25 sqrt(dpad)            fp16 subnormal absolute error of a, summed against |b|
//    + 2^-20                       every fp32 evaluation of lo/hi/threshold arithmetic
// c2 = 2^-24 sqrt(dpad)            fp16 subnormal absolute error of b, summed against |a| <= 1+
// The GPU test "filter_error_bound" measures the observed error against this bound.
inline double filter_c1(int dpad) {
  return std::ldexp(1.0, -10) * (1.0 + std::ldexp(1.0, -9)) + (dpad + 4) * std::ldexp(1.0, -22) +
         std::ldexp(1.0, -25) * std::sqrt((double)dpad) + std::ldexp(1.0, -20);
}
inline double filter_c2(int dpad) { return std::ldexp(1.0, -24) * std::sqrt((double)dpad); }

}  // namespace rmips

// ---------------------------------------------------------------------------------------
// The index (opaque to callers).
struct rmips_index_s {
  int64_t n = 0, m = 0;
  int64_t mprime = 0;       // items the top-k_max lists are built over: the first mprime of the
                            // norm-sorted P (Alg. 1 line 6); mprime = m is the exact index
  int d = 0, dpad = 0, kmax = 0, build_flags = 0;
  int ldh = 0;              // row stride of U16 / P16 / Q16 in halves: d rounded up to 16 (whole 32-byte
                            // sectors, so a row streams 2 ldh bytes; TMA boxes past it are zero-filled);
                            // dpad = d rounded up to 64 is the K-block geometry of the kernels
  int pd = 0;               // P32 row pitch in floats: d rounded up to 8 (whole 32-byte sectors)
  int device = 0;
  int64_t nblocks = 0;      // 128-user tiles (the kernels' work unit)
  int bsz = rmips::kTileU;  // users per Lemma-3 block (Eq. 1): one tile for the exact index, ceil(log2 n)
                            // for a P' index (the paper's O(log n))
  int64_t nlb = 0;          // Lemma-3 blocks, ceil(n / bsz)
  int64_t overflow_rows = 0;
  int64_t cand_total = 0;   // candidates kept by the build filter (sum over non-overflowed rows)
  int64_t tiles_done = 0;   // (128-user tile, item tile) contractions issued by the tensor-core build
  int build_kernel = 0;     // 0 SIMT, 1 k_build_tc, 2 k_build_tcq (A in TMEM), 3 k_build_tcq (A streamed)
  int cand_slots = 0;       // candidate slots per row of the build filter (128 or 256)
  float pscale = 1.f;       // items are scaled by 2^e before fp16 rounding
  double c1 = 0, c2 = 0;    // filter error constants (see common.cuh)

  // norm-sorted stores (Alg. 1 line 5)
  int32_t* perm_u = nullptr;   // [n] sorted position -> original user id
  int32_t* perm_p = nullptr;   // [m] sorted position -> original item id
  double* unorm = nullptr;     // [n] ||u|| fp64 (sorted order)
  float* unu = nullptr;        // [n] nu = fp32 scale used to unit-normalise the fp16 user rows
  double* pnorm = nullptr;     // [m] ||p|| fp64 (sorted order)
  float* perr = nullptr;       // [m] filter error bound of item p in scaled score units
  __half* U16 = nullptr;       // [n][ldh] fp16 u/nu (sorted)
  float* U32 = nullptr;        // [n][d] fp32 u (sorted) -- exact path
  __half* P16 = nullptr;       // [m][ldh] fp16 p*2^e (sorted)
  float* P32 = nullptr;        // [m][pd] fp32 p (sorted, zero-padded rows) -- exact path

  // exact lower-bound arrays (Def. 4), column-major by rank: x[j*n + u]
  double* tau = nullptr;       // [kmax][n] (j+1)-th largest u.p over P, fp64 (sorted users)
  int32_t* ids = nullptr;      // [kmax][n] original item id of that value
  float* thr = nullptr;        // [kmax][n] tau/nu in fp32 (filter threshold, unscaled)
  float* tb = nullptr;         // [kmax][nlb] Lemma 3: L^j(B) / ||u_first(B)||, rounded down

  void* arena = nullptr;       // the single allocation every array above lives in
  void* list_arena = nullptr;  // tau / ids / thr / tb after an in-place extension of k_max (NEXT-2)
  cudaStream_t last_stream = nullptr;  // stream of the last call (rmips_free_index frees on it)
  // query workspace (grown on demand)
  void* ws = nullptr;
  size_t ws_bytes = 0;
  size_t bits_off = 0, bits_len = 0;  // all-zero bit-matrix region of ws (query output)
  int64_t pair_cap = 0;
  unsigned long long* d_counters = nullptr;  // [kNumCounters + 4]
  int* d_flags = nullptr;                    // [4]
  rmips_stats_t stats{};
  double phase_ms[16] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
};
