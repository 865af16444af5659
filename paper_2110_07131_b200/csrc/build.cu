// build.cu -- index build (Alg. 1, with L_i over ALL of P per BASELINE north star).
//
//   B1 k_norms          norms (Alg. 1 lines 1-4) + finite check + max |p_j|
//   B2 cub radix sort   one norm sort of [items | users], descending, ties by ascending id (line 5,
//                       P:279; reading R6), split into the two permutations
//   B3 k_prep_*         permute; fp16 filter operands (u/nu, p*2^e); fp32 exact copies
//   B4 k_build_simt     SIMT contraction + candidate epilogue (the tcgen05 version is build_tc.cu)
//   B5 k_exact_select   fp64 re-evaluation of the candidates, exact top-k_max (lines 7-9)
//   B5' k_exact_row_full exact fallback for rows whose candidate buffer overflowed
//   B6 k_blocks         block table, Eq. (1) divided by ||u_first|| for Lemma 3
#include <cub/cub.cuh>

#include <mutex>
#include <vector>

#include "cand.cuh"
#include "common.cuh"
#include "internal.h"

namespace rmips {

// ------------------------------------------------------------------------------ B1
// keys[r] = bits of the fp64 norm (non-negative, so its bits order like the value) | topbit.
// A CTA stages its kNormRows rows in shared memory with coalesced loads (odd row stride: no bank
// conflicts), then each thread sums its own row left to right (the oracle's order).
constexpr int kNormRows = 128;
constexpr int kNormThreads = 512;  // all load (more bytes in flight); the first kNormRows sum the rows
__global__ void __launch_bounds__(kNormThreads)
k_norms(const float* __restrict__ X, int64_t rows, int d, uint64_t* __restrict__ keys,
        uint64_t topbit, int* __restrict__ flags, unsigned int* __restrict__ maxabs_bits, bool staged) {
  extern __shared__ float xs[];
  const int ds = d | 1;
  const int64_t r0 = blockIdx.x * (int64_t)kNormRows;
  const int nr = (int)(rows - r0 < kNormRows ? rows - r0 : kNormRows);
  const float* src = X + r0 * d;
  float mx = 0.f;
  bool fin = true;
  // the block's rows are one contiguous run of nr * d floats, 16-byte aligned when X is (r0 * d * 4 is
  // a multiple of 512): 16-byte loads, eight independent ones (128 bytes) in flight per thread (scalar
  // loads kept too few bytes in flight: 1.2 TB/s on configs[4])
  const int tot = nr * d;
  const float inv_d = 1.f / (float)d;  // row of element e: floor((e + 0.5) / d), exact for e < 2^17, d <= 1024
  auto take = [&](int e, float v) {
    fin &= isfinite(v);
    mx = fmaxf(mx, fabsf(v));
    if (staged) {
      const int rr = __float2int_rz(((float)e + 0.5f) * inv_d);
      xs[rr * ds + (e - rr * d)] = v;
    }
  };
  // (a caller's view may start anywhere: unaligned X takes the scalar tail loop for every element)
  const int n4 = (reinterpret_cast<uintptr_t>(X) & 15u) == 0 ? tot >> 2 : 0;
  const float4* src4 = reinterpret_cast<const float4*>(src);
  for (int i0 = threadIdx.x; i0 < n4; i0 += 8 * kNormThreads) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * kNormThreads;
      v[u] = i < n4 ? __ldg(src4 + i) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * kNormThreads;
      if (i < n4) {
        take(4 * i, v[u].x);
        take(4 * i + 1, v[u].y);
        take(4 * i + 2, v[u].z);
        take(4 * i + 3, v[u].w);
      }
    }
  }
  for (int e = 4 * n4 + threadIdx.x; e < tot; e += kNormThreads) take(e, __ldg(src + e));  // (tot % 4 tail, unaligned X)
  __syncthreads();
  if (threadIdx.x < nr) {
    double s = 0.0;
    if (staged) {  // (a shared-memory pointer of its own: LDS, not generic loads)
      const float* x = xs + threadIdx.x * ds;
#pragma unroll 8
      for (int j = 0; j < d; ++j) s = __fma_rn((double)x[j], (double)x[j], s);
    } else {  // d > 400: the 128 rows do not fit in shared memory; each thread re-reads its row (L2)
      const float* x = src + (int64_t)threadIdx.x * d;
      for (int j = 0; j < d; ++j) s = __fma_rn((double)__ldg(x + j), (double)__ldg(x + j), s);
    }
    keys[r0 + threadIdx.x] = (uint64_t)__double_as_longlong(sqrt(s)) | topbit;
  }
  if (__any_sync(0xffffffffu, !fin) && (threadIdx.x & 31) == 0) atomicOr(flags, kFlagNonfinite);
  if (maxabs_bits) {
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0 && isfinite(mx)) atomicMax(maxabs_bits, __float_as_uint(mx));
  }
}

__global__ void k_iota(int32_t* v, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = (int32_t)i;
}

// Split the one sorted [items | users] sequence into the two norm-sorted permutations (and the
// inverse user permutation for the user prep).
__global__ void k_split_sorted(const uint64_t* __restrict__ keys, const int32_t* __restrict__ vals, int64_t m,
                               int64_t n, double* __restrict__ pnorm, int32_t* __restrict__ perm_p,
                               double* __restrict__ unorm, int32_t* __restrict__ perm_u, int32_t* __restrict__ inv_u) {
  int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= m + n) return;
  const double v = __longlong_as_double((long long)(keys[r] & 0x7fffffffffffffffull));
  if (r < m) {
    pnorm[r] = v, perm_p[r] = vals[r];
  } else {
    const int32_t o = vals[r] - (int32_t)m;
    unorm[r - m] = v, perm_u[r - m] = o;
    inv_u[o] = (int32_t)(r - m);
  }
}

// ------------------------------------------------------------------------------ B3
// Users: U16 = fp16(u / nu), nu = fp32(||u||) (1 for the zero vector); U32 = u (permuted).
// One warp per kPrepRows consecutive ORIGINAL rows: the reads of Q stream in order and each row is
// written to its norm-sorted place (whole 128-byte U16 rows; a row-gather version left the reads
// scattered: 0.68 / 0.52 ms on configs[3]); lane l handles the column pairs 2l, 2l + 64, ...
// keys_u[o] = bits of ||u_o|| (the sort's input keys: the same fp64 value as the sorted norms).
constexpr int kPrepRows = 8;
__global__ void k_prep_users(const float* __restrict__ Q, int64_t n, int d, int ldh,
                             const int32_t* __restrict__ inv_u, const uint64_t* __restrict__ keys_u,
                             __half* __restrict__ U16, float* __restrict__ U32, float* __restrict__ unu) {
  const int64_t o0 = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * kPrepRows;
  const int lane = threadIdx.x & 31;
  if (o0 >= n) return;
  int64_t r_l = 0;
  float nu_l = 1.f;
  if (lane < kPrepRows && o0 + lane < n) {
    r_l = inv_u[o0 + lane];
    nu_l = (float)__longlong_as_double((long long)keys_u[o0 + lane]);
    // the zero vector: nu = 1.  A norm above FLT_MAX has no fp32 nu that makes u/nu unit-norm (the
    // precondition of the filter bound): nu = NaN makes the row's filter scores and thresholds NaN,
    // so the build sends the row to the exact fallback (too few candidates) and every query pair
    // of the user to the exact path (NaN never classifies)
    if (isinf(nu_l)) nu_l = __int_as_float(0x7fc00000);
    else if (!(nu_l > 0.f)) nu_l = 1.f;
    unu[r_l] = nu_l;
  }
  for (int j = 2 * lane; j < ldh; j += 64) {
    float x0[kPrepRows], x1[kPrepRows];
#pragma unroll
    for (int i = 0; i < kPrepRows; ++i) {
      const float* q = Q + (o0 + i) * d;
      const bool live = o0 + i < n;
      x0[i] = live && j < d ? q[j] : 0.f;
      x1[i] = live && j + 1 < d ? q[j + 1] : 0.f;
    }
#pragma unroll
    for (int i = 0; i < kPrepRows; ++i) {
      const float nu = __shfl_sync(0xffffffffu, nu_l, i);
      const int64_t r = __shfl_sync(0xffffffffu, r_l, i);
      if (o0 + i < n) {
        reinterpret_cast<__half2*>(U16 + r * ldh)[j >> 1] =
            __halves2half2(__float2half_rn(x0[i] / nu), __float2half_rn(x1[i] / nu));
        if (j < d) U32[r * d + j] = x0[i];
        if (j + 1 < d) U32[r * d + j + 1] = x1[i];
      }
    }
  }
}

// Items: P16 = fp16(p * 2^e) with max|p*2^e| < 2^14; perr = filter error bound (scaled units).
// One warp per row as above; P32 is zero-padded to pd (a multiple of 8, <= ldh).
__global__ void k_prep_items(const float* __restrict__ P, int64_t m, int d, int ldh, int pd,
                             const int32_t* __restrict__ perm, const double* __restrict__ norm_sorted,
                             const unsigned int* __restrict__ maxabs_bits, double c1, double c2,
                             __half* __restrict__ P16, float* __restrict__ P32, float* __restrict__ perr,
                             float* __restrict__ scale_out) {
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= m) return;
  const float mx = __uint_as_float(*maxabs_bits);
  int ex = 0;
  if (mx > 0.f) frexpf(mx, &ex);               // mx < 2^ex
  int e = 14 - ex;
  e = max(-126, min(126, e));
  const float scale = ldexpf(1.f, e);
  const int64_t o = perm[r];
  const float* p = P + o * d;
#pragma unroll 4
  for (int j = 2 * lane; j < ldh; j += 64) {
    const float x0 = j < d ? p[j] : 0.f, x1 = j + 1 < d ? p[j + 1] : 0.f;
    reinterpret_cast<__half2*>(P16 + r * ldh)[j >> 1] = __halves2half2(__float2half_rn(x0 * scale), __float2half_rn(x1 * scale));
    if (j < pd) P32[r * pd + j] = x0;
    if (j + 1 < pd) P32[r * pd + j + 1] = x1;
  }
  if (lane == 0) {
    const double b = norm_sorted[r] * (double)scale;
    perr[r] = __double2float_ru((c1 * b + c2) * (1.0 + 1e-6));
    if (r == 0) *scale_out = scale;
  }
}

// ------------------------------------------------------------------------------ B4 (SIMT)
// One thread per user row; 128 rows per CTA; items streamed through smem 32 at a time.
// Scores use the same fp16 operands and fp32 accumulation as the tensor-core kernel, so the
// same error bound applies.  Correctness path and the RMIPS_BUILD_SIMT option.
template <int DPAD>
__global__ void __launch_bounds__(128, 1)
k_build_simt(const __half* __restrict__ U16, const __half* __restrict__ P16, const float* __restrict__ perr,
             int ldh, int64_t n, int64_t m, int kmax, int32_t* __restrict__ cand, int32_t* __restrict__ ccount,
             int32_t* __restrict__ ovf_list, int* __restrict__ ovf_count) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const CandSmem sm = CandSmem::at(smem_raw);                               // candidate buffers
  __half2* us = reinterpret_cast<__half2*>(smem_raw + kCandSmemBytes);     // [DPAD/2][128]
  __half* ps = reinterpret_cast<__half*>(us + (DPAD / 2) * 128);   // [DPAD][32] (fp16: exact copies of P16)

  const int tid = threadIdx.x;
  const int64_t row = blockIdx.x * (int64_t)128 + tid;
  const bool live = row < n;
  // stage this CTA's 128 user rows, transposed, as half2 pairs
  for (int i = tid; i < 128 * (DPAD / 2); i += 128) {
    int r = i / (DPAD / 2), k2 = i % (DPAD / 2);
    int64_t gr = blockIdx.x * (int64_t)128 + r;
    __half2 v = __floats2half2_rn(0.f, 0.f);
    if (gr < n && 2 * k2 < ldh) v = reinterpret_cast<const __half2*>(U16)[gr * (ldh / 2) + k2];
    us[k2 * 128 + r] = v;
  }
  CandRow me = cand_init(live);
  const float e0x2 = cand_e0x2(perr);

  for (int64_t base = 0; base < m; base += 32) {
    __syncthreads();
    for (int i = tid; i < 32 * DPAD; i += 128) {
      int jj = i / DPAD, k = i % DPAD;
      __half v = __float2half_rn(0.f);
      if (base + jj < m && k < ldh) v = P16[(base + jj) * ldh + k];
      ps[k * 32 + jj] = v;
    }
    __syncthreads();
    float s[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) s[j] = 0.f;
#pragma unroll 2
    for (int k2 = 0; k2 < DPAD / 2; ++k2) {
      float2 a = __half22float2(us[k2 * 128 + tid]);
      const __half2* p0 = reinterpret_cast<const __half2*>(ps + (2 * k2) * 32);
      const __half2* p1 = reinterpret_cast<const __half2*>(ps + (2 * k2 + 1) * 32);
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const float2 b0 = __half22float2(p0[q]), b1 = __half22float2(p1[q]);
        s[2 * q + 0] = fmaf(a.x, b0.x, s[2 * q + 0]);
        s[2 * q + 1] = fmaf(a.x, b0.y, s[2 * q + 1]);
        s[2 * q + 0] = fmaf(a.y, b1.x, s[2 * q + 0]);
        s[2 * q + 1] = fmaf(a.y, b1.y, s[2 * q + 1]);
      }
    }
    const float NEG = -__int_as_float(0x7f800000);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (base + j >= m) s[j] = NEG;
    float E = __ldg(perr + base);
    cand_chunk([&](int j) { return s[j]; }, E, (int)base, me, sm, tid, e0x2, kmax);
  }
  cand_finish(me, sm, tid, e0x2, kmax, m, row, n, cand, kCand, ccount, ovf_list, ovf_count);
}

// ------------------------------------------------------------------------------ B5
// Warp per user row (grid-stride): exact fp64 value of every candidate (dot64 order, DESIGN.md
// R7), then the k_max largest by (value desc, original item id asc) with a warp bitonic sort,
// written to the column-major tables.  Candidate item rows are staged in shared memory 32 at a
// time with coalesced loads (the rows are scattered in P32), then each lane runs the sequential
// fp64 sum of its own candidate from shared memory.
struct SelKey {
  double v;
  int id;
};
// (value desc, id asc); non-short-circuit operators keep it branch-free (predicate logic only)
__device__ __forceinline__ bool sel_better(const SelKey& a, const SelKey& b) {
  return (a.v > b.v) | ((a.v == b.v) & (a.id < b.id));
}
__device__ __forceinline__ SelKey shfl_xor_key(const SelKey& k, int m) {
  SelKey r;
  r.v = __shfl_xor_sync(0xffffffffu, k.v, m);
  r.id = __shfl_xor_sync(0xffffffffu, k.id, m);
  return r;
}

// Bitonic sort of 32*E keys held striped (element e = i*32 + lane in key[i]), best first.
template <int E>
__device__ __forceinline__ void warp_bitonic(SelKey (&key)[E]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {  // partner in the same lane, register i ^ (j / 32)
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int ip = i ^ (j >> 5);
          if (ip > i) {
            const int e = i * 32 + lane;
            const bool up = (e & k) == 0;  // this k-block sorts best-first
            const bool ob = sel_better(key[ip], key[i]), mb = sel_better(key[i], key[ip]);
            const bool sw = up ? ob : mb;
            const SelKey a = key[i], b = key[ip];
            key[i].v = sw ? b.v : a.v;
            key[i].id = sw ? b.id : a.id;
            key[ip].v = sw ? a.v : b.v;
            key[ip].id = sw ? a.id : b.id;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int e = i * 32 + lane;
          const SelKey o = shfl_xor_key(key[i], j);
          const bool up = (e & k) == 0;
          const bool lower = (e & j) == 0;  // this element sits at the lower index of the pair
          // the lower index keeps the better key when sorting best-first, the worse otherwise
          const bool ob = sel_better(o, key[i]), mb = sel_better(key[i], o);
          const bool take = (lower == up) ? ob : mb;
          key[i].v = take ? o.v : key[i].v;
          key[i].id = take ? o.id : key[i].id;
        }
      }
    }
  }
}

// Fast path of the same sort: the value alone as an order-preserving 64-bit integer (larger key =
// larger value; dot64 never returns -0, so key equality is value equality) with the id carried
// along.  One unsigned compare and three selects per compare-exchange instead of the two-field
// comparator.  Ties in value are left in an unspecified id order, so the caller checks the sorted
// run for adjacent equal keys and re-sorts with warp_bitonic when it finds one.
__device__ __forceinline__ uint64_t sel_okey(double v) {
  const uint64_t b = (uint64_t)__double_as_longlong(v);
  return b ^ ((b >> 63) ? ~0ull : (1ull << 63));
}
__device__ __forceinline__ double sel_oval(uint64_t k) {
  return __longlong_as_double((long long)(k ^ ((k >> 63) ? (1ull << 63) : ~0ull)));
}
template <int E>
__device__ __forceinline__ void warp_bitonic_u64(uint64_t (&key)[E], int (&id)[E]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32) {
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const int ip = i ^ (j >> 5);
          if (ip > i) {
            const bool up = ((i * 32 + lane) & k) == 0;
            const bool sw = up == (key[ip] > key[i]);
            const uint64_t a = key[i], b = key[ip];
            const int ia = id[i], ib = id[ip];
            key[i] = sw ? b : a;
            key[ip] = sw ? a : b;
            id[i] = sw ? ib : ia;
            id[ip] = sw ? ia : ib;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) {
          const uint64_t o = __shfl_xor_sync(0xffffffffu, key[i], j);
          const int oi = __shfl_xor_sync(0xffffffffu, id[i], j);
          // keep the larger key at the lower index of an ascending-best block, the smaller otherwise
          // (equal keys: the two lanes of a pair may both take, duplicating one id; the caller's
          // tie check then re-sorts from its own copy of the unsorted keys)
          const bool keep_big = ((((i * 32 + lane) & k) == 0) == ((lane & j) == 0));
          const bool take = keep_big == (o > key[i]);
          key[i] = take ? o : key[i];
          id[i] = take ? oi : id[i];
        }
      }
    }
  }
}

// Sort the first E*32 keys of key[] best first: the integer fast path, then (only when two real
// keys share a value) the two-field comparator from the unsorted copy.
template <int E, int NK>
__device__ __forceinline__ void sel_sort(SelKey (&key)[NK], int cnt) {
  const int lane = threadIdx.x & 31;
  uint64_t k[E];
  int id[E];
#pragma unroll
  for (int i = 0; i < E; ++i) k[i] = sel_okey(key[i].v), id[i] = key[i].id;
  warp_bitonic_u64<E>(k, id);
  bool tie = false;
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const uint64_t dn = __shfl_down_sync(0xffffffffu, k[i], 1);
    uint64_t nx = dn;
    if (i + 1 < E) {
      const uint64_t w0 = __shfl_sync(0xffffffffu, k[i + 1 < E ? i + 1 : i], 0);
      if (lane == 31) nx = w0;
    }
    tie |= (i * 32 + lane + 1 < cnt) & (nx == k[i]);
  }
  if (__any_sync(0xffffffffu, tie)) {
    SelKey kk[E];
#pragma unroll
    for (int i = 0; i < E; ++i) kk[i] = key[i];
    warp_bitonic<E>(kk);
#pragma unroll
    for (int i = 0; i < E; ++i) key[i] = kk[i];
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) key[i].v = sel_oval(k[i]), key[i].id = id[i];
  }
}

// Filter threshold of a finite list value: fp32(tau / nu).  When that is not a finite fp32 (|tau / nu|
// above FLT_MAX, or nu = NaN for a user whose norm exceeds FLT_MAX) it is NaN, which the query filter
// never rejects or accepts against (every comparison is false): the pair goes to the exact path.
// (An infinite threshold would wrongly accept (-inf) or reject (+inf) outright.)  -inf list padding
// (k > m) keeps -inf: fewer than k items exist, so every user is in the set.
__device__ __forceinline__ float thr_of(double v, float nu) {
  const float t = (float)(v / (double)nu);
  return isfinite(t) ? t : __int_as_float(0x7fc00000);
}

// 256-bit read-only global load (LDG.256; the address is 32-byte aligned)
__device__ __forceinline__ void ldg_nc_v8(const float* p, float (&v)[8]) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

#ifndef RMIPS_SEL_WARPS
#define RMIPS_SEL_WARPS 8
#endif
#ifndef RMIPS_SEL_ROWS
#define RMIPS_SEL_ROWS 32
#endif
constexpr int kSelWarps = RMIPS_SEL_WARPS;
constexpr int kSelRows = RMIPS_SEL_ROWS;  // rows per CTA block: each rank's outputs are written as one coalesced run
constexpr int kSelStride = kSelRows + 1;  // odd stage stride: a warp's 32 ranks of one row hit 32 banks
// One CTA per block of kSelRows consecutive rows (warp w takes rows w, w + 8, ...); a warp
// evaluates one row at a time: one candidate per lane per round (16-byte loads of the
// sector-padded item row; the zero padding adds fma(0, 0, s) = s exactly, s never -0), then a
// bitonic sort (value desc, original id asc).  The sorted lists are staged in shared memory
// [rank][row] and written per rank as one contiguous run of the block's rows: the column-major
// tables (tau, ids, thr: rank-major, users contiguous) then take full sectors instead of one
// 4- or 8-byte piece of a sector per (row, rank).
// MAXC = candidate slots per row (the build's cstride: 128, or 256 for k_max > 80).
// Occupancy: the kernel is bound by L1 wavefronts and L2 latency of the row gathers, so resident warps
// matter more than a few spilled registers: 4 CTAs per SM (64 registers, 104 bytes of spill) for
// 128 slots, 3 for 256.  Measured against the unconstrained 114 registers (2 CTAs per SM): configs[3]
// 4.82 -> 2.97 ms, configs[4] 11.0 -> 9.1 ms, configs[1] 0.378 -> 0.292 ms (same box; a
// preloaded-rows variant, every 256-bit load of a row issued before its chain, was 15 % slower).
template <int MAXC>
__global__ void __launch_bounds__(32 * kSelWarps, MAXC == 128 ? 4 : 3)
k_exact_select(const float* __restrict__ U32, const float* __restrict__ P32, const int32_t* __restrict__ perm_p,
               const float* __restrict__ unu, const int32_t* __restrict__ cand, const int32_t* __restrict__ ccount,
               int64_t n, int d, int pd, int kmax, double* __restrict__ tau, int32_t* __restrict__ ids,
               float* __restrict__ thr, unsigned long long* __restrict__ cand_total) {
  // shared: per warp the user row [pd] (fp64, zero-padded); the block's staged lists
  extern __shared__ __align__(16) double ssel[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int NK = MAXC / 32;                  // candidate keys per lane
  const int kc = kmax < MAXC ? kmax : MAXC;      // ranks staged (beyond MAXC: -inf, only when m < k_max)
  double* urow = ssel + (size_t)w * pd;
  double* stau = ssel + (size_t)kSelWarps * pd;                    // [kc][kSelStride]
  int32_t* sids = reinterpret_cast<int32_t*>(stau + (size_t)kc * kSelStride);
  float* sthr = reinterpret_cast<float*>(sids + (size_t)kc * kSelStride);
  unsigned long long my_total = 0;
  const int64_t nblk = (n + kSelRows - 1) / kSelRows;
  constexpr int kPer = kSelRows / kSelWarps;  // rows per warp per block
  // the next row's count, first two rounds of candidate positions and user values are loaded one
  // row ahead (the chain count -> positions -> item rows is otherwise three dependent latencies)
  auto row_of = [&](int64_t q) {  // q-th row of this warp: block blockIdx.x + (q / kPer) gridDim.x
    const int64_t b = blockIdx.x + (q / kPer) * (int64_t)gridDim.x;
    return b * kSelRows + w + kSelWarps * (int)(q % kPer);
  };
  int cnt_n = -1, pn0 = 0, pn1 = 0;
  float un[8];
  auto prefetch = [&](int64_t r) {
    cnt_n = -1;
    if (r < n) {
      cnt_n = ccount[r];
      pn0 = cand[r * MAXC + lane];
      pn1 = cand[r * MAXC + 32 + lane];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int t = lane + 32 * i;
        un[i] = t < d ? U32[r * d + t] : 0.f;
      }
    }
  };
  int64_t q = 0;
  prefetch(row_of(0));
  for (int64_t b = blockIdx.x; b < nblk; b += gridDim.x) {
    for (int j = 0; j < kPer; ++j, ++q) {
      const int64_t row = row_of(q);
      const int rloc = w + kSelWarps * j;
      const int cnt = cnt_n, pc0 = pn0, pc1 = pn1;
      float uc[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) uc[i] = un[i];
      prefetch(row_of(q + 1));
      if (row >= n) continue;
      if (cnt < 0) {  // overflowed: k_exact_row_full rewrites the row after this kernel
        for (int r = lane; r < kc; r += 32) stau[r * kSelStride + rloc] = -CUDART_INF, sids[r * kSelStride + rloc] = -1,
                                            sthr[r * kSelStride + rloc] = -CUDART_INF_F;
        continue;
      }
      my_total += cnt;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int t = lane + 32 * i;
        if (t < pd) urow[t] = (double)uc[i];  // zero padding for d <= t < pd
      }
      for (int t = 256 + lane; t < pd; t += 32) urow[t] = t < d ? (double)U32[row * d + t] : 0.0;  // d > 256
      __syncwarp();
      SelKey key[NK];
#pragma unroll
      for (int i = 0; i < NK; ++i) key[i].v = -CUDART_INF, key[i].id = 0x7fffffff;
      // candidates c and c + 32 of a lane as two interleaved chains (twice the loads in flight)
#pragma unroll
      for (int i = 0; i < NK; i += 2) {
        if (32 * i >= cnt) break;  // warp-uniform
        const int c0 = 32 * i + lane, c1 = c0 + 32;
        const bool l0 = c0 < cnt, l1 = c1 < cnt;
        int pos0 = 0, pos1 = 0;  // inactive lanes read item row 0 and discard it
        if (l0) pos0 = i == 0 ? pc0 : cand[row * MAXC + c0];
        if (l1) pos1 = i == 0 ? pc1 : cand[row * MAXC + c1];
        const float* pr0 = P32 + (int64_t)pos0 * pd;  // pd = round_up(d, 8): 32-byte rows
        const float* pr1 = P32 + (int64_t)pos1 * pd;
        double s0 = 0.0, s1 = 0.0;  // dot64: left-to-right fp64 sums of exact fp32 x fp32 products
        if (32 * i + 32 < cnt) {    // warp-uniform: both chains have work
#pragma unroll 2
          for (int t = 0; t < pd; t += 8) {
            float a[8], bb[8];
            ldg_nc_v8(pr0 + t, a);
            if (l1) {
              ldg_nc_v8(pr1 + t, bb);
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) bb[e] = 0.f;
            }
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const double2 uu = *reinterpret_cast<const double2*>(urow + t + e);
              s0 = __fma_rn((double)a[e], uu.x, s0);
              s1 = __fma_rn((double)bb[e], uu.x, s1);
              s0 = __fma_rn((double)a[e + 1], uu.y, s0);
              s1 = __fma_rn((double)bb[e + 1], uu.y, s1);
            }
          }
        } else {                    // one chain (rows with at most 32 * i + 32 candidates)
#pragma unroll 2
          for (int t = 0; t < pd; t += 8) {
            float a[8];
            if (l0) {
              ldg_nc_v8(pr0 + t, a);
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e) a[e] = 0.f;
            }
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
              const double2 uu = *reinterpret_cast<const double2*>(urow + t + e);
              s0 = __fma_rn((double)a[e], uu.x, s0);
              s0 = __fma_rn((double)a[e + 1], uu.y, s0);
            }
          }
        }
        if (l0) key[i].v = s0, key[i].id = perm_p[pos0];
        if (l1) key[i + 1].v = s1, key[i + 1].id = perm_p[pos1];
      }
      if (cnt <= 32) {  // one key per lane: 15 compare-exchange steps instead of 21 (64) or 28 (128)
        sel_sort<1, NK>(key, cnt);
      } else if (cnt <= 64) {
        sel_sort<2, NK>(key, cnt);
      } else if (NK == 4 || cnt <= 128) {
        sel_sort<4, NK>(key, cnt);
      } else {
        sel_sort<(NK > 4 ? NK : 4), NK>(key, cnt);
      }
      const float nu = unu[row];
#pragma unroll
      for (int i = 0; i < NK; ++i) {
        const int rank = i * 32 + lane;
        if (rank < kc) {
          const bool ok = rank < cnt;
          stau[rank * kSelStride + rloc] = ok ? key[i].v : -CUDART_INF;
          sids[rank * kSelStride + rloc] = ok ? key[i].id : -1;
          sthr[rank * kSelStride + rloc] = ok ? thr_of(key[i].v, nu) : -CUDART_INF_F;
        }
      }
    }
    __syncthreads();  // the block's lists are staged: one coalesced run per rank
    const int64_t r0 = b * kSelRows;
    const int nr = (int)(n - r0 < kSelRows ? n - r0 : kSelRows);
    for (int e = threadIdx.x; e < kmax * kSelRows; e += blockDim.x) {
      const int rank = e / kSelRows, r = e % kSelRows;
      if (r >= nr) continue;
      const bool st = rank < kc;
      tau[(int64_t)rank * n + r0 + r] = st ? stau[rank * kSelStride + r] : -CUDART_INF;
      ids[(int64_t)rank * n + r0 + r] = st ? sids[rank * kSelStride + r] : -1;
      thr[(int64_t)rank * n + r0 + r] = st ? sthr[rank * kSelStride + r] : -CUDART_INF_F;
    }
    __syncthreads();  // before the next block's lists overwrite the stage
  }
  if (lane == 0 && my_total) atomicAdd(cand_total, my_total);
}

// B5': exact top-k_max of a whole row (fp64 over all of P), for overflowed rows.  One CTA per
// listed row; scratch holds the m exact values; k_max rounds of a block argmax in the order
// (value desc, original id asc).  Slow, simple, rare (massive ties / duplicate items).
__global__ void __launch_bounds__(256)
k_exact_row_full(const float* __restrict__ U32, const float* __restrict__ P32, const int32_t* __restrict__ perm_p,
                 const float* __restrict__ unu, const int32_t* __restrict__ ovf_list, const int* __restrict__ ovf_count,
                 int64_t n, int64_t m, int d, int pd, int kmax, double* __restrict__ scratch, double* __restrict__ tau,
                 int32_t* __restrict__ ids, float* __restrict__ thr) {
  __shared__ double bv[256];
  __shared__ int bo[256];
  __shared__ int64_t bp[256];
  const int nrows = *ovf_count;
  double* sc = scratch + blockIdx.x * m;
  for (int t = blockIdx.x; t < nrows; t += gridDim.x) {
    const int64_t row = ovf_list[t];
    const float* u = U32 + row * d;
    for (int64_t j = threadIdx.x; j < m; j += blockDim.x) sc[j] = dot64(u, P32 + j * pd, d);
    __syncthreads();
    double pv = CUDART_INF;
    int po = -1;
    const float nu = unu[row];
    for (int r = 0; r < kmax; ++r) {
      double best = -CUDART_INF;
      int bestid = 0x7fffffff;
      int64_t bestpos = -1;
      for (int64_t j = threadIdx.x; j < m; j += blockDim.x) {
        double v = sc[j];
        int o = perm_p[j];
        bool after = (v < pv) || (v == pv && o > po);  // strictly after the previous pick
        bool better = (v > best) || (v == best && o < bestid);
        if (after && better) { best = v; bestid = o; bestpos = j; }
      }
      bv[threadIdx.x] = best; bo[threadIdx.x] = bestid; bp[threadIdx.x] = bestpos;
      __syncthreads();
      for (int s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s) {
          double v2 = bv[threadIdx.x + s];
          int o2 = bo[threadIdx.x + s];
          if (bp[threadIdx.x + s] >= 0 &&
              (bp[threadIdx.x] < 0 || v2 > bv[threadIdx.x] || (v2 == bv[threadIdx.x] && o2 < bo[threadIdx.x]))) {
            bv[threadIdx.x] = v2; bo[threadIdx.x] = o2; bp[threadIdx.x] = bp[threadIdx.x + s];
          }
        }
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        bool ok = bp[0] >= 0;
        tau[(int64_t)r * n + row] = ok ? bv[0] : -CUDART_INF;
        ids[(int64_t)r * n + row] = ok ? bo[0] : -1;
        thr[(int64_t)r * n + row] = ok ? thr_of(bv[0], nu) : -CUDART_INF_F;
      }
      pv = bv[0];
      po = bo[0];
      bool ok = bp[0] >= 0;
      __syncthreads();
      if (!ok) pv = -CUDART_INF, po = 0x7fffffff;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------ B6
// tb[j][B] = L^j(B) / ||u_first(B)|| rounded down, L^j(B) = min over members tau_j (Eq. 1).
// Lemma 3 (strict form R1) keeps query q for block B iff ||q|| >= tb (q norm
// rounded up); the queries of a batch are norm-sorted, so the kept ones are a prefix.
// One warp per (block B, rank j): the block's kTileU values of column j are read coalesced (lane
// r reads rows lo + r, lo + r + 32, ...) and min-reduced.
__global__ void k_blocks(const double* __restrict__ tau, const double* __restrict__ unorm, int64_t n, int kmax,
                         int64_t nblocks, int bsz, float* __restrict__ tb) {
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= nblocks * kmax) return;
  const int64_t B = wid % nblocks;
  const int j = (int)(wid / nblocks);
  const int64_t lo = B * bsz, hi = min(n, lo + bsz);
  double L = CUDART_INF;
  for (int64_t i = lo + lane; i < hi; i += 32) L = fmin(L, tau[(int64_t)j * n + i]);
#pragma unroll
  for (int o = 16; o; o >>= 1) L = fmin(L, __shfl_xor_sync(0xffffffffu, L, o));
  if (lane == 0) {
    const double uf = unorm[lo];
    float t;
    if (!(L > 0.0)) t = -CUDART_INF_F;           // L <= 0 (or -inf): ||u|| ||q|| >= 0 >= L, prune nothing
    else if (uf == 0.0) t = CUDART_INF_F;        // all members are zero vectors: u.q = 0 < L
    else t = __double2float_rd((L / uf) * (1.0 - 1e-12));
    tb[(int64_t)j * nblocks + B] = t;
  }
}

// ------------------------------------------------------------------------------ host driver
static inline unsigned nblk(int64_t work, int t) { return (unsigned)((work + t - 1) / t); }

template <int DPAD>
static cudaError_t launch_build_simt(const BuildCtx& c, cudaStream_t st) {
  size_t smem = (size_t)kCandSmemBytes + (DPAD / 2) * 128 * 4 + DPAD * 32 * 2;
  cudaError_t e = set_smem_attr((const void*)k_build_simt<DPAD>, (int)smem);
  if (e != cudaSuccess) return e;
  k_build_simt<DPAD><<<nblk(c.idx->n, 128), 128, smem, st>>>(c.idx->U16, c.idx->P16, c.idx->perr, c.idx->ldh, c.idx->n,
                                                             c.mb, c.idx->kmax, c.cand, c.ccount,
                                                             c.ovf_list, c.ovf_count); count_launch();
  return cudaGetLastError();
}

cudaError_t build_simt(const BuildCtx& c, cudaStream_t st) {
  c.idx->build_kernel = 0;
  c.idx->cand_slots = kCand;
  switch (c.idx->dpad) {
    case 64: return launch_build_simt<64>(c, st);
    case 128: return launch_build_simt<128>(c, st);
    case 192: return launch_build_simt<192>(c, st);
    case 256: return launch_build_simt<256>(c, st);
    default: return cudaErrorInvalidValue;
  }
}

// B2 as a CUDA graph: the radix sort is ~20 small launches and memsets whose host enqueue time
// (~5 us each) exceeds their device time, so the GPU idles through the prep phase.  The iota +
// sort sequence is captured once per (stream, size) — when that size is built a second time —
// into a graph over persistent buffers and replayed with one launch.  Buffers are stream-ordered: builds on one stream reuse them in
// order; different streams get different entries.  At most kSortCache entries (the oldest is
// freed with cudaFree, which waits for the device).
namespace {
struct SortGraph {
  cudaStream_t st = nullptr;
  int dev = -1;
  int64_t tot = 0;
  uint64_t* keys = nullptr;  // [2 tot]: in, out
  int32_t* vals = nullptr;   // [2 tot]: in, out
  void* tmp = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaEvent_t done = nullptr;  // recorded after the last read of keys / vals by the previous build
  bool used = false;           // done has been recorded at least once
  int busy = 0;  // host threads between sort_graph_get and sort_graph_put (never evicted then)
};
constexpr int kSortCache = 4;
std::mutex g_sort_mu;
std::vector<SortGraph*> g_sort;
// (stream, size, device) of recent builds: a graph is captured only when a size repeats, so
// one-off sizes do not pay the capture (they take the direct path)
struct SortSeen {
  cudaStream_t st;
  int64_t tot;
  int dev;
};
std::vector<SortSeen> g_sort_seen;
void sort_graph_free(SortGraph* g) {
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->done) cudaEventDestroy(g->done);
  cudaFree(g->keys);
  cudaFree(g->vals);
  cudaFree(g->tmp);
  delete g;
}
SortGraph* sort_graph_get(cudaStream_t st, int64_t tot) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_sort_mu);
  for (size_t i = 0; i < g_sort.size(); ++i)
    if (g_sort[i]->st == st && g_sort[i]->tot == tot && g_sort[i]->dev == dev) {
      SortGraph* g = g_sort[i];
      // another host thread is enqueueing on these buffers right now (same stream handle: the
      // legacy NULL stream, or cudaStreamPerThread, which is a different stream per thread): take
      // the direct path with this build's own scratch instead
      if (g->busy) return nullptr;
      g_sort.erase(g_sort.begin() + i);
      g_sort.push_back(g);  // most recently used last
      ++g->busy;
      return g;
    }
  bool seen = false;
  for (const SortSeen& s : g_sort_seen) seen |= s.st == st && s.tot == tot && s.dev == dev;
  if (!seen) {
    if (g_sort_seen.size() >= 16) g_sort_seen.erase(g_sort_seen.begin());
    g_sort_seen.push_back(SortSeen{st, tot, dev});
    return nullptr;
  }
  SortGraph* g = new SortGraph;
  g->st = st; g->dev = dev; g->tot = tot;
  size_t tb = 0;
  cudaStream_t cs = nullptr;
  cudaGraph_t graph = nullptr;
  bool ok = cub::DeviceRadixSort::SortPairsDescending((void*)nullptr, tb, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                                      (const int32_t*)nullptr, (int32_t*)nullptr, (int)tot, 0, 64) ==
                cudaSuccess &&
            cudaMalloc(&g->keys, 2 * tot * sizeof(uint64_t)) == cudaSuccess &&
            cudaMalloc(&g->vals, 2 * tot * sizeof(int32_t)) == cudaSuccess && cudaMalloc(&g->tmp, tb) == cudaSuccess &&
            cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming) == cudaSuccess &&
            cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    k_iota<<<(unsigned)((tot + 255) / 256), 256, 0, cs>>>(g->vals, tot);
    size_t tb2 = tb;
    cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(g->tmp, tb2, g->keys, g->keys + tot, g->vals,
                                                              g->vals + tot, (int)tot, 0, 64, cs);
    ok = cudaStreamEndCapture(cs, &graph) == cudaSuccess && e == cudaSuccess &&
         cudaGraphInstantiate(&g->exec, graph, 0) == cudaSuccess;
  }
  if (graph) cudaGraphDestroy(graph);
  if (cs) cudaStreamDestroy(cs);
  if (!ok) {
    cudaGetLastError();
    sort_graph_free(g);
    return nullptr;
  }
  if ((int)g_sort.size() >= kSortCache) {
    size_t i = 0;
    while (i < g_sort.size() && g_sort[i]->busy) ++i;
    if (i == g_sort.size()) {  // every entry is being enqueued right now: do not cache
      sort_graph_free(g);
      return nullptr;
    }
    sort_graph_free(g_sort[i]);
    g_sort.erase(g_sort.begin() + i);
  }
  ++g->busy;
  g_sort.push_back(g);
  return g;
}
// The build's last read of the buffers (k_prep_users / k_prep_items) is enqueued on st: record
// that point, so that the next build on the same stream HANDLE but a different stream
// (cudaStreamPerThread from another thread) waits for it before overwriting the keys.
void sort_graph_put(SortGraph* g, cudaStream_t st) {
  if (!g) return;
  cudaEventRecord(g->done, st);
  std::lock_guard<std::mutex> lk(g_sort_mu);
  g->used = true;
  --g->busy;
}
}  // namespace

// Zero up to four small device regions (word counts) in one launch instead of four memsets.
__global__ void k_zero4(uint32_t* a, int na, uint32_t* b, int nb, uint32_t* c, int nc, uint32_t* d, int nd) {
  pdl_enter();  // (PDL: see launch_pdl)
  const int t = threadIdx.x;
  if (t < na) a[t] = 0u;
  if (t < nb) b[t] = 0u;
  if (t < nc) c[t] = 0u;
  if (t < nd) d[t] = 0u;
}
cudaError_t zero4(cudaStream_t st, void* a, int na, void* b, int nb, void* c, int nc, void* d, int nd) {
  CK_PDL(launch_pdl(k_zero4, dim3(1), dim3(128), 0, st, static_cast<uint32_t*>(a), na, static_cast<uint32_t*>(b), nb, static_cast<uint32_t*>(c),
                             nc, static_cast<uint32_t*>(d), nd));
  count_launch();
  return cudaGetLastError();
}

cudaError_t build_prep(BuildCtx& c, const float* Q, const float* P, cudaStream_t st) {
  rmips_index_s* x = c.idx;
  const int64_t n = x->n, m = x->m;
  const int d = x->d, ldh = x->ldh;
  // B1: norms as sort keys of one concatenated [items | users] sequence (items carry the top
  // bit, so a descending sort puts them first); non-finite check; max |p_j|
  const int64_t tot = m + n;
  const bool staged = (size_t)kNormRows * (d | 1) * sizeof(float) <= 200 * 1024;
  const size_t nsm = staged ? (size_t)kNormRows * (d | 1) * sizeof(float) : 0;
  if (nsm > 48 * 1024) {
    cudaError_t e = set_smem_attr((const void*)k_norms, (int)nsm);
    if (e != cudaSuccess) return e;
  }
  SortGraph* sg = sort_graph_get(st, tot);  // (nullptr: the direct path below)
  if (sg && sg->used) {
    cudaError_t e = cudaStreamWaitEvent(st, sg->done, 0);  // the previous user is done with the buffers
    if (e != cudaSuccess) {
      sort_graph_put(sg, st);
      return e;
    }
  }
  uint64_t* kin = sg ? sg->keys : c.nkey;
  uint64_t* kout = kin + tot;
  int32_t* vin = sg ? sg->vals : c.nval;
  int32_t* vout = vin + tot;
  k_norms<<<nblk(m, kNormRows), kNormThreads, nsm, st>>>(P, m, d, kin, 1ull << 63, x->d_flags, c.maxabs, staged);
  count_launch();
  if (n) k_norms<<<nblk(n, kNormRows), kNormThreads, nsm, st>>>(Q, n, d, kin + m, 0ull, x->d_flags, nullptr, staged);
  if (n) count_launch();
  // B2: one stable radix sort (descending norm, ties by ascending index: reading R6)
  if (sg) {
    cudaError_t e = cudaGraphLaunch(sg->exec, st);
    count_launch(1 + kCubSortKernels);
    if (e != cudaSuccess) {
      sort_graph_put(sg, st);
      return e;
    }
  } else {
    k_iota<<<nblk(tot, 256), 256, 0, st>>>(vin, tot); count_launch();
    size_t tb = c.cub_bytes;
    cudaError_t e = cub::DeviceRadixSort::SortPairsDescending(c.cub_tmp, tb, kin, kout, vin, vout, (int)tot, 0, 64, st);
    count_launch(kCubSortKernels);
    if (e != cudaSuccess) return e;
  }
  k_split_sorted<<<nblk(tot, 256), 256, 0, st>>>(kout, vout, m, n, x->pnorm, x->perm_p, x->unorm, x->perm_u,
                                                 c.inv_u);
  count_launch();
  // B3
  if (n)
    k_prep_users<<<nblk((n + kPrepRows - 1) / kPrepRows * 32, 256), 256, 0, st>>>(Q, n, d, ldh, c.inv_u, kin + m, x->U16,
                                                                               x->U32, x->unu); count_launch();
  k_prep_items<<<nblk(m * 32, 256), 256, 0, st>>>(P, m, d, ldh, x->pd, x->perm_p, x->pnorm, c.maxabs, x->c1, x->c2,
                                                    x->P16, x->P32, x->perr, c.scale_dev); count_launch();
  sort_graph_put(sg, st);  // last use of the sort buffers (kin) is enqueued
  return cudaGetLastError();
}

size_t build_cub_bytes(int64_t n, int64_t m) {
  size_t a = 0;
  cub::DeviceRadixSort::SortPairsDescending((void*)nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                            (const int32_t*)nullptr, (int32_t*)nullptr, (int)(n + m), 0, 64);
  return a;
}

template <int MAXC>
static cudaError_t launch_select(BuildCtx& c, cudaStream_t st) {
  rmips_index_s* x = c.idx;
  const int kc = x->kmax < MAXC ? x->kmax : MAXC;
  const size_t smem = (size_t)kSelWarps * x->pd * sizeof(double) + (size_t)kc * kSelStride * (8 + 4 + 4);
  if (smem > 48 * 1024) {
    cudaError_t e = set_smem_attr((const void*)k_exact_select<MAXC>, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, x->device);
  const int64_t want = (x->n + kSelRows - 1) / kSelRows;
  const int grid = (int)(want < (int64_t)sms * 8 ? want : (int64_t)sms * 8);
  k_exact_select<MAXC><<<grid, 32 * kSelWarps, smem, st>>>(x->U32, x->P32, x->perm_p, x->unu, c.cand, c.ccount, x->n,
                                                           x->d, x->pd, x->kmax, x->tau, x->ids, x->thr, c.cand_total);
  count_launch();
  return cudaGetLastError();
}

cudaError_t build_select(BuildCtx& c, cudaStream_t st) {
  if (c.idx->n == 0) return cudaSuccess;
  return c.cstride == 256 ? launch_select<256>(c, st) : launch_select<kCand>(c, st);
}

cudaError_t build_fallback(BuildCtx& c, int nrows, double* scratch, int grid, cudaStream_t st) {
  rmips_index_s* x = c.idx;
  if (nrows <= 0) return cudaSuccess;
  k_exact_row_full<<<grid, 256, 0, st>>>(x->U32, x->P32, x->perm_p, x->unu, c.ovf_list, c.ovf_count, x->n, c.mb,
                                         x->d, x->pd, x->kmax, scratch, x->tau, x->ids, x->thr); count_launch();
  return cudaGetLastError();
}

cudaError_t build_blocks(BuildCtx& c, cudaStream_t st) {
  rmips_index_s* x = c.idx;
  if (x->n == 0) return cudaSuccess;
  k_blocks<<<nblk(x->nlb * x->kmax * 32, 256), 256, 0, st>>>(x->tau, x->unorm, x->n, x->kmax, x->nlb, x->bsz,
                                                             x->tb);
  count_launch();
  return cudaGetLastError();
}

}  // namespace rmips
