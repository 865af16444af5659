// epiq.cuh -- the candidate epilogue's per-tile fast path and out-of-line slow path, shared by the
// tensor-core build kernels that use the candpol.cuh policies (build_tcq.cu, build_tc2cta.cu).
#pragma once
#include "candpol.cuh"
#include "common.cuh"
#include "sm100.cuh"

namespace rmips {

#ifdef RMIPS_EPI_PROFILE
extern __device__ unsigned long long g_epi_prof[4][256];  // build_tc.cu
#endif

// Fast path of one 64-column half (scores of this thread's row): 3-input max trees and one
// compare per 32-column chunk.  Returns a warp-uniform 2-bit mask of the chunks in which some
// lane may append.  Padding columns of a ragged last tile (TMA zero fill) are not masked here: at
// worst they flag a chunk, and the slow path masks them before anything is appended.
__device__ __forceinline__ uint32_t epiq_fast(const uint32_t (&h)[64], float E0, float E1, float theta) {
  uint32_t bits = 0;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    const float mx = sm100::max32_bits(h + 32 * c);
    bits |= (uint32_t)__any_sync(0xffffffffu, __fadd_ru(mx, c ? E1 : E0) >= theta) << c;
  }
  return bits;
}

// Slow path (one copy in the kernel, so the hot loop stays inside the instruction cache):
// re-read each flagged chunk of the current accumulator stage from TMEM, append and refresh.
template <class Pol>
static __device__ __noinline__ typename Pol::Row epiq_slow(uint32_t bits, uint32_t taddr, int base0, int mi, float4 E4,
                                                    typename Pol::Row me, typename Pol::Buf sb, int rr, float e0x2,
                                                    int kmax) {
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
    const float E = c == 0 ? E4.x : c == 1 ? E4.y : c == 2 ? E4.z : E4.w;
    float g4[8];
#pragma unroll
    for (int g = 0; g < 8; ++g)
      g4[g] = fmaxf(fmaxf(__uint_as_float(r[4 * g]), __uint_as_float(r[4 * g + 1])),
                    fmaxf(__uint_as_float(r[4 * g + 2]), __uint_as_float(r[4 * g + 3])));
#ifdef RMIPS_EPI_PROFILE
    const long long p0 = clock64();
#endif
    Pol::append([&](int j) { return __uint_as_float(r[j]); }, g4, E, pos0, mi, me, sb, rr);
#ifdef RMIPS_EPI_PROFILE
    const long long p1 = clock64();
    const bool rf = __any_sync(0xffffffffu, me.cnt > Pol::kSlots - 32);
#endif
    Pol::maybe_refresh(me, sb, rr, e0x2, kmax);
#ifdef RMIPS_EPI_PROFILE
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&g_epi_prof[2][0], 1ull);
      atomicAdd(&g_epi_prof[2][1], (unsigned long long)(p1 - p0));
      atomicAdd(&g_epi_prof[2][2], (unsigned long long)(clock64() - p1));
      atomicAdd(&g_epi_prof[2][3], (unsigned long long)rf);
    }
#endif
  }
  return me;
}

}  // namespace rmips
