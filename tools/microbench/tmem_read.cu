// Development microbenchmark: TMEM -> register read throughput per SM (tcgen05.ld.32x32b.x32).
// W warps (4 quadrants x W/4) each read NCOL columns per iteration for ITER iterations.
#include <cstdio>
#include <cstdint>
#include "../../paper_2110_07131_b200/csrc/sm100.cuh"
using namespace rmips::sm100;

template <int W>
__global__ void __launch_bounds__(32 * W, 1) k(uint64_t* out, int iters, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) { tmem_alloc(smem_u32(&slot), 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[4][32];
    tmem_ld32(tm, r[0]); tmem_ld32(tm + 32, r[1]); tmem_ld32(tm + 64, r[2]); tmem_ld32(tm + 96, r[3]);
    tmem_ld_wait(r[0]); reg_fence(r[1]); reg_fence(r[2]); reg_fence(r[3]);
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int j = 0; j < 32; j += 2) acc = fmaxf(acc, fmaxf(__uint_as_float(r[c][j]), __uint_as_float(r[c][j + 1])));
  }
  const long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.f) *sink = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_dealloc(slot, 512);
}

template <int W>
void run(int iters) {
  uint64_t* d; float* s; cudaMalloc(&d, 148 * 8); cudaMalloc(&s, 4);
  k<W><<<148, 32 * W>>>(d, iters, s);
  cudaDeviceSynchronize();
  uint64_t h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const double bytes = (double)W * 32 * 128 * 4 * iters;  // per SM
  printf("warps %d: %.1f cycles per iteration, %.1f B/clk/SM TMEM read (err %s)\n", W, (double)h[0] / iters,
         bytes / h[0], cudaGetErrorString(cudaGetLastError()));
}
int main() { run<4>(10000); run<8>(10000); run<16>(10000); return 0; }
