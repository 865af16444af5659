// Development microbenchmark: tcgen05.mma issue / execution rate per SM for M = 128, K = 16 fp16,
// N = 64..256, A from shared memory (ss) or tensor memory (ts), optionally one tcgen05.commit every
// C MMAs (the build kernel commits once per 4-MMA K block).  One CTA per SM; one elected lane issues.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mma_rate.cu -o mma_rate
#include <cstdio>
#include <cstdint>
#include "../../paper_2110_07131_b200/csrc/sm100.cuh"
using namespace rmips::sm100;

template <int N, bool TS, int C>
__global__ void __launch_bounds__(128, 1) k(uint64_t* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += 128) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar[0]), 1); mbar_init(smem_u32(&bar[1]), 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(smem_u32(&slot), 512); tmem_relinquish(); }
  fence_proxy_async();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = slot;
  const uint32_t sA = smem_u32(sm), sB = sA + 16384;
  constexpr uint32_t idesc = idesc_f16_f32(128, N);
  const uint64_t adesc = sdesc_sw128(sA), bdesc = sdesc_sw128(sB);
  long long t0 = 0, t1 = 0;
  if (warp == 0) {
    if (TS && elect_one()) {
      for (int kk = 0; kk < 4; ++kk) tmem_cp_128x256b(tm + 384 + 8 * kk, adesc + 2 * kk);
    }
    __syncwarp();
    t0 = clock64();
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tm + (i & 1) * (N <= 192 ? 192 : 256) * 0;  // one accumulator region
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          if (TS) mma_f16_ts(d, tm + 384 + 8 * kk, bdesc + 2 * kk, idesc, 1);
          else mma_f16(d, adesc + 2 * kk, bdesc + 2 * kk, idesc, 1);
          if (C == 1) mma_commit(smem_u32(&bar[0]));
        }
        if (C == 4) mma_commit(smem_u32(&bar[0]));
      }
      __syncwarp();
    }
    if (elect_one()) mma_commit(smem_u32(&bar[1]));
    __syncwarp();
    mbar_wait(smem_u32(&bar[1]), ph);
    t1 = clock64();
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (warp == 0) tmem_dealloc(slot, 512);
}

template <int N, bool TS, int C>
void run(int iters) {
  uint64_t* d; cudaMalloc(&d, 148 * 8);
  const int smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(k<N, TS, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<N, TS, C><<<148, 128, smem>>>(d, iters);  // warm
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<N, TS, C><<<148, 128, smem>>>(d, iters);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  uint64_t h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const double mmas = 4.0 * iters;
  const double tf = 2.0 * 128 * N * 16 * mmas * 148 / (ms / 1e3) / 1e12;
  printf("N %3d %s commit/%d: %.1f cycles per MMA (ideal %d), %.0f TFLOP/s over the launch (%s)\n", N, TS ? "ts" : "ss", C,
         (double)h[0] / mmas, N / 2, tf, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  const int it = 20000;
  run<64, true, 4>(it); run<128, true, 4>(it); run<192, true, 4>(it); run<256, true, 4>(it);
  run<64, false, 4>(it); run<128, false, 4>(it); run<192, false, 4>(it); run<256, false, 4>(it);
  run<128, true, 1>(it); run<128, true, 0>(it); run<256, true, 1>(it);
  return 0;
}
