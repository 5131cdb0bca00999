// Micro-benchmark: cycles per tcgen05.mma (kind::f16) for SS vs TS operand
// sources and N = 64/128/256, one CTA per SM, operands resident in smem.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2510_18121_b200/csrc/cuda umma_rate.cu -o umma_rate
#include <cstdio>
#include <cuda_runtime.h>
#include "sm100.cuh"
using namespace cad_dev;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t sa = smem_u32(smem), sb = sa + 32768;
  unsigned long long t0 = 0, t1 = 0;
  if (warp == 0) {
    constexpr uint32_t idesc = idesc_bf16(128, N, false, false);
    if (elect_one()) {
      t0 = clock64();
      for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
          if (TS)
            umma_ts(tmem + 256, tmem + k * 8, sw128_desc(sb + (k >> 2) * (N * 128) + (k & 3) * 32, 16, 1024), idesc, k > 0);
          else
            umma_ss(tmem + 256, sw128_desc(sa + off, 16, 1024), sw128_desc(sb + (k >> 2) * (N * 128) + (k & 3) * 32, 16, 1024), idesc, k > 0);
        }
      }
      umma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    t1 = clock64();
    if (elect_one() && blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_free<512>(tmem);
}

template <int N, bool TS>
void run(const char* name, unsigned long long* d, int iters) {
  auto k = bench<N, TS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
  k<<<148, 128, 100000>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double per = double(c) / (iters * 8.0);
  const double ideal = 128.0 * N / 256.0;
  printf("%-10s N=%3d: %.1f cycles/MMA (ideal %.0f) -> %.0f%% of tensor peak  err=%s\n", name, N, per, ideal,
         100.0 * ideal / per, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int iters = 4000;
  run<64, false>("SS", d, iters);
  run<128, false>("SS", d, iters);
  run<256, false>("SS", d, iters);
  run<64, true>("TS", d, iters);
  run<128, true>("TS", d, iters);
  run<256, true>("TS", d, iters);
  return 0;
}
