// Micro-benchmark: issue timestamps of back-to-back tcgen05.mma (SS, 128x128x16)
// from an idle tensor pipe -> issue cost per MMA and the depth of the MMA queue
// (issue starts stalling once the queue is full).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --expt-relaxed-constexpr -I../../paper_2510_18121_b200/csrc/cuda umma_queue.cu -o umma_queue
#include <cstdio>
#include <cuda_runtime.h>
#include "ca_common.cuh"
#include "ca_mma.cuh"
using namespace cad_dev;

__global__ void __launch_bounds__(128, 1) bench(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t sa = smem_u32(smem), sb = sa + kTileBytes;
  constexpr uint32_t idesc = idesc_bf16(128, 128, false, false);
  if (warp == 0) {
    unsigned long long t[17];
    t[0] = clock64();
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      issue_qk(tmem, sa, sb);  // 8 MMAs, converged warp + elect.sync (as in the kernels)
      t[i + 1] = clock64();
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long te = clock64();
    if (lane == 0 && blockIdx.x == 0) {
      for (int i = 0; i <= 16; ++i) out[i] = t[i] - t[0];
      out[65] = te - t[0];
    }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) tmem_free<512>(tmem);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 66 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * kTileBytes);
  for (int r = 0; r < 2; ++r) bench<<<1, 128, 3 * kTileBytes>>>(d);
  cudaDeviceSynchronize();
  unsigned long long h[66];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("issue timestamps (cycles since first issue):\n");
  printf("after each group of 8 MMAs: ");
  for (int i = 1; i <= 16; ++i) printf("%llu ", h[i]);
  printf("\n");
  printf("all complete at %llu (128 x 64 = 8192 ideal)  err=%s\n", h[65], cudaGetErrorString(cudaGetLastError()));
  return 0;
}
