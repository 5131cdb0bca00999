// Micro-benchmark: the dK/dV kernel's per-iteration MMA mix (S^T, dP^T: SS
// K-major N=128; dV, dK: TS with an MN-major smem B) with and without a
// concurrent 64 KB/iteration bulk global->smem copy stream (the Q/dO TMA
// traffic). Prints cycles per 128x128x16 MMA (ideal 64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --expt-relaxed-constexpr -I../../paper_2510_18121_b200/csrc/cuda umma_bwd.cu -o umma_bwd
#include <cstdio>
#include <cuda_runtime.h>
#include "ca_common.cuh"
#include "ca_mma.cuh"
using namespace cad_dev;

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(dst), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

template <int COPY>
__global__ void __launch_bounds__(384, 1) bench(unsigned long long* out, const uint8_t* gsrc, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, cbar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init(&cbar, 1); fence_barrier_init(); done = 0; }
  if (warp == 8) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t sK = smem_u32(smem), sV = sK + kTileBytes, sQ = sK + 2 * kTileBytes, sDO = sK + 3 * kTileBytes;
  const uint32_t sCopy = sK + 4 * kTileBytes;  // 2 x 32 KB landing zone
  const uint32_t tS = tmem, tDP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;
  if (warp == 8) {
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      issue_pv(tDV, tS, tS + 64, sDO, true);
      issue_qk(tS, sK, sQ);
      issue_pv(tDK, tDP, tDP + 64, sQ, true);
      issue_qk(tDP, sV, sDO);
    }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    if (lane == 0) done = 1;
  } else if (warp == 9 && COPY && lane == 0) {
    uint32_t ph = 0;
    const uint8_t* src = gsrc + (size_t)blockIdx.x * (1 << 20);
    int n = 0;
    while (!done) {
      mbar_expect_tx(&cbar, 2 * kTileBytes);
      bulk_g2s(sCopy, src + (n & 15) * 65536, kTileBytes, &cbar);
      bulk_g2s(sCopy + kTileBytes, src + (n & 15) * 65536 + kTileBytes, kTileBytes, &cbar);
      mbar_wait(&cbar, ph);
      ph ^= 1;
      ++n;
      // pace: one 64 KB copy per ~COPY cycles
      unsigned long long t = clock64();
      while (clock64() - t < (unsigned long long)COPY) {}
    }
    if (blockIdx.x == 0) out[1] = n;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 8) tmem_free<512>(tmem);
}

template <int COPY>
void run(const char* name, unsigned long long* d, const uint8_t* g, int iters) {
  auto k = bench<COPY>;
  const int sm = 6 * kTileBytes + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k<<<148, 384, sm>>>(d, g, iters);
  cudaDeviceSynchronize();
  unsigned long long c[2] = {0, 0};
  cudaMemcpy(c, d, 16, cudaMemcpyDeviceToHost);
  printf("%-34s %.1f cycles/MMA (ideal 64), %llu copies  err=%s\n", name, double(c[0]) / (iters * 32.0),
         COPY ? c[1] : 0ull, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  uint8_t* g;
  cudaMalloc(&d, 16);
  cudaMalloc(&g, (size_t)148 << 20);
  cudaMemset(g, 0, (size_t)148 << 20);
  const int iters = 2000;
  run<0>("dkdv MMA mix", d, g, iters);
  run<1>("dkdv MMA mix + 64KB copies (max)", d, g, iters);
  run<2000>("dkdv MMA mix + 64KB / 2000 cyc", d, g, iters);
  run<3000>("dkdv MMA mix + 64KB / 3000 cyc", d, g, iters);
  return 0;
}
