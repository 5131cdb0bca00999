// Micro-benchmark: latency of a 64-column tcgen05.ld (2 x 32x32b.x32 + wait)
// and of a 32-column tcgen05.st (+ wait) by 8 element-wise warps, with the
// tensor pipe idle vs running the dK/dV MMA mix (QK^T SS + PV TS into TMEM).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --expt-relaxed-constexpr -I../../paper_2510_18121_b200/csrc/cuda tmem_lat.cu -o tmem_lat
#include <cstdio>
#include <cuda_runtime.h>
#include "ca_common.cuh"
#include "ca_mma.cuh"
using namespace cad_dev;

template <bool MMA>
__global__ void __launch_bounds__(384, 1) bench(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) done = 0;
  if (warp == 8) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t sq = smem_u32(smem), sk = sq + 2 * kTileBytes, sv = sq + 4 * kTileBytes;
  if (warp == 8) {
    if (MMA) {
      for (int it = 0; it < 3000; ++it) {
        issue_pv(tmem + 256, tmem + 0, tmem + 32, sv, true);     // dV-like (A from TMEM cols 0..63)
        issue_qk(tmem + 0, sk, sq);                               // S^T-like into [0,128)
        issue_pv(tmem + 384, tmem + 128, tmem + 160, sq, true);  // dK-like
        issue_qk(tmem + 128, sk + kTileBytes, sq + kTileBytes);   // dP^T-like into [128,256)
      }
    } else {
      unsigned long long t = clock64();
      while (clock64() - t < 3000ull * 2048) {}
    }
    __syncwarp();
    if (lane == 0) done = 1;
  } else if (warp < 8) {
    const uint32_t lsel = ((warp & 3) * 32) << 16;
    unsigned long long ld_cyc = 0, st_cyc = 0, n = 0;
    uint32_t acc = 0;
    while (!done) {
      uint32_t r0[32], r1[32];
      unsigned long long t0 = clock64();
      tmem_ld32(tmem + lsel + 64 * (warp >> 2), r0);
      tmem_ld32(tmem + lsel + 64 * (warp >> 2) + 32, r1);
      tmem_wait_ld();
      unsigned long long t1 = clock64();
      uint32_t pk[16];
      for (int i = 0; i < 16; ++i) pk[i] = r0[i] ^ r1[i + 16];
      acc ^= r0[31] ^ r1[0];
      tmem_st16(tmem + lsel + 128 + 64 * (warp >> 2), pk);
      tmem_wait_st();
      unsigned long long t2 = clock64();
      ld_cyc += t1 - t0;
      st_cyc += t2 - t1;
      ++n;
      unsigned long long t = clock64();
      while (clock64() - t < 400) {}  // some spacing, like the kernels' math
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = ld_cyc; out[1] = st_cyc; out[2] = n; out[3] = acc; }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 8) tmem_free<512>(tmem);
}

template <bool MMA>
void run(const char* name, unsigned long long* d) {
  auto k = bench<MMA>;
  const int sm = 6 * kTileBytes + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k<<<148, 384, sm>>>(d);
  cudaDeviceSynchronize();
  unsigned long long h[4];
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("%-22s ld(64 cols)+wait: %.0f cycles, st(16 cols)+wait: %.0f cycles (n=%llu) err=%s\n", name,
         double(h[0]) / h[2], double(h[1]) / h[2], h[2], cudaGetErrorString(cudaGetLastError()));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 32);
  run<false>("tensor pipe idle", d);
  run<true>("dK/dV MMA mix running", d);
  return 0;
}
