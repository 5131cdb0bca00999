// Micro-benchmark: tensor-pipe rate of the forward's MMA mix (QK^T SS N=128 +
// PV TS, two heads) while 8 other warps stress TMEM with tcgen05.ld/st as the
// softmax does. Prints cycles per 128x128x16 MMA (ideal 64).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2510_18121_b200/csrc/cuda umma_mix.cu -o umma_mix
#include <cstdio>
#include <cuda_runtime.h>
#include "ca_common.cuh"
#include "ca_mma.cuh"
using namespace cad_dev;

template <int LOAD, int MIX>
__global__ void __launch_bounds__(384, 1) bench(unsigned long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int done;
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); done = 0; }
  if (warp == 8) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t sq = smem_u32(smem), sk = sq + 2 * kTileBytes, sv = sq + 4 * kTileBytes;
  if (warp == 8) {
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int h = 0; h < 2; ++h) {
        if (MIX & 1) issue_pv(tmem + 256 + h * 128, tmem + h * 128, tmem + h * 128 + 32, sv, true);
        if (MIX & 2) issue_qk(tmem + h * 128, sq + h * kTileBytes, sk);
      }
    }
    if (MIX == 0) { while (clock64() - t0 < 2000000ull) {} }
    if (elect_one()) umma_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (lane == 0 && blockIdx.x == 0) out[0] = t1 - t0;
    if (lane == 0) done = 1;
  } else if (warp < 8 && LOAD) {
    const int h = warp >> 2;
    const uint32_t lane_sel = ((warp & 3) * 32) << 16;
    const uint32_t s_tmem = tmem + lane_sel + h * 128;
    float acc = 0.f;
    unsigned long long n_ld = 0, c_ld = 0;
    while (!done) {
      const unsigned long long ta = clock64();
      uint32_t r[32];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        tmem_ld32(s_tmem + c * 32, r);
        tmem_wait_ld();
        for (int i = 0; i < 32; ++i) acc += __uint_as_float(r[i]);
      }
      c_ld += clock64() - ta;
      ++n_ld;
      if (LOAD >= 2) {
        uint32_t pk[16];
        for (int i = 0; i < 16; ++i) pk[i] = __float_as_uint(acc) + i;
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_st16(s_tmem + c * 16, pk);
        tmem_wait_st();
      }
    }
    if (acc == 12345.f) out[1] = 1;
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[2] = c_ld; out[3] = n_ld; }
  }
  tc_fence_before(); __syncthreads();
  if (warp == 8) tmem_free<512>(tmem);
}

template <int LOAD, int MIX>
void run(const char* name, unsigned long long* d, int iters) {
  auto k = bench<LOAD, MIX>;
  const int sm = 6 * kTileBytes + 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  k<<<148, 384, sm>>>(d, iters);
  cudaDeviceSynchronize();
  unsigned long long c = 0, h[4] = {0, 0, 0, 0};
  cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  c = h[0];
  const int per_it = MIX == 0 ? 1 : 2 * (((MIX & 1) ? 8 : 0) + ((MIX & 2) ? 8 : 0));
  printf("%-28s %.1f cycles/MMA (ideal 64); 128-col tcgen05.ld row: %.0f cycles  err=%s\n", name,
         double(c) / (iters * per_it), h[3] ? double(h[2]) / h[3] : 0.0, cudaGetErrorString(cudaGetLastError()));
  cudaMemset(d, 0, 32);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 32);
  cudaMemset(d, 0, 32);
  const int iters = 2000;
  run<0, 2>("QK only", d, iters);
  run<0, 1>("PV only", d, iters);
  run<0, 3>("PV+QK", d, iters);
  run<1, 3>("PV+QK, tmem ld", d, iters);
  run<2, 3>("PV+QK, tmem ld+st", d, iters);
  run<1, 2>("QK, tmem ld", d, iters);
  run<1, 0>("no MMA, tmem ld", d, iters);
  run<1, 1>("PV, tmem ld", d, iters);
  return 0;
}
