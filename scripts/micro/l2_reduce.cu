// Micro-benchmark: fp32 reduce-add throughput into global memory, the cost
// that decides whether dQ partials can be accumulated inside the dK/dV
// kernel (DESIGN.md §7b/§8). Every CTA repeatedly adds one 64 KB partial
// (a 128 x 128 fp32 dQ tile) into a target tile chosen from a working set of
// W bytes, by
//   bulk : cp.reduce.async.bulk.global.shared::cta.add.f32 in CHUNK-byte pieces
//   rowv4: red.global.add.v4.f32, one 512 B row per thread (TMEM 32x32b layout)
//   coal : red.global.add.v4.f32, consecutive threads on consecutive 16 B
//   store: plain st.global.v4 of the same bytes (write-bandwidth reference)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_reduce l2_reduce.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kTile = 128 * 128 * 4;  // bytes of one partial

__device__ __forceinline__ uint32_t tile_of(int cta, int it, int n_tiles, int spread) {
  // consecutive CTAs sweep the same tiles `spread` apart (the dK/dV pairs of
  // one document and head walk the same q tiles at different times)
  return static_cast<uint32_t>((static_cast<long long>(cta) * spread + it) % n_tiles);
}

template <int CHUNK>
__global__ void __launch_bounds__(128, 1) k_bulk(float* dst, int n_tiles, int iters, int spread) {
  extern __shared__ __align__(128) float src[];
  for (int i = threadIdx.x; i < kTile / 4; i += blockDim.x) src[i] = 1.f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(src));
  for (int it = 0; it < iters; ++it) {
    char* t = reinterpret_cast<char*>(dst) + static_cast<size_t>(tile_of(blockIdx.x, it, n_tiles, spread)) * kTile;
#pragma unroll 1
    for (int c = 0; c < kTile; c += CHUNK)
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(t + c), "r"(s + c),
                   "n"(CHUNK)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void __launch_bounds__(128) k_rowv4(float* dst, int n_tiles, int iters, int spread) {
  for (int it = 0; it < iters; ++it) {
    float* t = dst + static_cast<size_t>(tile_of(blockIdx.x, it, n_tiles, spread)) * (kTile / 4);
    float* row = t + threadIdx.x * 128;
#pragma unroll 8
    for (int c = 0; c < 128; c += 4)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + c), "f"(1.f), "f"(1.f), "f"(1.f),
                   "f"(1.f)
                   : "memory");
  }
}

__global__ void __launch_bounds__(128) k_coal(float* dst, int n_tiles, int iters, int spread) {
  for (int it = 0; it < iters; ++it) {
    float* t = dst + static_cast<size_t>(tile_of(blockIdx.x, it, n_tiles, spread)) * (kTile / 4);
#pragma unroll 8
    for (int c = threadIdx.x * 4; c < kTile / 4; c += 128 * 4)
      asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(t + c), "f"(1.f), "f"(1.f), "f"(1.f),
                   "f"(1.f)
                   : "memory");
  }
}

__global__ void __launch_bounds__(128) k_store(float* dst, int n_tiles, int iters, int spread) {
  for (int it = 0; it < iters; ++it) {
    float4* t = reinterpret_cast<float4*>(dst + static_cast<size_t>(tile_of(blockIdx.x, it, n_tiles, spread)) * (kTile / 4));
#pragma unroll 8
    for (int c = threadIdx.x; c < kTile / 16; c += 128) t[c] = make_float4(1.f, 1.f, 1.f, (float)it);
  }
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t max_bytes = size_t(2) << 30;
  float* dst;
  if (cudaMalloc(&dst, max_bytes) != cudaSuccess) return 1;
  cudaMemset(dst, 0, max_bytes);
  cudaFuncSetAttribute(k_bulk<8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTile);
  cudaFuncSetAttribute(k_bulk<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTile);
  cudaFuncSetAttribute(k_bulk<65536>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTile);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 400;
  const size_t ws_list[] = {size_t(8) << 20, size_t(32) << 20, size_t(96) << 20, size_t(512) << 20, max_bytes};
  const int spreads[] = {1, 7};
  const char* names[] = {"bulk8K", "bulk16K", "bulk64K", "rowv4", "coal", "store"};
  for (int ctas_per_sm = 1; ctas_per_sm <= 2; ++ctas_per_sm) {
    const int grid = sms * ctas_per_sm;
    for (size_t ws : ws_list)
      for (int spread : spreads) {
        const int n_tiles = static_cast<int>(ws / kTile);
        for (int m = 0; m < 6; ++m) {
          float best = 1e30f;
          for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            switch (m) {
              case 0: k_bulk<8192><<<grid, 128, kTile>>>(dst, n_tiles, iters, spread); break;
              case 1: k_bulk<16384><<<grid, 128, kTile>>>(dst, n_tiles, iters, spread); break;
              case 2: k_bulk<65536><<<grid, 128, kTile>>>(dst, n_tiles, iters, spread); break;
              case 3: k_rowv4<<<grid, 128>>>(dst, n_tiles, iters, spread); break;
              case 4: k_coal<<<grid, 128>>>(dst, n_tiles, iters, spread); break;
              default: k_store<<<grid, 128>>>(dst, n_tiles, iters, spread); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            if (ms < best) best = ms;
          }
          const double bytes = double(grid) * iters * kTile;
          printf("ctas/sm %d ws %6zu MB spread %d %-8s %8.3f ms %8.1f GB/s  %s\n", ctas_per_sm, ws >> 20, spread, names[m],
                 best, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
        }
      }
  }
  return 0;
}
