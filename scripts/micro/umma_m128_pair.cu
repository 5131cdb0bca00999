// Probe: where does an M=128 cta_group::2 tcgen05.mma put D, with
//   A = 128 x 256 (M x K), CTA r holding rows [64r, 64r+64) for all K, MN-major SW128
//   B = 256 x 128 (K x N), CTA r holding columns [64r, 64r+64) for all K, MN-major SW128
// (the dQ = dS K shape a fused dK/dV/dQ pair kernel needs). The host swizzles
// both operands into each CTA's shared-memory image; the kernel copies them
// in, runs 16 K-steps, dumps each CTA's TMEM (128 lanes x 128 columns) and
// the host locates every reference D entry in the dumps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2510_18121_b200/csrc/cuda umma_m128_pair.cu -o umma_m128_pair
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace cad_dev;

constexpr int kBuf = 32768;  // bytes per operand per CTA (256 rows x 128 B)

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const uint8_t* img, float* dump, uint32_t idesc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t rank = cluster_rank();
  const uint32_t warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint8_t* src = img + size_t(rank) * 2 * kBuf;
  for (int i = threadIdx.x; i < 2 * kBuf / 16; i += 128)
    reinterpret_cast<uint4*>(smem)[i] = reinterpret_cast<const uint4*>(src)[i];
  fence_proxy_async_smem();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc_2sm<512>(&tbase);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = tbase;
  // clear D's possible footprint with a sentinel
  {
    uint32_t s[32];
    for (int k = 0; k < 32; ++k) s[k] = __float_as_uint(-12345.f);
    for (int c = 0; c < 512; c += 32) tmem_st32(tmem + ((warp * 32) << 16) + c, s);
    tmem_wait_st();
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t sa = smem_u32(smem), sb = sa + kBuf;
  if (rank == 0 && warp == 0) {
    if (elect_one()) {
      for (int s = 0; s < 16; ++s)
        umma_ss_2sm(tmem + 128, sw128_desc(sa + s * 2048, 16384, 1024), sw128_desc(sb + s * 2048, 16384, 1024),
                    idesc, s > 0 ? 1u : 0u);
      umma_commit_pair(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float* out = dump + size_t(rank) * 128 * 512;
  for (int c = 0; c < 512; c += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((warp * 32) << 16) + c, r);
    tmem_wait_ld();
    for (int k = 0; k < 32; ++k) out[(warp * 32 + lane) * 512 + c + k] = __uint_as_float(r[k]);
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) tmem_free_2sm<512>(tmem);
}

static uint16_t bf(float x) {
  __nv_bfloat16 b = __float2bfloat16(x);
  uint16_t u;
  memcpy(&u, &b, 2);
  return u;
}
static float fb(uint16_t u) {
  uint32_t v = uint32_t(u) << 16;
  float f;
  memcpy(&f, &v, 4);
  return f;
}
// element (row, e) of a [rows x 64] bf16 MN-major SW128 image (128 B rows)
static size_t sw(int row, int e) {
  const size_t logical = size_t(row) * 128 + size_t(e) * 2;
  return logical ^ (((logical >> 7) & 7) << 4);
}

int main() {
  const int M = 128, K = 256, N = 128;
  std::vector<float> A(M * K), B(K * N);
  unsigned s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 65536.f - 0.5f; };
  for (auto& x : A) x = fb(bf(rnd()));
  for (auto& x : B) x = fb(bf(rnd()));
  std::vector<uint8_t> img(2 * 2 * kBuf, 0);
  for (int r = 0; r < 2; ++r) {
    uint8_t* a = img.data() + size_t(r) * 2 * kBuf;
    uint8_t* b = a + kBuf;
    for (int k = 0; k < K; ++k)
      for (int e = 0; e < 64; ++e) {
        const uint16_t va = bf(A[(64 * r + e) * K + k]);  // A[m][k], m = 64r + e
        const uint16_t vb = bf(B[k * N + 64 * r + e]);    // B[k][n], n = 64r + e
        memcpy(a + sw(k, e), &va, 2);
        memcpy(b + sw(k, e), &vb, 2);
      }
  }
  std::vector<double> D(M * N);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double acc = 0;
      for (int k = 0; k < K; ++k) acc += double(A[m * K + k]) * B[k * N + n];
      D[m * N + n] = acc;
    }
  uint8_t* dimg;
  float* ddump;
  cudaMalloc(&dimg, img.size());
  cudaMalloc(&ddump, 2 * 128 * 512 * 4);
  cudaMemcpy(dimg, img.data(), img.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kBuf);
  probe<<<2, 128, 2 * kBuf>>>(dimg, ddump, idesc_bf16(128, 128, true, true));
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> dump(2 * 128 * 512);
  cudaMemcpy(dump.data(), ddump, dump.size() * 4, cudaMemcpyDeviceToHost);
  // locate each TMEM value among the reference entries
  std::vector<std::pair<double, int>> sorted;
  for (int i = 0; i < M * N; ++i) sorted.push_back({D[i], i});
  std::sort(sorted.begin(), sorted.end());
  int found = 0, sentinel = 0, other = 0;
  std::vector<int> hit(M * N, 0);
  for (int r = 0; r < 2; ++r)
    for (int lane = 0; lane < 128; ++lane)
      for (int c = 0; c < 512; ++c) {
        const float v = dump[(size_t(r) * 128 + lane) * 512 + c];
        if (v == -12345.f) { ++sentinel; continue; }
        auto it = std::lower_bound(sorted.begin(), sorted.end(), std::make_pair(double(v) - 1e-3, -1));
        int best = -1;
        double bd = 1e9;
        for (auto j = it; j != sorted.end() && j->first <= v + 1e-3; ++j)
          if (std::fabs(j->first - v) < bd) { bd = std::fabs(j->first - v); best = j->second; }
        if (best < 0) { ++other; continue; }
        ++found;
        ++hit[best];
        const int m = best / N, n = best % N;
        const bool show = (lane % 32 == 0 || lane % 32 == 1 || lane % 32 == 31) && (c % 64 == 0 || c % 64 == 1 || c % 64 == 63);
        if (show) printf("cta %d lane %3d col %3d -> D[m=%3d][n=%3d]\n", r, lane, c - 128, m, n);
      }
  int missing = 0;
  for (int i = 0; i < M * N; ++i) missing += hit[i] == 0;
  printf("found %d, sentinel %d, unmatched %d, reference entries never seen %d\n", found, sentinel, other, missing);
  return 0;
}
