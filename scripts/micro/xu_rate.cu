// Throughput of the softmax instruction mix on one SM: ex2.approx, cvt.rn.bf16x2.f32,
// max, fma, fma.f32x2.  Prints lanes/clk/SM for each.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(float* out, int iters, unsigned long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  uint32_t acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      if (OP == 1) { uint32_t r; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7])); acc ^= r; }
      if (OP == 2) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]));
      if (OP == 3) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]));
      if (OP == 4) {
        uint64_t x = (uint64_t(__float_as_uint(a[i])) << 32) | __float_as_uint(a[(i + 1) & 7]);
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(x));
        a[i] = __uint_as_float(uint32_t(x));
      }
      if (OP == 5) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 3) & 7]), "f"(a[(i + 5) & 7]));
    }
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
}

template <int OP>
void run(const char* name, int threads) {
  float* o; unsigned long long* c;
  cudaMalloc(&o, 4096 * 4); cudaMalloc(&c, 8);
  int iters = 4096;
  k<OP><<<1, threads>>>(o, iters, c);
  k<OP><<<1, threads>>>(o, iters, c);
  unsigned long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  double ops = double(iters) * 8 * threads;
  printf("%-14s threads %4d : %.2f lanes/clk/SM\n", name, threads, ops / h);
  cudaFree(o); cudaFree(c);
}

int main() {
  for (int t : {128, 256, 512}) {
    run<0>("ex2", t); run<1>("cvt.bf16x2", t); run<2>("max", t); run<3>("fma", t); run<4>("fma.f32x2", t);
    run<5>("max3", t);
  }
  return 0;
}
