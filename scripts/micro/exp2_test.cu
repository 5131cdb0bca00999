#include <cstdio>
#include <cmath>
#include "sm100.cuh"
using namespace cad_dev;
__global__ void k(const float* x, float* y, int n) {
  int i = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (i + 1 >= n) return;
  float a = x[i], b = x[i + 1];
  exp2_fma2(a, b);
  y[i] = a; y[i + 1] = b;
}
int main() {
  const int n = 4096;
  float hx[n], hy[n];
  for (int i = 0; i < n; ++i) hx[i] = -140.f + 150.f * i / n;
  hx[0] = -INFINITY; hx[3] = -INFINITY; hx[4] = -200.f; hx[5] = -127.f;
  float *dx, *dy;
  cudaMalloc(&dx, n * 4); cudaMalloc(&dy, n * 4);
  cudaMemcpy(dx, hx, n * 4, cudaMemcpyHostToDevice);
  k<<<8, 256>>>(dx, dy, n);
  cudaMemcpy(hy, dy, n * 4, cudaMemcpyDeviceToHost);
  double worst = 0; int wi = 0;
  for (int i = 0; i < n; ++i) {
    double r = std::exp2((double)hx[i]);
    double e = r > 1e-30 ? std::fabs(hy[i] - r) / r : std::fabs(hy[i] - r);
    if (!(e <= worst)) { worst = e; wi = i; }
  }
  printf("worst rel err %g at x=%g (got %g want %g); x=%g -> %g; x=0 -> %g\n", worst, hx[wi], hy[wi], std::exp2((double)hx[wi]), hx[0], hy[0], hy[n*140/150]);
  for (int i = 0; i < 6; ++i) printf("x=%g got %g\n", hx[i], hy[i]);
  for (int i = 1000; i < 4096; i += 500) printf("x=%g got %g want %g\n", hx[i], hy[i], std::exp2((double)hx[i]));
}
