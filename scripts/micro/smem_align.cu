// Prints the shared-space address of dynamic shared memory (alignment check)
// and the opt-in per-block maximum.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(unsigned* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  if (threadIdx.x == 0) {
    out[0] = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    out[1] = 0;
    smem[232448 - 1] = 1;
  }
}
int main() {
  unsigned* d; cudaMalloc(&d, 8);
  int mx = 0; cudaDeviceGetAttribute(&mx, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  k<<<1, 32, mx>>>(d);
  unsigned h[2]; cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  printf("optin max %d, dynamic smem base 0x%x (mod 1024 = %u), static bar 0x%x, err=%s\n", mx, h[0], h[0] % 1024, h[1],
         cudaGetErrorString(cudaGetLastError()));
}
