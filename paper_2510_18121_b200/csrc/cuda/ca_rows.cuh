// TMEM row helpers shared by the backward kernels (thread = TMEM lane =
// tile row): 64-column loads, bf16 packing back into TMEM, and the epilogue
// store of an accumulator row to global memory.
#pragma once

#include <cuda_bf16.h>

#include "sm100.cuh"

namespace cad_dev {

__device__ __forceinline__ void load_row64(uint32_t taddr, float (&x)[64]) {
  uint32_t r[32];
  tmem_ld32(taddr, r);
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(r[i]);
  tmem_ld32(taddr + 32, r);
#pragma unroll
  for (int i = 0; i < 32; ++i) x[32 + i] = __uint_as_float(r[i]);
  tmem_wait_ld();
}

// 64 fp32 -> 32 packed bf16x2 columns at taddr.
__device__ __forceinline__ void store_bf16_64(uint32_t taddr, const float (&x)[64]) {
  uint32_t pk[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) pk[i] = pack_bf16(x[2 * i], x[2 * i + 1]);
  tmem_st32(taddr, pk);
}

// Epilogue helper: TMEM row (64 fp32 columns at taddr) * mul -> bf16 -> 128
// contiguous bytes at dst (if valid).
__device__ __forceinline__ void tmem_row_to_global(uint32_t taddr, float mul, __nv_bfloat16* dst,
                                                   bool valid) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    tmem_wait_ld();
    uint4 w[4];
    uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      wp[i] = pack_bf16(__uint_as_float(r[2 * i]) * mul, __uint_as_float(r[2 * i + 1]) * mul);
    if (valid) {
      uint4* d = reinterpret_cast<uint4*>(dst + c * 32);
#pragma unroll
      for (int i = 0; i < 4; ++i) d[i] = w[i];
    }
  }
}

// Same 64 columns, scaled, into row `row` of a 128-row x 64-column bf16
// SW128 plane in shared memory (the layout a 64 x 128-row TMA box stores).
__device__ __forceinline__ void tmem_row_to_smem_sw128(uint32_t taddr, float mul, uint8_t* plane, uint32_t row) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    tmem_wait_ld();
    uint4 w[4];
    uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
    for (int i = 0; i < 16; ++i)
      wp[i] = pack_bf16(__uint_as_float(r[2 * i]) * mul, __uint_as_float(r[2 * i + 1]) * mul);
    uint8_t* line = plane + row * 128;
#pragma unroll
    for (int i = 0; i < 4; ++i) *reinterpret_cast<uint4*>(line + (((c * 4 + i) ^ (row & 7)) << 4)) = w[i];
  }
}

// 64 TMEM columns of this thread's row, scaled and packed to bf16x2.
__device__ __forceinline__ void tmem_row_to_regs_bf16(uint32_t taddr, float mul, uint32_t (&pk)[32]) {
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t r[32];
    tmem_ld32(taddr + c * 32, r);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 16; ++i)
      pk[16 * c + i] = pack_bf16(__uint_as_float(r[2 * i]) * mul, __uint_as_float(r[2 * i + 1]) * mul);
  }
}
// 32 packed bf16x2 (64 columns) into row `row` of a SW128 plane.
__device__ __forceinline__ void regs_to_smem_sw128(const uint32_t (&pk)[32], uint8_t* plane, uint32_t row) {
  uint8_t* line = plane + row * 128;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    *reinterpret_cast<uint4*>(line + ((j ^ (row & 7)) << 4)) =
        make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
}

}  // namespace cad_dev
