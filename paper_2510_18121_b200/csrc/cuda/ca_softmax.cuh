// Online-softmax step of the CA forward for one 128 x 128 S tile held in TMEM
// (thread = query row), shared by the single-CTA and the CTA-pair forward.
//
// Per tile and thread: 128 FP32 scores -> row max (FMNMX3 tree) -> 128
// exponentials in the log2 domain -> bf16 P written back over the first 64
// columns of S. B200's MUFU retires 16 ex2/clk/SM, exactly the tensor-core
// time of the QK^T + PV pair for the same tile, so a fixed subset of the
// exponentials (kEmuMask, one bit per column pair of a 32-column chunk) runs
// as a degree-3 polynomial on the FMA pipe (exp2_fma2, rel. err < 1e-4,
// below the bf16 rounding of P). P is released in two halves: after kv
// columns [0,64) the caller's release(0) lets the MMA warp start the first
// K-half of O += P V while the second half is still being exponentiated.
//
// Math is the reference's causal-softmax definition (P/src/oracle.cpp:50-54)
// with lazy rescaling: the running max m only moves when a tile's max exceeds
// it by more than 2^8, in which case O (TMEM) and l are rescaled first.
#pragma once

#include "sm100.cuh"

#ifndef SOFTMAX_TL
#define SOFTMAX_TL(ev, it)
#endif

namespace cad_dev {

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// kEmuMask: 16 bits, one per column pair of a 32-column chunk; 1 = that pair
// uses the polynomial exp2. The CTA-pair forward runs best with 4 of 16 pairs
// (0x1111, measured), the single-CTA forward with none.
template <uint32_t kEmuMask, class Release>
__device__ __forceinline__ void softmax_tile(uint32_t s_tmem, uint32_t o_tmem, bool first, bool masked,
                                             int limit, float scale_log2, float& m, float& l,
                                             Release&& release, int tl = 0) {
  float s[128];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t r[32];
    tmem_ld32(s_tmem + c * 32, r);
#pragma unroll
    for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(r[i]);
  }
  tmem_wait_ld();
  SOFTMAX_TL(5, tl);
  if (masked) {
#pragma unroll
    for (int c = 0; c < 128; ++c)
      if (c > limit) s[c] = -INFINITY;
  }
  // Row max: 8 independent FMNMX3 chains, then a 3-level tree.
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = s[i];
#pragma unroll
  for (int r = 0; r < 60; ++r) acc[r & 7] = fmax3(acc[r & 7], s[8 + 2 * r], s[9 + 2 * r]);
  const float mx = fmax3(fmax3(acc[0], acc[1], acc[2]), fmax3(acc[3], acc[4], acc[5]), fmaxf(acc[6], acc[7]));
  const float m_tile = mx * scale_log2;
  SOFTMAX_TL(6, tl);
  if (first) {
    m = m_tile;
  } else if (m_tile > m + 8.0f) {
    const float f = ex2(m - m_tile);
    l *= f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t r[32];
      tmem_ld32(o_tmem + c * 32, r);
      tmem_wait_ld();
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * f);
      tmem_st32(o_tmem + c * 32, r);
    }
    m = m_tile;
  }
  const uint64_t sc2 = f2(scale_log2, scale_log2), nm2 = f2(-m, -m);
  uint64_t sum0 = f2(0.f, 0.f), sum1 = sum0;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t pk[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float a, b;
      f2_split(ffma2(f2(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), sc2, nm2), a, b);
      if ((kEmuMask >> i) & 1) {
        exp2_fma2(a, b);
      } else {
        a = ex2(a);
        b = ex2(b);
      }
      if (i & 1) sum1 = fadd2(sum1, f2(a, b));
      else sum0 = fadd2(sum0, f2(a, b));
      pk[i] = pack_bf16(a, b);
    }
    tmem_st16(s_tmem + c * 16, pk);
    if (c == 1) {
      tmem_wait_st();
      tc_fence_before();
      release(0);
      SOFTMAX_TL(7, tl);
    }
  }
  float s0, s1, s2, s3;
  f2_split(sum0, s0, s1);
  f2_split(sum1, s2, s3);
  l += (s0 + s1) + (s2 + s3);
  tmem_wait_st();
  tc_fence_before();
  release(1);
}

}  // namespace cad_dev
