// The two tcgen05 MMA shapes every CA kernel is built from (all tiles
// 128 x 128 bf16, SW128 planes of 64 d-values as TMA lands them):
//   issue_qk: D  = A B^T with A, B both K-major (row tiles, d contiguous):
//             S = Q K^T (fwd, dq), S^T = K Q^T and dP^T = V dO^T (dkdv),
//             dP = dO V^T (dq).
//   issue_pv: D += A B with A = bf16 operand in TMEM (2 values per column,
//             lane = output row) and B an MN-major row tile:
//             O += P V (fwd), dV += P^T dO and dK += dS^T Q (dkdv),
//             dQ += dS K (dq).
#pragma once

#include "ca_common.cuh"
#include "sm100.cuh"

namespace cad_dev {

// The issue helpers are called by the whole (converged) MMA warp, so the
// descriptors stay warp-uniform (uniform registers); one elect.sync-chosen
// lane issues the tcgen05 ops and the commits. (Issuing from a lane-0-only
// branch makes ptxas wrap every UTCHMMA in an R2UR/ELECT waterfall loop:
// ~100 cycles per MMA, which throttled the tensor pipe.)

// D = A B^T: M=128, N=128, K=128 (d) as 8 steps of 16.
__device__ __forceinline__ void issue_qk(uint32_t d_tmem, uint32_t a_smem, uint32_t b_smem) {
  constexpr uint32_t idesc = idesc_bf16(128, 128, false, false);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t off = (k >> 2) * (kTileBytes / 2) + (k & 3) * 32;
    umma_ss(d_tmem, sw128_desc(a_smem + off, 16, 1024), sw128_desc(b_smem + off, 16, 1024), idesc,
            k > 0 ? 1u : 0u);
  }
}

// D (+)= A B: M=128, N=128 (d), K=128 as 8 steps of 16. A (bf16 in TMEM):
// k-steps 0-3 read columns a_lo + 8k, steps 4-7 read a_hi + 8(k-4), so the
// two 64-wide K halves may live in separate TMEM column ranges. B is
// MN-major (d contiguous): LBO = 16 KB between the two 64-wide d planes,
// SBO = 1 KB per 8 rows of K.
__device__ __forceinline__ void issue_pv(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi,
                                         uint32_t b_smem, bool accumulate) {
  constexpr uint32_t idesc = idesc_bf16(128, 128, false, true);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t a = k < 4 ? a_lo + k * 8 : a_hi + (k - 4) * 8;
    umma_ts(d_tmem, a, sw128_desc(b_smem + k * 2048, kTileBytes / 2, 1024), idesc,
            (accumulate || k > 0) ? 1u : 0u);
  }
}

// One K-half (kv rows [64*half, 64*half+64)) of issue_pv: P released in halves.
__device__ __forceinline__ void issue_pv_half(uint32_t d_tmem, uint32_t a, uint32_t b_smem, int half,
                                              bool accumulate) {
  constexpr uint32_t idesc = idesc_bf16(128, 128, false, true);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    umma_ts(d_tmem, a + k * 8, sw128_desc(b_smem + (half * 4 + k) * 2048, kTileBytes / 2, 1024), idesc,
            (accumulate || half > 0 || k > 0) ? 1u : 0u);
}

// D = A B^T with a 128-row A tile and an N-row B tile (N = 64 or 128),
// K = 128 (d). Each operand is two SW128 planes of 64 d-values; a plane of
// an R-row tile is R*128 bytes.
template <int N>
__device__ __forceinline__ void issue_qk_n(uint32_t d_tmem, uint32_t a_smem, uint32_t b_smem) {
  constexpr uint32_t idesc = idesc_bf16(128, N, false, false);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t kin = (k & 3) * 32;
    umma_ss(d_tmem, sw128_desc(a_smem + (k >> 2) * (kTileBytes / 2) + kin, 16, 1024),
            sw128_desc(b_smem + (k >> 2) * (N * 128) + kin, 16, 1024), idesc, k > 0 ? 1u : 0u);
  }
}

// D (+)= A B with K = KR rows of an MN-major B tile (KR x 128 d, two planes
// of KR*128 bytes) and A (bf16, M=128 lanes) in TMEM columns a + 8k.
template <int KR>
__device__ __forceinline__ void issue_pv_k(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_smem,
                                           bool accumulate) {
  constexpr uint32_t idesc = idesc_bf16(128, 128, false, true);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < KR / 16; ++k) {
    umma_ts(d_tmem, a_tmem + k * 8, sw128_desc(b_smem + k * 2048, KR * 128, 1024), idesc,
            (accumulate || k > 0) ? 1u : 0u);
  }
}

// Warp-level commit by the elected (issuing) lane.
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  if (elect_one()) umma_commit(bar);
  __syncwarp();
}

}  // namespace cad_dev
