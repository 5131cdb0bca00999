// CA forward on a CTA pair (cluster of 2, tcgen05 .cta_group::2).
//
// Same algorithm as ca_fwd.cu (online softmax, lazy rescale, bottom-right
// causal mask of P/src/oracle.cpp:50-54), but the S = Q K^T and O += P V
// MMAs are M=256 pair instructions issued by the even CTA: each CTA supplies
// its own 128 query rows (A) and HALF of the B operand (64 kv rows of K for
// S, 64 d-columns of V for PV). A 128x128 SS MMA on one SM reads 8 KB of
// shared memory per 64 cycles, which is the SM's whole shared-memory
// bandwidth (measured: scripts/micro/umma_rate.cu); the pair form reads 6 KB,
// leaving room for the TMA traffic and halving the K/V bytes each SM loads.
//
// A pair serves 4 query heads of one KV head (GQA group >= 4): CTA r holds
// heads head0 + 2r + {0,1} in its two softmax warpgroups, exactly like the
// single-CTA kernel; TMEM per CTA: S0 S1 O0 O1 (512 columns).
#define CAD_KERNEL_TAG "ca_fwd2"  // names this file in the mbarrier-timeout report
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "../host/cad_status.hpp"
#include "ca_common.cuh"
#include "ca_mma.cuh"
#include "ca_softmax.cuh"
#include "sm100.cuh"

namespace cad_dev {
namespace fwd2 {

#ifndef CAD_EMU_MASK
#define CAD_EMU_MASK 0x1111
#endif
constexpr uint32_t kPairEmuMask = CAD_EMU_MASK;  // 4 of 16 exp2 pairs on the FMA pipe (measured best)
constexpr int kThreads = 384;
#ifndef CAD_FWD2_TMA_STORE
#define CAD_FWD2_TMA_STORE 1
#endif
#ifndef CAD_FWD2_STAGES
#define CAD_FWD2_STAGES 3
#endif
constexpr int kStages = CAD_FWD2_STAGES;
constexpr uint32_t kHalfBytes = kTileBytes / 2;           // 16 KB: half a K or V tile
constexpr uint32_t kQOff = 0;                             // 2 x 32 KB
constexpr uint32_t kKOff = 2 * kTileBytes;                // kStages x 16 KB (64 kv rows x 128 d)
constexpr uint32_t kVOff = kKOff + kStages * kHalfBytes;  // kStages x 16 KB (128 kv rows x 64 d)
// O staging per softmax warpgroup (head): 128 rows x 128 d bf16 as two
// SW128 planes, written out by TMA stores (coalesced, asynchronous); rows
// of a partial last tile go out with per-thread stores instead.
constexpr uint32_t kOStOff = kVOff + kStages * kHalfBytes;
constexpr uint32_t kBarOff = kOStOff + (CAD_FWD2_TMA_STORE ? 2 * kTileBytes : 0);
constexpr uint32_t kSmemBytes = kBarOff + 256 + 1024;

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
  uint64_t s_full[2], p_half[2], p_full[2], o_full[2], o_free[2];
  uint32_t tmem_base;
};

struct Params {
  CUtensorMap tm_q, tm_k64, tm_v, tm_o;  // tm_k64: 64-row boxes
  const DevTask* tasks;
  const FwdUnit* units;  // nh == 4: heads head0..head0+3
  int n_units;
  const int32_t* sched;  // per-CTA work lists (CtaLists)
  int h_q;
  int group;
  __nv_bfloat16* o;
  float* lse;
  int64_t q_rows;
  float scale_log2;
};

// S = Q K^T, M=256 (128 q rows per CTA), N=128 kv rows (64 per CTA), K=128.
__device__ __forceinline__ void issue_qk_pair(uint32_t d_tmem, uint32_t q_smem, uint32_t k_smem) {
  constexpr uint32_t idesc = idesc_bf16(256, 128, false, false);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t kin = (k & 3) * 32;
    umma_ss_2sm(d_tmem, sw128_desc(q_smem + (k >> 2) * (kTileBytes / 2) + kin, 16, 1024),
                sw128_desc(k_smem + (k >> 2) * (kHalfBytes / 2) + kin, 16, 1024), idesc, k > 0 ? 1u : 0u);
  }
}

// O += P V for one K-half (kv rows [64*half, 64*half+64)): M=256, N=128 d
// (64 per CTA: one MN-major plane); P from TMEM.
__device__ __forceinline__ void issue_pv_pair_half(uint32_t d_tmem, uint32_t p, uint32_t v_smem, int half,
                                                   bool accumulate) {
  constexpr uint32_t idesc = idesc_bf16(256, 128, false, true);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    umma_ts_2sm(d_tmem, p + k * 8, sw128_desc(v_smem + (half * 4 + k) * 2048, kHalfBytes, 1024), idesc,
                (accumulate || half > 0 || k > 0) ? 1u : 0u);
}

__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  if (elect_one()) umma_commit_pair(bar);
  __syncwarp();
}

__global__ void __launch_bounds__(kThreads, 1) ca_fwd_pair_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars* bars = reinterpret_cast<Bars*>(smem + kBarOff);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&p.tm_q);
    tma_prefetch(&p.tm_k64);
    tma_prefetch(&p.tm_v);
    mbar_init(&bars->q_full, 2);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&bars->k_full[i], 2);
      mbar_init(&bars->k_empty[i], 1);
      mbar_init(&bars->v_full[i], 2);
      mbar_init(&bars->v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_half[i], 256);
      mbar_init(&bars->p_full[i], 256);
      mbar_init(&bars->o_full[i], 1);
      mbar_init(&bars->o_free[i], 256);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc_2sm<512>(&bars->tmem_base);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == 8) {
      // ---------------------------------------------------------- producer (both CTAs)
      if (lane == 0) {
        uint32_t q_it = 0, ks = 0, kph = 0, vs = 0, vph = 0;
        for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
          const int u = sched_unit(p.sched, n_pairs, ui);
          const FwdUnit un = p.units[u];
          const DevTask tk = p.tasks[un.task];
          const int hk = un.head0 / p.group;
          mbar_wait(&bars->q_empty, (q_it & 1) ^ 1);
          ++q_it;
          if (leader) mbar_expect_tx(&bars->q_full, 4 * kTileBytes);
          else mbar_arrive_leader(&bars->q_full);
          const int qrow = tk.q_off + un.tile * kTile;
          for (int s = 0; s < 2; ++s) {
            uint8_t* dst = smem + kQOff + s * kTileBytes;
            const int head = un.head0 + 2 * rank + s;
            tma_load_3d_2sm(&p.tm_q, &bars->q_full, dst, 0, qrow, head);
            tma_load_3d_2sm(&p.tm_q, &bars->q_full, dst + kTileBytes / 2, 64, qrow, head);
          }
          for (int j = 0; j < un.n_kv; ++j) {
            const int krow = tk.kv_off + j * kTile;
            mbar_wait(&bars->k_empty[ks], kph ^ 1);
            if (leader) mbar_expect_tx(&bars->k_full[ks], 2 * kHalfBytes);
            else mbar_arrive_leader(&bars->k_full[ks]);
            uint8_t* kd = smem + kKOff + ks * kHalfBytes;
            tma_load_3d_2sm(&p.tm_k64, &bars->k_full[ks], kd, 0, krow + 64 * rank, hk);
            tma_load_3d_2sm(&p.tm_k64, &bars->k_full[ks], kd + kHalfBytes / 2, 64, krow + 64 * rank, hk);
            if (++ks == kStages) { ks = 0; kph ^= 1; }
            mbar_wait(&bars->v_empty[vs], vph ^ 1);
            if (leader) mbar_expect_tx(&bars->v_full[vs], 2 * kHalfBytes);
            else mbar_arrive_leader(&bars->v_full[vs]);
            tma_load_3d_2sm(&p.tm_v, &bars->v_full[vs], smem + kVOff + vs * kHalfBytes, 64 * rank, krow, hk);
            if (++vs == kStages) { vs = 0; vph ^= 1; }
          }
        }
      }
    } else if (warp == 9 && leader) {
      // ---------------------------------------------------------- MMA (even CTA)
      uint32_t q_it = 0, ks = 0, kph = 0, vs = 0, vph = 0;
      uint32_t pph[2] = {0, 0}, fph[2] = {0, 0};
      for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
        const int u = sched_unit(p.sched, n_pairs, ui);
        const FwdUnit un = p.units[u];
        const int n = un.n_kv;
        mbar_wait(&bars->q_full, q_it & 1);
        ++q_it;
        mbar_wait(&bars->k_full[ks], kph);
        tc_fence_after();
        for (int h = 0; h < 2; ++h) {
          issue_qk_pair(tmem + h * 128, sbase + kQOff + h * kTileBytes, sbase + kKOff + ks * kHalfBytes);
          commit_pair(&bars->s_full[h]);
        }
        commit_pair(&bars->k_empty[ks]);
        if (++ks == kStages) { ks = 0; kph ^= 1; }
        if (n == 1) commit_pair(&bars->q_empty);
        for (int j = 0; j < n; ++j) {
          mbar_wait(&bars->v_full[vs], vph);
          tc_fence_after();
          for (int h = 0; h < 2; ++h) {
            mbar_wait(&bars->p_half[h], pph[h]);
            if (j == 0) {
              mbar_wait(&bars->o_free[h], fph[h] ^ 1);
              fph[h] ^= 1;
            }
            tc_fence_after();
            issue_pv_pair_half(tmem + 256 + h * 128, tmem + h * 128, sbase + kVOff + vs * kHalfBytes, 0, j > 0);
            mbar_wait(&bars->p_full[h], pph[h]);
            pph[h] ^= 1;
            tc_fence_after();
            issue_pv_pair_half(tmem + 256 + h * 128, tmem + h * 128 + 32, sbase + kVOff + vs * kHalfBytes, 1, true);
            if (j == n - 1) {
              commit_pair(&bars->o_full[h]);
            } else {
              if (h == 0) {
                mbar_wait(&bars->k_full[ks], kph);
                tc_fence_after();
              }
              issue_qk_pair(tmem + h * 128, sbase + kQOff + h * kTileBytes, sbase + kKOff + ks * kHalfBytes);
              commit_pair(&bars->s_full[h]);
            }
          }
          commit_pair(&bars->v_empty[vs]);
          if (++vs == kStages) { vs = 0; vph ^= 1; }
          if (j < n - 1) {
            commit_pair(&bars->k_empty[ks]);
            if (++ks == kStages) { ks = 0; kph ^= 1; }
            if (j + 1 == n - 1) commit_pair(&bars->q_empty);
          }
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ------------------------------------------------------------ softmax (both CTAs)
    const int h = warp >> 2;
    const uint32_t row = (warp & 3) * 32 + lane;
    const uint32_t lane_sel = ((warp & 3) * 32) << 16;
    const uint32_t s_tmem = tmem + lane_sel + h * 128;
    const uint32_t o_tmem = tmem + lane_sel + 256 + h * 128;
    uint32_t sph = 0, oph = 0;
    for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
      const int u = sched_unit(p.sched, n_pairs, ui);
      const FwdUnit un = p.units[u];
      const DevTask tk = p.tasks[un.task];
      const int shift = tk.kv_len - tk.n_q;
      const int qi = un.tile * kTile + row;
      const int pos = shift + qi;
      const int first_masked_tile = (shift + un.tile * kTile) >> 7;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < un.n_kv; ++j) {
        mbar_wait_warp(&bars->s_full[h], sph);
        sph ^= 1;
        tc_fence_after();
        softmax_tile<kPairEmuMask>(s_tmem, o_tmem, j == 0, j >= first_masked_tile, pos - j * kTile, p.scale_log2, m, l,
                     [&](int half) { mbar_arrive_leader(half ? &bars->p_full[h] : &bars->p_half[h]); });
      }
      mbar_wait_warp(&bars->o_full[h], oph);
      oph ^= 1;
      tc_fence_after();
      const bool valid = qi < tk.n_q;
      const float inv = 1.f / l;
      const int head = un.head0 + 2 * rank + h;
      __nv_bfloat16* orow = p.o + ((int64_t)(tk.q_off + qi) * p.h_q + head) * kHeadDim;
      const bool full_tile = un.tile * kTile + kTile <= tk.n_q;  // uniform over the warpgroup
      if (CAD_FWD2_TMA_STORE && full_tile) {
        // stage the normalised rows in SW128 planes, one TMA store per plane
        uint8_t* st = smem + kOStOff + h * kTileBytes;
        if (row == 0) bulk_wait_read0();  // the previous unit's stores have read the staging
        named_sync(1 + h, 128);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld32(o_tmem + c * 32, r);
          tmem_wait_ld();
          uint4 w[4];
          uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            wp[i] = pack_bf16(__uint_as_float(r[2 * i]) * inv, __uint_as_float(r[2 * i + 1]) * inv);
          uint8_t* plane = st + (c >> 1) * (kTileBytes / 2) + row * 128;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            *reinterpret_cast<uint4*>(plane + ((((c & 1) * 4 + i) ^ (row & 7)) << 4)) = w[i];
        }
        fence_proxy_async_smem();
        named_sync(1 + h, 128);
        if (row == 0) {
          const int qrow0 = tk.q_off + un.tile * kTile;
          tma_store_3d(&p.tm_o, st, 0, qrow0, head);
          tma_store_3d(&p.tm_o, st + kTileBytes / 2, 64, qrow0, head);
          bulk_commit();
        }
      } else {
        // partial last tile of a task: per-thread stores of the valid rows
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld32(o_tmem + c * 32, r);
          tmem_wait_ld();
          uint4 w[4];
          uint32_t* wp = reinterpret_cast<uint32_t*>(w);
#pragma unroll
          for (int i = 0; i < 16; ++i)
            wp[i] = pack_bf16(__uint_as_float(r[2 * i]) * inv, __uint_as_float(r[2 * i + 1]) * inv);
          if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
            for (int i = 0; i < 4; ++i) dst[i] = w[i];
          }
        }
      }
      if (valid) p.lse[(int64_t)head * p.q_rows + tk.q_off + qi] = (m + __log2f(l)) * 0.69314718055994531f;
      tc_fence_before();
      mbar_arrive_leader(&bars->o_free[h]);
    }
  }

  if (CAD_FWD2_TMA_STORE && warp < 8 && (warp & 3) == 0 && lane == 0) bulk_wait0();  // staging read + stores done
  tc_fence_before();
  cluster_sync_all();
  if (warp == 9) tmem_free_2sm<512>(tmem);
}

}  // namespace fwd2

void preload_fwd2() {
  set_max_smem(reinterpret_cast<const void*>(fwd2::ca_fwd_pair_kernel), fwd2::kSmemBytes,
               "cudaFuncSetAttribute(fwd2)");
}

// Launch of the pair kernel (cluster dims 2); false if this plan has no pair units.
bool launch_fwd_pair(const cad_ca_plan* plan, const void* q, const void* k, const void* v, void* o, float* lse,
                     cudaStream_t stream) {
  if (plan->fwd2_units.empty()) return false;
  fwd2::Params p;
  make_tile_map(&p.tm_q, q, plan->shape.q_rows, plan->shape.h_q);
  make_tile_map(&p.tm_k64, k, plan->shape.kv_rows, plan->shape.h_kv, 64);
  make_tile_map(&p.tm_v, v, plan->shape.kv_rows, plan->shape.h_kv);
  make_tile_map(&p.tm_o, o, plan->shape.q_rows, plan->shape.h_q);
  p.tasks = plan->d_tasks;
  p.units = plan->d_fwd2;
  p.n_units = static_cast<int>(plan->fwd2_units.size());
  p.sched = plan->sched_fwd2.d;
  p.h_q = plan->shape.h_q;
  p.group = plan->shape.h_q / plan->shape.h_kv;
  p.o = static_cast<__nv_bfloat16*>(o);
  p.lse = lse;
  p.q_rows = plan->shape.q_rows;
  p.scale_log2 = plan->shape.softmax_scale * 1.4426950408889634f;
  set_max_smem(reinterpret_cast<const void*>(fwd2::ca_fwd_pair_kernel), fwd2::kSmemBytes,
               "cudaFuncSetAttribute(fwd2)");
  const int pairs = plan->sched_fwd2.G;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(fwd2::kThreads);
  cfg.dynamicSmemBytes = fwd2::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, fwd2::ca_fwd_pair_kernel, p), "ca_fwd_pair launch");
  return true;
}

}  // namespace cad_dev
