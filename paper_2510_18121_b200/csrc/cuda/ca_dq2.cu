// dQ on CTA pairs (cta_group::2), for GQA groups of an even size: a pair
// runs two query heads of one KV head on the same q tile (CTA r: head
// head0 + r) and every MMA is M=256 issued by the even CTA:
//   S = Q K^T and dP = dO V^T: A = this CTA's Q / dO tile, B = K / V split by
//     kv rows (CTA r holds kv rows [64r, 64r+64) of the tile, K-major),
//   dQ += dS K: A = dS from TMEM, B = K split by d columns (CTA r holds
//     d columns [64r, 64r+64) of all 128 kv rows, MN-major).
// Each CTA reads half of every B operand from its own shared memory, so the
// operand traffic per MMA drops by a quarter; the pool's B200s are power-
// capped and the CTA-pair forward ran 9 % faster than the single-CTA one.
// Element-wise work is identical to ca_bwd_dq_kernel (ca_bwd.cu); its
// arrivals go to the even CTA's barriers.
#define CAD_KERNEL_TAG "ca_dq2"  // names this file in the mbarrier-timeout report
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "../host/cad_status.hpp"
#include "ca_common.cuh"
#include "ca_mma.cuh"
#include "ca_rows.cuh"
#include "sm100.cuh"

namespace cad_dev {
namespace dq2 {

#ifndef CAD_DQ_EMU_MASK
#define CAD_DQ_EMU_MASK 0x1111  // 25 % of the exp2 pairs on the FMA pipe: measured -1 % (A/B, config 2)
#endif
constexpr uint32_t kDqEmuMask = CAD_DQ_EMU_MASK;
constexpr int kThreads = 384;
#ifndef CAD_DQ2_KSTAGES
#define CAD_DQ2_KSTAGES 3
#endif
#ifndef CAD_DQ2_VSTAGES
#define CAD_DQ2_VSTAGES 2
#endif
constexpr int kKStages = CAD_DQ2_KSTAGES, kVStages = CAD_DQ2_VSTAGES;
constexpr uint32_t kHalfBytes = kTileBytes / 2;  // 16 KB
constexpr uint32_t kQOff = 0;                    // own head: Q, dO (32 KB each)
constexpr uint32_t kDOOff = kTileBytes;
// K stage: [K-major: 64 kv rows x 128 d | MN-major: 128 kv rows x 64 d]
constexpr uint32_t kKOff = 2 * kTileBytes;
constexpr uint32_t kKStageBytes = 2 * kHalfBytes;
constexpr uint32_t kVOff = kKOff + kKStages * kKStageBytes;  // V stage: K-major 64 kv rows x 128 d
// dQ staging: one 16 KB SW128 plane per element-wise warpgroup (its 64 d
// columns of the tile), written out by a TMA store for full tiles
constexpr uint32_t kOStOff = kVOff + kVStages * kHalfBytes;
constexpr uint32_t kBarOff = kOStOff + kTileBytes;
constexpr uint32_t kSmemBytes = kBarOff + 256 + 1024;
static_assert(kSmemBytes <= 232448, "dQ pair shared memory");

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
  // ds_full per dS buffer (j & 1): the element-wise warps can finish dS(j+1)
  // before the MMA warp has observed dS(j) -- S(j+1) and dP(j+1) are issued
  // ahead of that wait -- and one barrier would then complete twice under a
  // lagging waiter, which then sleeps through both phases (a hang seen under
  // multi-GPU memory traffic)
  uint64_t s_full, dp_full, p_read, dp_read, ds_full[2], dq_full, dq_free;
  uint32_t tmem_base;
};

template <int N>
struct Ring {
  uint32_t i = 0, ph = 0;
  __device__ void next() {
    if (++i == N) { i = 0; ph ^= 1; }
  }
};

struct Params {
  CUtensorMap tm_q, tm_do, tm_k64, tm_k, tm_v64, tm_dq;  // *64: 64-row boxes
  const DevTask* tasks;
  const FwdUnit* units;  // nh == 2: heads head0, head0 + 1
  int n_units;
  const int32_t* sched;
  int group;
  int h_q;
  const float* lse2;
  const float* delta;
  __nv_bfloat16* dq;
  int64_t pitch;
  float scale;
  float scale_log2;
};

// D (M=256) = A B^T, A = 128 rows of this CTA (K-major), B = 64 rows per CTA (K-major)
__device__ __forceinline__ void issue_ab_pair(uint32_t d_tmem, uint32_t a_smem, uint32_t b_smem) {
  constexpr uint32_t idesc = idesc_bf16(256, 128, false, false);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t kin = (k & 3) * 32;
    umma_ss_2sm(d_tmem, sw128_desc(a_smem + (k >> 2) * (kTileBytes / 2) + kin, 16, 1024),
                sw128_desc(b_smem + (k >> 2) * (kHalfBytes / 2) + kin, 16, 1024), idesc, k > 0 ? 1u : 0u);
  }
}
// dQ (M=256, N=128 d: 64 per CTA) += dS (TMEM) K (MN-major 128 kv x 64 d per CTA)
__device__ __forceinline__ void issue_dq_pair(uint32_t d_tmem, uint32_t a_lo, uint32_t a_hi, uint32_t k_smem,
                                              bool accumulate) {
  constexpr uint32_t idesc = idesc_bf16(256, 128, false, true);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t a = k < 4 ? a_lo + k * 8 : a_hi + (k - 4) * 8;
    umma_ts_2sm(d_tmem, a, sw128_desc(k_smem + k * 2048, kHalfBytes, 1024), idesc, (accumulate || k > 0) ? 1u : 0u);
  }
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  if (elect_one()) umma_commit_pair(bar);
  __syncwarp();
}

__global__ void __launch_bounds__(kThreads, 1) ca_bwd_dq_pair_kernel(const __grid_constant__ Params p) {
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
    tma_prefetch(&p.tm_do);
    tma_prefetch(&p.tm_k64);
    tma_prefetch(&p.tm_k);
    tma_prefetch(&p.tm_v64);
    mbar_init(&bars->q_full, 2);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&bars->k_full[i], 2);
      mbar_init(&bars->k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
      mbar_init(&bars->v_full[i], 2);
      mbar_init(&bars->v_empty[i], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->p_read, 512);
    mbar_init(&bars->dp_read, 512);
    mbar_init(&bars->ds_full[0], 512);
    mbar_init(&bars->ds_full[1], 512);
    mbar_init(&bars->dq_full, 1);
    mbar_init(&bars->dq_free, 512);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc_2sm<512>(&bars->tmem_base);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const uint32_t tS = tmem, tDP = tmem + 128, tDQ = tmem + 256, tDS = tmem + 384;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (warp == 8 && lane == 0) {
      // ---------------------------------------------------------- producer (both CTAs)
      uint32_t q_it = 0;
      Ring<kKStages> kr;
      Ring<kVStages> vr;
      for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
        const int u = sched_unit(p.sched, n_pairs, ui);
        const FwdUnit un = p.units[u];
        const DevTask tk = p.tasks[un.task];
        const int hk = un.head0 / p.group;
        const int head = un.head0 + int(rank);
        const int qrow = tk.q_off + un.tile * kTile;
        dbg_mark(0, 0x1000 + (ui & 0xfff));
        mbar_wait(&bars->q_empty, (q_it & 1) ^ 1);
        ++q_it;
        if (leader) mbar_expect_tx(&bars->q_full, 4 * kTileBytes);
        else mbar_arrive_leader(&bars->q_full);
        tma_load_3d_2sm(&p.tm_q, &bars->q_full, smem + kQOff, 0, qrow, head);
        tma_load_3d_2sm(&p.tm_q, &bars->q_full, smem + kQOff + kTileBytes / 2, 64, qrow, head);
        tma_load_3d_2sm(&p.tm_do, &bars->q_full, smem + kDOOff, 0, qrow, head);
        tma_load_3d_2sm(&p.tm_do, &bars->q_full, smem + kDOOff + kTileBytes / 2, 64, qrow, head);
        for (int j = 0; j < un.n_kv; ++j) {
          const int krow = tk.kv_off + j * kTile;
          dbg_mark(0, 0x20000 + (j & 0xffff));
          mbar_wait(&bars->k_empty[kr.i], kr.ph ^ 1);
          if (leader) mbar_expect_tx(&bars->k_full[kr.i], 2 * kKStageBytes);
          else mbar_arrive_leader(&bars->k_full[kr.i]);
          uint8_t* kd = smem + kKOff + kr.i * kKStageBytes;
          tma_load_3d_2sm(&p.tm_k64, &bars->k_full[kr.i], kd, 0, krow + 64 * rank, hk);
          tma_load_3d_2sm(&p.tm_k64, &bars->k_full[kr.i], kd + kHalfBytes / 2, 64, krow + 64 * rank, hk);
          tma_load_3d_2sm(&p.tm_k, &bars->k_full[kr.i], kd + kHalfBytes, 64 * rank, krow, hk);
          kr.next();
          dbg_mark(0, 0x30000 + (j & 0xffff));
          mbar_wait(&bars->v_empty[vr.i], vr.ph ^ 1);
          if (leader) mbar_expect_tx(&bars->v_full[vr.i], 2 * kHalfBytes);
          else mbar_arrive_leader(&bars->v_full[vr.i]);
          uint8_t* vd = smem + kVOff + vr.i * kHalfBytes;
          tma_load_3d_2sm(&p.tm_v64, &bars->v_full[vr.i], vd, 0, krow + 64 * rank, hk);
          tma_load_3d_2sm(&p.tm_v64, &bars->v_full[vr.i], vd + kHalfBytes / 2, 64, krow + 64 * rank, hk);
          vr.next();
        }
      }
    } else if (warp == 9 && leader) {
      // ---------------------------------------------------------- MMA (even CTA)
      uint32_t q_it = 0, dq_it = 0, pr_ph = 0, dr_ph = 0, ds_ph[2] = {0, 0};
      Ring<kKStages> kr;
      Ring<kVStages> vr;
      auto sKk = [&](uint32_t i) { return sbase + kKOff + i * kKStageBytes; };
      auto sKm = [&](uint32_t i) { return sbase + kKOff + i * kKStageBytes + kHalfBytes; };
      auto sVk = [&](uint32_t i) { return sbase + kVOff + i * kHalfBytes; };
      for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
        const int u = sched_unit(p.sched, n_pairs, ui);
        const FwdUnit un = p.units[u];
        const int n = un.n_kv;
        dbg_mark(1, 0x10000 + (ui & 0xffff));
        mbar_wait(&bars->q_full, q_it & 1);
        ++q_it;
        const uint32_t sQ = sbase + kQOff, sDO = sbase + kDOOff;
        dbg_mark(1, 0x20000 + (ui & 0xffff));
        mbar_wait(&bars->k_full[kr.i], kr.ph);
        tc_fence_after();
        issue_ab_pair(tS, sQ, sKk(kr.i));  // S(0)
        commit_pair(&bars->s_full);
        mbar_wait(&bars->v_full[vr.i], vr.ph);
        tc_fence_after();
        issue_ab_pair(tDP, sDO, sVk(vr.i));  // dP(0)
        commit_pair(&bars->dp_full);
        commit_pair(&bars->v_empty[vr.i]);
        vr.next();
        if (n == 1) commit_pair(&bars->q_empty);  // Q / dO read for the last time
        for (int j = 0; j < n; ++j) {
          const uint32_t kcur = kr.i;
          kr.next();
          dbg_mark(1, 0x40000 + (j & 0xffff));
          mbar_wait(&bars->p_read, pr_ph);
          pr_ph ^= 1;
          if (j + 1 < n) {
            dbg_mark(1, 0x50000 + (j & 0xffff));
            mbar_wait(&bars->k_full[kr.i], kr.ph);
            tc_fence_after();
            issue_ab_pair(tS, sQ, sKk(kr.i));  // S(j+1)
            commit_pair(&bars->s_full);
          }
          dbg_mark(1, 0x60000 + (j & 0xffff));
          mbar_wait(&bars->dp_read, dr_ph);
          dr_ph ^= 1;
          if (j + 1 < n) {
            dbg_mark(1, 0x70000 + (j & 0xffff));
            mbar_wait(&bars->v_full[vr.i], vr.ph);
            tc_fence_after();
            issue_ab_pair(tDP, sDO, sVk(vr.i));  // dP(j+1)
            commit_pair(&bars->dp_full);
            commit_pair(&bars->v_empty[vr.i]);
            vr.next();
            // last reads of Q / dO issued: the next unit's tiles load under
            // this unit's last exponentials, dQ MMA and epilogue
            if (j + 2 == n) commit_pair(&bars->q_empty);
          }
          dbg_mark(1, 0x80000 + (j & 0xffff));
          mbar_wait(&bars->ds_full[j & 1], ds_ph[j & 1]);
          ds_ph[j & 1] ^= 1;
          if (j == 0) {
            dbg_mark(1, 0x90000 + (ui & 0xffff));
            mbar_wait(&bars->dq_free, (dq_it & 1) ^ 1);
            ++dq_it;
          }
          tc_fence_after();
          const uint32_t ds = tDS + (j & 1) * 64;
          issue_dq_pair(tDQ, ds, ds + 32, sKm(kcur), j > 0);  // dQ += dS K
          commit_pair(&bars->k_empty[kcur]);
        }
        commit_pair(&bars->dq_full);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    const int w = warp >> 2;                    // kv column half [64w, 64w+64)
    const uint32_t r = (warp & 3) * 32 + lane;  // q row within the tile
    const uint32_t lsel = ((warp & 3) * 32) << 16;
    const int c0 = 64 * w;
    uint32_t s_ph = 0, dp_ph = 0, dq_ph = 0;
    for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
      const int u = sched_unit(p.sched, n_pairs, ui);
      const FwdUnit un = p.units[u];
      const DevTask tk = p.tasks[un.task];
      const int shift = tk.kv_len - tk.n_q;
      const int qi = un.tile * kTile + r;
      const bool valid = qi < tk.n_q;
      const int64_t row = int64_t(tk.q_off) + qi;
      const int head = un.head0 + int(rank);  // this CTA's query head
      const float lse2 = valid ? -p.lse2[int64_t(head) * p.pitch + row] : 0.f;
      const float dd = valid ? -p.delta[int64_t(head) * p.pitch + row] : 0.f;
      const int pos = valid ? shift + qi : -1;  // invalid rows see nothing
      const bool all_rows = un.tile * kTile + kTile <= tk.n_q;
      for (int j = 0; j < un.n_kv; ++j) {
        if (r == 0) dbg_mark(2 + w, 0x10000 + (j & 0xffff));
        mbar_wait_warp(&bars->s_full, s_ph);
        s_ph ^= 1;
        tc_fence_after();
        float x[64];
        load_row64(tS + lsel + c0, x);
        tc_fence_before();
        mbar_arrive_leader(&bars->p_read);
        const int lim = pos - (j * kTile + c0);  // last visible column
        // mask-free (CTA-uniform) when every row of the tile is a query and
        // its first row already sees this warpgroup's last column
        const bool full = all_rows && shift + un.tile * kTile - (j * kTile + c0) >= 63;
        const uint64_t sc2 = f2(p.scale_log2, p.scale_log2), nl2 = f2(-lse2, -lse2);
#pragma unroll
        for (int k = 0; k < 64; k += 2) {
          float a, b;
          f2_split(ffma2(f2(x[k], x[k + 1]), sc2, nl2), a, b);
          if ((kDqEmuMask >> (k / 4)) & 1) {
            exp2_fma2(a, b);
          } else {
            a = ex2(a);
            b = ex2(b);
          }
          x[k] = a;
          x[k + 1] = b;
        }
        if (!full) {
#pragma unroll
          for (int k = 0; k < 64; ++k) x[k] = k <= lim ? x[k] : 0.f;
        }
        if (r == 0) dbg_mark(2 + w, 0x20000 + (j & 0xffff));
        mbar_wait_warp(&bars->dp_full, dp_ph);
        dp_ph ^= 1;
        tc_fence_after();
        float y[64];
        load_row64(tDP + lsel + c0, y);
        tc_fence_before();
        mbar_arrive_leader(&bars->dp_read);
        const uint64_t nd2 = f2(-dd, -dd);
#pragma unroll
        for (int k = 0; k < 64; k += 2)
          f2_split(fmul2(f2(x[k], x[k + 1]), fadd2(f2(y[k], y[k + 1]), nd2)), y[k], y[k + 1]);
        store_bf16_64(tDS + lsel + (j & 1) * 64 + 32 * w, y);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive_leader(&bars->ds_full[j & 1]);
      }
      if (r == 0) dbg_mark(2 + w, 0x30000 + (ui & 0xffff));
      mbar_wait_warp(&bars->dq_full, dq_ph);
      dq_ph ^= 1;
      tc_fence_after();
      if (all_rows) {
        uint8_t* st = smem + kOStOff + w * (kTileBytes / 2);
        if (r == 0) bulk_wait_read0();  // the previous unit's store has read the staging
        named_sync(1 + w, 128);
        tmem_row_to_smem_sw128(tDQ + lsel + c0, p.scale, st, r);
        fence_proxy_async_smem();
        named_sync(1 + w, 128);
        if (r == 0) {
          tma_store_3d(&p.tm_dq, st, c0, tk.q_off + un.tile * kTile, head);
          bulk_commit();
        }
      } else {
        tmem_row_to_global(tDQ + lsel + c0, p.scale, p.dq + (row * p.h_q + head) * kHeadDim + c0, valid);
      }
      tc_fence_before();
      mbar_arrive_leader(&bars->dq_free);
    }
  }
  if (warp < 8 && (warp & 3) == 0 && lane == 0) bulk_wait0();  // dQ staging read + stores done
  tc_fence_before();
  cluster_sync_all();
  if (warp == 9) tmem_free_2sm<512>(tmem);
}

}  // namespace dq2

void preload_dq2() {
  set_max_smem(reinterpret_cast<const void*>(dq2::ca_bwd_dq_pair_kernel), dq2::kSmemBytes,
               "cudaFuncSetAttribute(dq2)");
}

// Launch of the pair dQ kernel (cluster dims 2); false if the plan has no pair units.
bool launch_dq_pair(const cad_ca_plan* plan, const void* q, const void* k, const void* v, const void* dout,
                    const float* lse2, const float* delta, int64_t pitch, void* dq, cudaStream_t stream) {
  if (plan->dq2_units.empty()) return false;
  const cad_ca_shape& sh = plan->shape;
  dq2::Params p;
  make_tile_map(&p.tm_q, q, sh.q_rows, sh.h_q);
  make_tile_map(&p.tm_do, dout, sh.q_rows, sh.h_q);
  make_tile_map(&p.tm_k64, k, sh.kv_rows, sh.h_kv, 64);
  make_tile_map(&p.tm_k, k, sh.kv_rows, sh.h_kv);
  make_tile_map(&p.tm_v64, v, sh.kv_rows, sh.h_kv, 64);
  make_tile_map(&p.tm_dq, dq, sh.q_rows, sh.h_q);
  p.tasks = plan->d_tasks;
  p.units = plan->d_dq2;
  p.n_units = static_cast<int>(plan->dq2_units.size());
  p.sched = plan->sched_dq2.d;
  p.group = sh.h_q / sh.h_kv;
  p.h_q = sh.h_q;
  p.lse2 = lse2;
  p.delta = delta;
  p.dq = static_cast<__nv_bfloat16*>(dq);
  p.pitch = pitch;
  p.scale = sh.softmax_scale;
  p.scale_log2 = sh.softmax_scale * 1.4426950408889634f;
  set_max_smem(reinterpret_cast<const void*>(dq2::ca_bwd_dq_pair_kernel), dq2::kSmemBytes,
               "cudaFuncSetAttribute(dq2)");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * plan->sched_dq2.G);
  cfg.blockDim = dim3(dq2::kThreads);
  cfg.dynamicSmemBytes = dq2::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, dq2::ca_bwd_dq_pair_kernel, p), "ca_bwd_dq_pair launch");
  return true;
}

}  // namespace cad_dev
