// CA forward on sm_100a: O = softmax(scale * Q K^T + bottom-right causal
// mask) V and LSE, over a list of document-packed CA-tasks.
//
// Replaces the analytical kernel stand-in task_layer_seconds ->
// profile_lookup (P/src/sim.cpp:22-30, P/src/cost.cpp:149-162); the mask is
// the reference's causal pair definition (P/src/oracle.cpp:50-54): query i of
// a task sees keys 0 .. kv_len - n_q + i.
//
// Structure (one persistent CTA per SM, 12 warps):
//   warp 8      TMA producer: Q tiles of the unit, then a 2-deep ring of K
//               and a 2-deep ring of V tiles (128 kv rows x 128 d, SW128).
//   warp 9      MMA issuer (one thread): S_h = Q_h K^T into TMEM, then
//               O_h += P_h V with P_h read from TMEM (tcgen05 .kind::f16,
//               BF16 in, FP32 accumulate).
//   warps 0-7   two softmax warpgroups, one per query head of the unit
//               (GQA: both heads share the K/V tiles). Thread = query row:
//               the S row is read from TMEM, masked, exponentiated (online
//               softmax in the log2 domain with lazy rescaling), written back
//               as bf16 P into the S columns, and at the end O/l and the LSE
//               are written out.
// TMEM (512 columns): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
// The MMA order PV_h(j) -> S_h(j+1) lets softmax h overlap with the other
// head's MMAs (ping-pong across the two heads).
#define CAD_KERNEL_TAG "ca_fwd"  // names this file in the mbarrier-timeout report
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "../host/cad_status.hpp"
#include "ca_common.cuh"
#include "ca_mma.cuh"
#include "ca_softmax.cuh"
#include "sm100.cuh"

namespace cad_dev {

namespace fwd {

#ifndef CAD_EMU_MASK
#define CAD_EMU_MASK 0x0000
#endif
constexpr uint32_t kFwdEmuMask = CAD_EMU_MASK;  // no polynomial exp2 (measured best)
constexpr int kThreads = 384;  // softmax warpgroups 0,1 + control warpgroup (TMA, MMA, 2 idle)
constexpr uint32_t kQOff = 0;                   // 2 x 32 KB
constexpr uint32_t kKOff = 2 * kTileBytes;      // 2 x 32 KB
constexpr uint32_t kVOff = 4 * kTileBytes;      // 2 x 32 KB
constexpr uint32_t kBarOff = 6 * kTileBytes;
constexpr uint32_t kSmemBytes = kBarOff + 256 + 1024;  // + barriers + alignment slack

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[2], k_empty[2], v_full[2], v_empty[2];
  uint64_t s_full[2], p_half[2], p_full[2], o_full[2], o_free[2];
  uint32_t tmem_base;
};

struct Params {
  CUtensorMap tm_q, tm_k, tm_v;
  const DevTask* tasks;
  const FwdUnit* units;
  int n_units;
  const int32_t* sched;  // per-CTA work lists (CtaLists)
  int h_q;
  int group;  // h_q / h_kv
  __nv_bfloat16* o;
  float* lse;
  int64_t q_rows;
  float scale_log2;  // softmax scale * log2(e)
};

__global__ void __launch_bounds__(kThreads, 1) ca_fwd_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars* bars = reinterpret_cast<Bars*>(smem + kBarOff);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 8 && lane == 0) {
    tma_prefetch(&p.tm_q);
    tma_prefetch(&p.tm_k);
    tma_prefetch(&p.tm_v);
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->k_full[i], 1);
      mbar_init(&bars->k_empty[i], 1);
      mbar_init(&bars->v_full[i], 1);
      mbar_init(&bars->v_empty[i], 1);
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_half[i], 128);
      mbar_init(&bars->p_full[i], 128);
      mbar_init(&bars->o_full[i], 1);
      mbar_init(&bars->o_free[i], 128);
    }
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp >= 8) {
    // Control warpgroup: hand registers to the softmax warpgroups. The CTA
    // pool holds 384 x 168 registers; 4 warps giving back 112 each fund 8
    // warps taking 56 more each (168 -> 224).
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (warp == 8) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      uint32_t q_it = 0, ks = 0, kph = 0, vs = 0, vph = 0;
      for (int ui = sched_begin(p.sched, blockIdx.x); ui < sched_end(p.sched, blockIdx.x); ++ui) {
        const int u = sched_unit(p.sched, gridDim.x, ui);
        const FwdUnit un = p.units[u];
        const DevTask tk = p.tasks[un.task];
        const int hk = un.head0 / p.group;  // the KV head shared by the unit's query heads
        dbg_mark(0, 0x100);
        mbar_wait(&bars->q_empty, (q_it & 1) ^ 1);
        mbar_expect_tx(&bars->q_full, un.nh * kTileBytes);
        const int qrow = tk.q_off + un.tile * kTile;
        for (int h = 0; h < un.nh; ++h) {
          uint8_t* dst = smem + kQOff + h * kTileBytes;
          tma_load_3d(&p.tm_q, &bars->q_full, dst, 0, qrow, un.head0 + h);
          tma_load_3d(&p.tm_q, &bars->q_full, dst + kTileBytes / 2, 64, qrow, un.head0 + h);
        }
        ++q_it;
        for (int j = 0; j < un.n_kv; ++j) {
          const int krow = tk.kv_off + j * kTile;
          dbg_mark(0, 0x200 + j);
          mbar_wait(&bars->k_empty[ks], kph ^ 1);
          mbar_expect_tx(&bars->k_full[ks], kTileBytes);
          uint8_t* kd = smem + kKOff + ks * kTileBytes;
          tma_load_3d(&p.tm_k, &bars->k_full[ks], kd, 0, krow, hk);
          tma_load_3d(&p.tm_k, &bars->k_full[ks], kd + kTileBytes / 2, 64, krow, hk);
          if (++ks == 2) { ks = 0; kph ^= 1; }
          dbg_mark(0, 0x300 + j);
          mbar_wait(&bars->v_empty[vs], vph ^ 1);
          mbar_expect_tx(&bars->v_full[vs], kTileBytes);
          uint8_t* vd = smem + kVOff + vs * kTileBytes;
          tma_load_3d(&p.tm_v, &bars->v_full[vs], vd, 0, krow, hk);
          tma_load_3d(&p.tm_v, &bars->v_full[vs], vd + kTileBytes / 2, 64, krow, hk);
          if (++vs == 2) { vs = 0; vph ^= 1; }
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    uint32_t q_it = 0, ks = 0, kph = 0, vs = 0, vph = 0;
    uint32_t pph[2] = {0, 0}, fph[2] = {0, 0};
    for (int ui = sched_begin(p.sched, blockIdx.x); ui < sched_end(p.sched, blockIdx.x); ++ui) {
      const int u = sched_unit(p.sched, gridDim.x, ui);
      const FwdUnit un = p.units[u];
      const int n = un.n_kv, nh = un.nh;
      dbg_mark(1, 0x100);
      mbar_wait(&bars->q_full, q_it & 1);
      ++q_it;
      dbg_mark(1, 0x200);
      mbar_wait(&bars->k_full[ks], kph);
      tc_fence_after();
      for (int h = 0; h < nh; ++h) {
        issue_qk(tmem + h * 128, sbase + kQOff + h * kTileBytes, sbase + kKOff + ks * kTileBytes);
        mma_commit(&bars->s_full[h]);
      }
      mma_commit(&bars->k_empty[ks]);
      if (++ks == 2) { ks = 0; kph ^= 1; }
      if (n == 1) mma_commit(&bars->q_empty);
      for (int j = 0; j < n; ++j) {
        dbg_mark(1, 0x300 + j);
        mbar_wait(&bars->v_full[vs], vph);
        tc_fence_after();
        for (int h = 0; h < nh; ++h) {
          dbg_mark(1, 0x400 + j * 16 + h);
          mbar_wait(&bars->p_half[h], pph[h]);
          if (j == 0) {
            mbar_wait(&bars->o_free[h], fph[h] ^ 1);
            fph[h] ^= 1;
          }
          tc_fence_after();
          issue_pv_half(tmem + 256 + h * 128, tmem + h * 128, sbase + kVOff + vs * kTileBytes, 0, j > 0);
          mbar_wait(&bars->p_full[h], pph[h]);
          pph[h] ^= 1;
          tc_fence_after();
          issue_pv_half(tmem + 256 + h * 128, tmem + h * 128 + 32, sbase + kVOff + vs * kTileBytes, 1, true);
          if (j == n - 1) {
            mma_commit(&bars->o_full[h]);
          } else {
            if (h == 0) {
              dbg_mark(1, 0x600 + j);
              mbar_wait(&bars->k_full[ks], kph);
              tc_fence_after();
            }
            issue_qk(tmem + h * 128, sbase + kQOff + h * kTileBytes, sbase + kKOff + ks * kTileBytes);
            mma_commit(&bars->s_full[h]);
          }
        }
        mma_commit(&bars->v_empty[vs]);
        if (++vs == 2) { vs = 0; vph ^= 1; }
        if (j < n - 1) {
          mma_commit(&bars->k_empty[ks]);
          if (++ks == 2) { ks = 0; kph ^= 1; }
          if (j + 1 == n - 1) mma_commit(&bars->q_empty);
        }
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ------------------------------------------------------------ softmax
    const int h = warp >> 2;                 // which head slot
    const uint32_t row = (warp & 3) * 32 + lane;
    const uint32_t lane_sel = ((warp & 3) * 32) << 16;
    const uint32_t s_tmem = tmem + lane_sel + h * 128;
    const uint32_t o_tmem = tmem + lane_sel + 256 + h * 128;
    uint32_t sph = 0, oph = 0;
    for (int ui = sched_begin(p.sched, blockIdx.x); ui < sched_end(p.sched, blockIdx.x); ++ui) {
      const int u = sched_unit(p.sched, gridDim.x, ui);
      const FwdUnit un = p.units[u];
      if (h >= un.nh) continue;
      const DevTask tk = p.tasks[un.task];
      const int shift = tk.kv_len - tk.n_q;
      const int qi = un.tile * kTile + row;          // query index within the task
      const int pos = shift + qi;                    // its absolute key position
      const int first_masked_tile = (shift + un.tile * kTile) >> 7;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < un.n_kv; ++j) {
        if (row == 0) dbg_mark(2 + h, 0x100 + j);
        mbar_wait_warp(&bars->s_full[h], sph);
        sph ^= 1;
        tc_fence_after();
        softmax_tile<kFwdEmuMask>(s_tmem, o_tmem, j == 0, j >= first_masked_tile, pos - j * kTile, p.scale_log2, m, l,
                     [&](int half) { mbar_arrive(half ? &bars->p_full[h] : &bars->p_half[h]); });
        if (row == 0) dbg_mark(2 + h, 0x200 + j);
      }
      // ---- epilogue: O / l, LSE
      mbar_wait_warp(&bars->o_full[h], oph);
      oph ^= 1;
      tc_fence_after();
      const bool valid = qi < tk.n_q;
      const float inv = 1.f / l;
      const int head = un.head0 + h;
      __nv_bfloat16* orow = p.o + ((int64_t)(tk.q_off + qi) * p.h_q + head) * kHeadDim;
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
      if (valid) p.lse[(int64_t)head * p.q_rows + tk.q_off + qi] = (m + __log2f(l)) * 0.69314718055994531f;
      tc_fence_before();
      mbar_arrive(&bars->o_free[h]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_free<512>(tmem);
}

}  // namespace fwd

void preload_fwd() {
  set_max_smem(reinterpret_cast<const void*>(fwd::ca_fwd_kernel), fwd::kSmemBytes, "cudaFuncSetAttribute(fwd)");
}

}  // namespace cad_dev

extern "C" int cad_ca_fwd(const cad_ca_plan* plan, const void* q, const void* k, const void* v,
                          void* o, float* lse, void* stream) {
  using namespace cad_dev;
  return cad::guarded([&] {
    if (!plan || !q || !k || !v || !o || !lse) throw cad::DomainError("null argument");
    if (plan->fwd_units.empty()) return;
    DeviceGuard dg(plan->device);
    static const bool pair_off = std::getenv("CAD_FWD_PAIR") && std::getenv("CAD_FWD_PAIR")[0] == '0';
    if (!pair_off && launch_fwd_pair(plan, q, k, v, o, lse, static_cast<cudaStream_t>(stream))) return;
    fwd::Params p;
    make_tile_map(&p.tm_q, q, plan->shape.q_rows, plan->shape.h_q);
    make_tile_map(&p.tm_k, k, plan->shape.kv_rows, plan->shape.h_kv);
    make_tile_map(&p.tm_v, v, plan->shape.kv_rows, plan->shape.h_kv);
    p.tasks = plan->d_tasks;
    p.units = plan->d_fwd;
    p.n_units = static_cast<int>(plan->fwd_units.size());
    p.sched = plan->sched_fwd.d;
    p.h_q = plan->shape.h_q;
    p.group = plan->shape.h_q / plan->shape.h_kv;
    p.o = static_cast<__nv_bfloat16*>(o);
    p.lse = lse;
    p.q_rows = plan->shape.q_rows;
    p.scale_log2 = plan->shape.softmax_scale * 1.4426950408889634f;
    set_max_smem(reinterpret_cast<const void*>(fwd::ca_fwd_kernel), fwd::kSmemBytes, "cudaFuncSetAttribute(fwd)");
    const int grid = plan->sched_fwd.G;
    fwd::ca_fwd_kernel<<<grid, fwd::kThreads, fwd::kSmemBytes, static_cast<cudaStream_t>(stream)>>>(p);
    cuda_check(cudaGetLastError(), "ca_fwd launch");
  });
}
