// Fused dK/dV/dQ on CTA pairs (cta_group::2), EXPERIMENTAL (CAD_BWD_FUSED=1;
// measured slower than the two-pass backward, profiles/r2_fused_bwd.md): the
// pair dK/dV kernel of ca_dkdv2.cu plus dQ = dS K accumulated in the same
// pass, so the backward does not recompute S and dP in a separate dQ kernel
// (5 tile GEMMs per (kv tile pair, q tile, head) instead of 7).
//
//   dQ(i) [q 128 x d 128] = dS(i) [q x 256 kv of the pair] K [256 kv x d]
// is one M=128 cta_group::2 MMA per iteration whose reduction runs over both
// CTAs' kv rows, so the pair adds ONE fp32 partial per (q tile, head) into
// the accumulator instead of two:
//   A: CTA r holds q rows [64r, 64r+64) of dS for all 256 kv rows (MN-major
//      SW128, 32 KB, double-buffered by iteration parity). The element-wise
//      threads of BOTH CTAs write it: a thread's q chunk ch (its kv row, q
//      columns [64ch + 32w, +32)) goes to CTA ch's buffer -- locally, or by
//      st.async with complete_tx on the peer's xchg_full barrier, which a
//      relay warp turns into an arrival on the MMA issuer's xchg_ready.
//   B: CTA r holds d columns [64r, 64r+64) of both kv tiles' K rows (a second,
//      MN-major view of K: one 16 KB plane per tile).
//   D: CTA r's TMEM lanes [0,64) = q 64r+lane, d [0,64); lanes [64,128) =
//      q 64r+lane-64, d [64,128) (measured: scripts/micro/umma_m128_pair.cu),
//      64 columns: the half of dP^T's columns the packed dS^T leaves free
//      (dS^T is packed into columns [64,128), P^T stays where ca_dkdv2 has it).
// Four reduce warps read the partial out (which frees the columns for
// dP^T(i+1)), stage it in that iteration's dS buffer (idle once dQ(i) has
// completed) and add it into an fp32 [rows][h_q][128] accumulator with TMA
// reduce-adds (cp.reduce.async.bulk.tensor .add.f32; ~6 TB/s of L2
// reductions measured, scripts/micro/l2_reduce.cu). Rows past a task's
// queries receive +0 (their dS is masked) and rows past the buffer are
// clipped by TMA. The host zeroes the accumulator before the launch and a
// conversion kernel writes scale * accumulator as bf16 dQ after it. fp32
// addition order varies from run to run: the two-pass backward (ca_dkdv2 +
// ca_dq2) is the default and deterministic.
//
// Shared memory per CTA: K, V (32 KB each), one Q and one dO tile (32 KB
// each, as two independently released halves: K-major rows [64r, 64r+64)
// for S^T / dP^T, MN-major columns [64r, 64r+64) for dK / dV; the producer
// runs one iteration ahead), the dQ view of K (32 KB), two dS / staging
// buffers (64 KB): 226 KB. dK/dV leave by direct global stores.
//
// Warps: 0-7 element-wise (thread = kv row), 8 TMA producer, 9 MMA issuer
// (even CTA), 10 dS relay, 11 idle, 12-15 dQ reduce (TMEM quadrant =
// warp % 4).
#define CAD_KERNEL_TAG "ca_dkdvq2"  // names this file in the mbarrier-timeout report
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
namespace kvq2 {

#ifndef CAD_KVQ2_EMU_MASK
#define CAD_KVQ2_EMU_MASK 0x1111
#endif
constexpr uint32_t kEmuMask = CAD_KVQ2_EMU_MASK;
// diagnostic builds only (wrong dQ): skip the TMA reduce-adds / the dS
// staging wait / the dQ MMA
#ifndef CAD_KVQ2_DIAG
#define CAD_KVQ2_DIAG 0
#endif
constexpr bool kNoReduce = CAD_KVQ2_DIAG & 1, kNoDstWait = CAD_KVQ2_DIAG & 2, kNoDqMma = CAD_KVQ2_DIAG & 4;
constexpr bool kNoDqFree = CAD_KVQ2_DIAG & 8, kNoXchg = CAD_KVQ2_DIAG & 16;
constexpr bool kNoExchange = CAD_KVQ2_DIAG & 32, kNoReadout = CAD_KVQ2_DIAG & 64;
#ifndef CAD_KVQ2_DQ_FIRST
#define CAD_KVQ2_DQ_FIRST 0
#endif

constexpr int kThreads = 512;
constexpr uint32_t kKOff = 0;
constexpr uint32_t kVOff = kTileBytes;
// Q and dO: one stage each, in two independently released halves:
// [K-major: q rows 64r..64r+63, two 8 KB d-planes (S^T / dP^T) | MN-major:
// all 128 q rows, d columns 64r..64r+63 (dK / dV)]. Each half is reloaded as
// soon as its own MMA has read it, so a single stage hides the load latency.
constexpr uint32_t kQOff = 2 * kTileBytes;
constexpr uint32_t kDOOff = 3 * kTileBytes;
constexpr uint32_t kKqOff = 4 * kTileBytes;  // dQ's B: [tile 2t | tile 2t+1] rows, d plane r
constexpr uint32_t kDsOff = 5 * kTileBytes;  // dQ's A x 2 (iteration parity): dS, q half r x 256 kv; staging
constexpr uint32_t kLseOff = 7 * kTileBytes;
constexpr uint32_t kDOff = kLseOff + 2 * 512;
constexpr uint32_t kBarOff = kDOff + 2 * 512;
constexpr uint32_t kSmemBytes = kBarOff + 256;
static_assert(kSmemBytes <= 232448, "fused dK/dV/dQ pair shared memory");

struct Bars {
  uint64_t kv_full, kv_empty, kq_full, kq_empty;
  uint64_t qk_full, qk_empty, qm_full, qm_empty, dok_full, dok_empty, dom_full, dom_empty;
  uint64_t lse_full[2], d_full[2];
  uint64_t s_full, dp_full, p_half, p_full, ds_half, ds_full, acc_full, acc_free;
  uint64_t dq_full, dq_free, dst_free[2], xchg_full, xchg_ready;
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "fused pair barriers");

struct Params {
  CUtensorMap tm_q, tm_q64, tm_k, tm_v, tm_do, tm_do64, tm_dqa;
  const float* nlse2;
  const float* ndelta;
  int64_t pitch;
  const DevTask* tasks;
  const KvUnit* units;  // tile = the pair's first kv tile
  const KvSeg* segs;
  int n_units;
  const int32_t* sched;
  int group;
  int h_kv;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  float scale;
  float scale_log2;
};

struct Cursor {
  int g, seg, qt;
  __device__ void start(const KvUnit& u, const KvSeg* segs) {
    g = 0;
    seg = u.seg_begin;
    qt = segs[seg].qt_hi - 1;
  }
  __device__ void next(const KvUnit& u, const KvSeg* segs, int group) {
    if (++g < group) return;
    g = 0;
    if (--qt >= segs[seg].qt_lo) return;
    if (++seg < u.seg_end) qt = segs[seg].qt_hi - 1;
  }
};

// The pair's iterations as one stream across its units (the producer runs
// one iteration ahead for the K-major halves).
struct Stream {
  int ui, end, i;
  KvUnit un;
  Cursor c;
  bool valid;
  __device__ void load(const Params& p, int n_pairs) {
    valid = ui < end;
    if (!valid) return;
    un = p.units[sched_unit(p.sched, n_pairs, ui)];
    c.start(un, p.segs);
    i = 0;
  }
  __device__ void start(const Params& p, int pair, int n_pairs) {
    ui = sched_begin(p.sched, pair);
    end = sched_end(p.sched, pair);
    load(p, n_pairs);
  }
  __device__ void next(const Params& p, int n_pairs) {
    if (++i < un.n_iter) {
      c.next(un, p.segs, p.group);
    } else {
      ++ui;
      load(p, n_pairs);
    }
  }
};

// ------------------------------------------------------------ cluster helpers
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void tma_reduce_add_3d(const void* desc, const void* src, int c0, int c1, int c2) {
  asm volatile(
      "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(desc)),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// ------------------------------------------------------------ MMA issue
// D (M=256 kv rows) = A B^T: A = this CTA's 128 K or V rows (K-major, 16 KB
// d-planes), B = its 64 Q or dO rows (K-major, 8 KB d-planes); N = 128 q.
__device__ __forceinline__ void issue_kq_pair(uint32_t d_tmem, uint32_t a_smem, uint32_t b_smem) {
  constexpr uint32_t idesc = idesc_bf16(256, 128, false, false);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t kin = (k & 3) * 32;
    umma_ss_2sm(d_tmem, sw128_desc(a_smem + (k >> 2) * (kTileBytes / 2) + kin, 16, 1024),
                sw128_desc(b_smem + (k >> 2) * (kTileBytes / 4) + kin, 16, 1024), idesc, k > 0 ? 1u : 0u);
  }
}
// dV += P^T dO, one K-half (q rows [64h, 64h+64)): A = packed P^T in TMEM
// (columns a + 8k), B = this CTA's 64 d columns of all q rows (MN-major).
__device__ __forceinline__ void issue_pv_pair_half(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_smem, int half,
                                                   bool accumulate) {
  constexpr uint32_t idesc = idesc_bf16(256, 128, false, true);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    umma_ts_2sm(d_tmem, a_tmem + k * 8, sw128_desc(b_smem + (half * 4 + k) * 2048, kTileBytes / 2, 1024), idesc,
                (accumulate || half > 0 || k > 0) ? 1u : 0u);
}
// dK += dS^T Q, one K-half: packed dS^T of warpgroup w, chunk h sits at
// dP^T columns 64 + 32w + 16h (k-steps 0-1: w = 0, 2-3: w = 1).
__device__ __forceinline__ void issue_dsq_pair_half(uint32_t d_tmem, uint32_t tdp, uint32_t b_smem, int half,
                                                    bool accumulate) {
  constexpr uint32_t idesc = idesc_bf16(256, 128, false, true);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    umma_ts_2sm(d_tmem, tdp + 64 + 32 * (k >> 1) + 16 * half + 8 * (k & 1),
                sw128_desc(b_smem + (half * 4 + k) * 2048, kTileBytes / 2, 1024), idesc,
                (accumulate || half > 0 || k > 0) ? 1u : 0u);
}
// dQ = dS K: M=128 (q), N=128 (d), K=256 (both CTAs' kv rows) in 16 steps;
// A and B MN-major, 2 KB per step of 16 kv rows.
__device__ __forceinline__ void issue_dq_pair(uint32_t d_tmem, uint32_t a_smem, uint32_t b_smem) {
  constexpr uint32_t idesc = idesc_bf16(128, 128, true, true);
  if (!elect_one()) return;
#pragma unroll
  for (int s = 0; s < 16; ++s)
    umma_ss_2sm(d_tmem, sw128_desc(a_smem + s * 2048, 16384, 1024), sw128_desc(b_smem + s * 2048, 16384, 1024),
                idesc, s > 0 ? 1u : 0u);
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  if (elect_one()) umma_commit_pair(bar);
  __syncwarp();
}

__global__ void __launch_bounds__(kThreads, 1) ca_bwd_dkdvq_pair_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars* bars = reinterpret_cast<Bars*>(smem + kBarOff);
  float* lse_rows = reinterpret_cast<float*>(smem + kLseOff);
  float* d_rows = reinterpret_cast<float*>(smem + kDOff);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (sbase & 1023) __trap();  // SW128 tiles need 1024-byte alignment
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&p.tm_q);
    tma_prefetch(&p.tm_q64);
    tma_prefetch(&p.tm_do64);
    tma_prefetch(&p.tm_k);
    tma_prefetch(&p.tm_v);
    tma_prefetch(&p.tm_do);
    tma_prefetch(&p.tm_dqa);
    mbar_init(&bars->kv_full, 2);
    mbar_init(&bars->kv_empty, 1);
    mbar_init(&bars->kq_full, 2);
    mbar_init(&bars->kq_empty, 1);
    for (uint64_t* f : {&bars->qk_full, &bars->qm_full, &bars->dok_full, &bars->dom_full}) mbar_init(f, 2);
    for (uint64_t* e : {&bars->qk_empty, &bars->qm_empty, &bars->dok_empty, &bars->dom_empty}) mbar_init(e, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->lse_full[i], 32);
      mbar_init(&bars->d_full[i], 32);
      mbar_init(&bars->dst_free[i], 8);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->p_half, 512);
    mbar_init(&bars->p_full, 512);
    mbar_init(&bars->ds_half, 512);
    mbar_init(&bars->ds_full, 512);
    mbar_init(&bars->acc_full, 1);
    mbar_init(&bars->acc_free, 512);
    mbar_init(&bars->dq_full, 1);
    mbar_init(&bars->dq_free, 8);
    mbar_init(&bars->xchg_full, 1);
    mbar_init(&bars->xchg_ready, 2);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc_2sm<512>(&bars->tmem_base);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const uint32_t tS = tmem, tDP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == 8) {
      // ---------------------------------------------------------- producer
      // Step `it` issues, in the order the MMAs of iteration it-1 free the
      // halves: dO MN-major(it) (+ -D rows), Q K-major(it+1) (+ -LSE rows;
      // the next unit's K/V first when it+1 starts one), Q MN-major(it)
      // (the unit's dQ view of K after it when it starts one), dO
      // K-major(it+1). Every half thus loads a full iteration before its MMA.
      // -LSE / -D rows alternate between two slots: slot j&1 was last read
      // by P(j-2) / dS(j-2), which precede S^T(j-1) / dV(j-1), whose
      // completion releases the halves waited for before writing them.
      uint32_t it = 0, kv_units = 0, kq_units = 0;
      uint8_t* q = smem + kQOff;
      uint8_t* d = smem + kDOOff;
      Stream A, B;
      A.start(p, pair, n_pairs);
      B = A;
      auto qrow_of = [&](const Stream& x) { return p.tasks[p.segs[x.c.seg].task].q_off + x.c.qt * kTile; };
      auto head_of = [&](const Stream& x) { return x.un.hk * p.group + x.c.g; };
      auto load_kv = [&](const Stream& x) {
        if (lane == 0) {
          const int krow = x.un.kv_off + (x.un.tile + int(rank)) * kTile;  // this CTA's kv tile
          mbar_wait(&bars->kv_empty, (kv_units & 1) ^ 1);
          if (leader) mbar_expect_tx(&bars->kv_full, 4 * kTileBytes);
          else mbar_arrive_leader(&bars->kv_full);
          tma_load_3d_2sm(&p.tm_k, &bars->kv_full, smem + kKOff, 0, krow, x.un.hk);
          tma_load_3d_2sm(&p.tm_k, &bars->kv_full, smem + kKOff + kTileBytes / 2, 64, krow, x.un.hk);
          tma_load_3d_2sm(&p.tm_v, &bars->kv_full, smem + kVOff, 0, krow, x.un.hk);
          tma_load_3d_2sm(&p.tm_v, &bars->kv_full, smem + kVOff + kTileBytes / 2, 64, krow, x.un.hk);
        }
        ++kv_units;
      };
      auto load_qk = [&](const Stream& x, uint32_t j) {  // Q K-major half + -LSE rows of iteration j
        const int qrow = qrow_of(x), head = head_of(x), qrow_r = qrow + 64 * int(rank);
        mbar_wait(&bars->qk_empty, (j & 1) ^ 1);
        if (lane == 0) {
          if (leader) mbar_expect_tx(&bars->qk_full, kTileBytes);
          else mbar_arrive_leader(&bars->qk_full);
          tma_load_3d_2sm(&p.tm_q64, &bars->qk_full, q, 0, qrow_r, head);
          tma_load_3d_2sm(&p.tm_q64, &bars->qk_full, q + kTileBytes / 4, 64, qrow_r, head);
        }
        const float* nl = p.nlse2 + int64_t(head) * p.pitch;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int col = lane + 32 * k;
          cp_async4(lse_rows + (j & 1) * 128 + col, nl + min(int64_t(qrow) + col, p.pitch - 1));
        }
        cp_async_arrive(&bars->lse_full[j & 1]);
      };
      auto load_dok = [&](const Stream& x, uint32_t j) {  // dO K-major half of iteration j
        const int qrow_r = qrow_of(x) + 64 * int(rank), head = head_of(x);
        mbar_wait(&bars->dok_empty, (j & 1) ^ 1);
        if (lane == 0) {
          if (leader) mbar_expect_tx(&bars->dok_full, kTileBytes);
          else mbar_arrive_leader(&bars->dok_full);
          tma_load_3d_2sm(&p.tm_do64, &bars->dok_full, d, 0, qrow_r, head);
          tma_load_3d_2sm(&p.tm_do64, &bars->dok_full, d + kTileBytes / 4, 64, qrow_r, head);
        }
      };
      if (A.valid) {
        load_kv(A);
        load_qk(A, 0);
        load_dok(A, 0);
      }
      for (; A.valid; ++it) {
        const int qrow = qrow_of(A), head = head_of(A);
        // dO MN-major(it), -D rows(it)
        mbar_wait(&bars->dom_empty, (it & 1) ^ 1);
        if (lane == 0) {
          if (leader) mbar_expect_tx(&bars->dom_full, kTileBytes);
          else mbar_arrive_leader(&bars->dom_full);
          tma_load_3d_2sm(&p.tm_do, &bars->dom_full, d + kTileBytes / 2, 64 * int(rank), qrow, head);
        }
        const float* nd = p.ndelta + int64_t(head) * p.pitch;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int col = lane + 32 * k;
          cp_async4(d_rows + (it & 1) * 128 + col, nd + min(int64_t(qrow) + col, p.pitch - 1));
        }
        cp_async_arrive(&bars->d_full[it & 1]);
        B.next(p, n_pairs);
        if (B.valid) {
          if (B.i == 0) load_kv(B);
          load_qk(B, it + 1);
        }
        // Q MN-major(it)
        mbar_wait(&bars->qm_empty, (it & 1) ^ 1);
        if (lane == 0) {
          if (leader) mbar_expect_tx(&bars->qm_full, kTileBytes);
          else mbar_arrive_leader(&bars->qm_full);
          tma_load_3d_2sm(&p.tm_q, &bars->qm_full, q + kTileBytes / 2, 64 * int(rank), qrow, head);
          if (A.i == 0) {
            // the unit's dQ view of K (d plane r of both tiles); the previous
            // unit's last dQ preceded dK(it-1), which qm_empty waited for
            const int krow0 = A.un.kv_off + A.un.tile * kTile;
            mbar_wait(&bars->kq_empty, (kq_units & 1) ^ 1);
            if (leader) mbar_expect_tx(&bars->kq_full, 2 * kTileBytes);
            else mbar_arrive_leader(&bars->kq_full);
            tma_load_3d_2sm(&p.tm_k, &bars->kq_full, smem + kKqOff, 64 * int(rank), krow0, A.un.hk);
            tma_load_3d_2sm(&p.tm_k, &bars->kq_full, smem + kKqOff + kTileBytes / 2, 64 * int(rank),
                            krow0 + kTile, A.un.hk);
          }
        }
        if (A.i == 0) ++kq_units;
        if (B.valid) load_dok(B, it + 1);
        A.next(p, n_pairs);
      }
    } else if (warp == 9 && leader) {
      // ---------------------------------------------------------- MMA (even CTA)
      uint32_t kv_it = 0, acc_it = 0, p_ph = 0, ds_ph = 0, nq = 0;
      uint32_t qk_ph = 0, qm_ph = 0, dok_ph = 0, dom_ph = 0;
      const uint32_t sK = sbase + kKOff, sV = sbase + kVOff, sQ = sbase + kQOff, sDO = sbase + kDOOff;
      const uint32_t sKq = sbase + kKqOff, sDs = sbase + kDsOff;
      for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
        const int u = sched_unit(p.sched, n_pairs, ui);
        const KvUnit un = p.units[u];
        const int n = un.n_iter;
        mbar_wait(&bars->kv_full, kv_it & 1);
        mbar_wait(&bars->qk_full, qk_ph);
        qk_ph ^= 1;
        tc_fence_after();
        issue_kq_pair(tS, sK, sQ);
        commit_pair(&bars->s_full);
        commit_pair(&bars->qk_empty);
        mbar_wait(&bars->dok_full, dok_ph);
        dok_ph ^= 1;
        if (nq > 0 && !kNoDqFree) mbar_wait(&bars->dq_free, (nq - 1) & 1);  // the last dQ partial left dP^T
        tc_fence_after();
        issue_kq_pair(tDP, sV, sDO);
        commit_pair(&bars->dp_full);
        commit_pair(&bars->dok_empty);
        if (n == 1) commit_pair(&bars->kv_empty);  // K / V read for the last time
        for (int i = 0; i < n; ++i) {
          // dV += P^T dO in two K-halves as the warpgroups release them
          mbar_wait(&bars->p_half, p_ph);
          if (i == 0) {
            mbar_wait(&bars->acc_free, (acc_it & 1) ^ 1);
            ++acc_it;
          }
          mbar_wait(&bars->dom_full, dom_ph);
          dom_ph ^= 1;
          tc_fence_after();
          issue_pv_pair_half(tDV, tS + 16, sDO + kTileBytes / 2, 0, i > 0);
          mbar_wait(&bars->p_full, p_ph);
          p_ph ^= 1;
          tc_fence_after();
          issue_pv_pair_half(tDV, tS + 80, sDO + kTileBytes / 2, 1, true);
          commit_pair(&bars->dom_empty);
          if (i + 1 < n) {
            mbar_wait(&bars->qk_full, qk_ph);
            qk_ph ^= 1;
            tc_fence_after();
            issue_kq_pair(tS, sK, sQ);  // S^T(i+1): runs after dV(i) read P^T (in order)
            commit_pair(&bars->s_full);
            commit_pair(&bars->qk_empty);
          }
          mbar_wait(&bars->ds_half, ds_ph);  // dK += dS^T Q, likewise in K-halves
          mbar_wait(&bars->qm_full, qm_ph);
          qm_ph ^= 1;
          tc_fence_after();
          issue_dsq_pair_half(tDK, tDP, sQ + kTileBytes / 2, 0, i > 0);
          mbar_wait(&bars->ds_full, ds_ph);  // also: the locally written dS halves
          ds_ph ^= 1;
          tc_fence_after();
#if CAD_KVQ2_DQ_FIRST
          // dQ(i) ahead of dK's second half: the partial's read-out overlaps
          // that half, but the dS exchange joins dK's critical path
          if (i == 0) mbar_wait(&bars->kq_full, kv_it & 1);
          mbar_wait(&bars->xchg_ready, nq & 1);  // the exchanged dS halves, both CTAs
          tc_fence_after();
          if (!kNoDqMma) issue_dq_pair(tDP, sDs + (nq & 1) * kTileBytes, sKq);
          commit_pair(&bars->dq_full);
          ++nq;
          if (i + 1 == n) commit_pair(&bars->kq_empty);
          issue_dsq_pair_half(tDK, tDP, sQ + kTileBytes / 2, 1, true);
          commit_pair(&bars->qm_empty);
#else
          issue_dsq_pair_half(tDK, tDP, sQ + kTileBytes / 2, 1, true);
          commit_pair(&bars->qm_empty);
          // dQ(i) into dP^T's columns [0, 64) once both CTAs hold dS(i)
          if (i == 0) mbar_wait(&bars->kq_full, kv_it & 1);
          if (!kNoExchange) mbar_wait(&bars->xchg_ready, nq & 1);
          tc_fence_after();
          if (!kNoDqMma) issue_dq_pair(tDP, sDs + (nq & 1) * kTileBytes, sKq);
          commit_pair(&bars->dq_full);
          ++nq;
          if (i + 1 == n) commit_pair(&bars->kq_empty);
#endif
          if (i + 1 < n) {
            mbar_wait(&bars->dok_full, dok_ph);
            dok_ph ^= 1;
            if (!kNoDqFree) mbar_wait(&bars->dq_free, (nq - 1) & 1);
            tc_fence_after();
            issue_kq_pair(tDP, sV, sDO);  // dP^T(i+1)
            commit_pair(&bars->dp_full);
            commit_pair(&bars->dok_empty);
            if (i + 2 == n) commit_pair(&bars->kv_empty);
          }
        }
        ++kv_it;
        commit_pair(&bars->acc_full);
      }
    } else if (warp == 10) {
      // ---------------------------------------------------------- dS relay
      // The peer's dS half lands here by st.async (complete_tx on xchg_full);
      // once all 16 KB are in, make them visible to the async proxy and tell
      // the MMA issuer (xchg_ready on the even CTA, one arrival per CTA).
      if (lane == 0 && !kNoExchange) {
        uint32_t it = 0;
        for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
          const int n = p.units[sched_unit(p.sched, n_pairs, ui)].n_iter;
          for (int i = 0; i < n; ++i, ++it) {
            if (!kNoXchg) {
              mbar_expect_tx(&bars->xchg_full, kTileBytes / 2);
              mbar_wait(&bars->xchg_full, it & 1);
            }
            fence_proxy_async_smem();
            mbar_arrive_leader(&bars->xchg_ready);
          }
        }
      }
      __syncwarp();
    } else if (warp >= 12) {
      // ---------------------------------------------------------- dQ reduce
      // Warp 12+qd reads TMEM lanes [32qd, 32qd+32) of the partial: q rows
      // 64r + 32(qd&1) + lane, d columns 64(qd>>1) + [0,64); stages them as
      // two SW128 32x32 fp32 boxes in its 8 KB of the iteration's dS buffer
      // (idle once dQ(i) has completed); TMA adds them into the accumulator.
      const uint32_t qd = warp & 3;
      const uint32_t tq = tDP + ((32 * qd) << 16);
      const uint32_t peer_dst_free = mapa(smem_u32(&bars->dst_free[0]), rank ^ 1);
      uint32_t it = 0;
      for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
        const int u = sched_unit(p.sched, n_pairs, ui);
        const KvUnit un = p.units[u];
        Cursor c;
        c.start(un, p.segs);
        for (int i = 0; i < un.n_iter; ++i, c.next(un, p.segs, p.group), ++it) {
          const DevTask tk = p.tasks[p.segs[c.seg].task];
          const int head = un.hk * p.group + c.g;
          const int row0 = tk.q_off + c.qt * kTile + 64 * int(rank) + 32 * int(qd & 1);
          uint8_t* stg = smem + kDsOff + (it & 1) * kTileBytes + qd * 8192;
          mbar_wait_warp(&bars->dq_full, it & 1);
          tc_fence_after();
#pragma unroll
          for (int b = 0; b < 2 && !kNoReadout; ++b) {
            uint32_t v[32];
            tmem_ld32(tq + 32 * b, v);
            tmem_wait_ld();
            if (b == 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive_leader(&bars->dq_free);  // dP^T(i+1) may overwrite
            }
            uint8_t* line = stg + b * 4096 + lane * 128;
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4)
              *reinterpret_cast<uint4*>(line + ((c4 ^ (lane & 7)) << 4)) =
                  make_uint4(v[4 * c4], v[4 * c4 + 1], v[4 * c4 + 2], v[4 * c4 + 3]);
          }
          if (kNoReadout) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_leader(&bars->dq_free);
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            const int d0 = 64 * int(qd >> 1);
            if (!kNoReduce) {
              tma_reduce_add_3d(&p.tm_dqa, stg, d0, row0, head);
              tma_reduce_add_3d(&p.tm_dqa, stg + 4096, d0 + 32, row0, head);
            }
            bulk_commit();
            bulk_wait_read0();  // staging read: the buffer may take dS(i+2)
            mbar_arrive(&bars->dst_free[it & 1]);
            asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(peer_dst_free + 8 * (it & 1))
                         : "memory");
          }
          __syncwarp();
        }
      }
      if (lane == 0) bulk_wait0();
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    // ------------------------------------------------------------ elementwise
    const int w = warp >> 2;                    // q column chunks, see below
    const uint32_t r = (warp & 3) * 32 + lane;  // kv row within the tile
    const uint32_t lsel = ((warp & 3) * 32) << 16;
    const int c0 = 64 * w;
    const uint32_t tSw = tS + lsel, tDPw = tDP + lsel;
    // this thread's row of the dQ A operand (kv row 128 rank + r) in CTA ch's
    // dS buffer; 16-byte chunks 4w..4w+3 (its 32 q values), SW128 swizzled
    const uint32_t ds_row = (128 * rank + r) * 128;
    const uint32_t ds_local = sbase + kDsOff + ds_row;
    const uint32_t ds_remote = mapa(ds_local, rank ^ 1);
    const uint32_t xchg_remote = mapa(smem_u32(&bars->xchg_full), rank ^ 1);
    uint32_t s_ph = 0, dp_ph = 0, acc_ph = 0, it = 0;
    for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
      const int u = sched_unit(p.sched, n_pairs, ui);
      const KvUnit un = p.units[u];
      const int kj = (un.tile + int(rank)) * kTile + r;  // key index relative to kv_off
      Cursor c;
      c.start(un, p.segs);
      for (int i = 0; i < un.n_iter; ++i, c.next(un, p.segs, p.group), ++it) {
        const DevTask tk = p.tasks[p.segs[c.seg].task];
        const int shift = tk.kv_len - tk.n_q;
        mbar_wait_warp(&bars->lse_full[it & 1], (it >> 1) & 1);  // the tile's -LSE rows (own copy)
        const uint32_t s_nlse = smem_u32(lse_rows + (it & 1) * 128), s_nd = smem_u32(d_rows + (it & 1) * 128);
        mbar_wait_warp(&bars->s_full, s_ph);
        s_ph ^= 1;
        tc_fence_after();
        // Warpgroup w owns q columns [32w, 32w+32) (chunk 0) and
        // [64+32w, 64+32w+32) (chunk 1): both warpgroups finish chunk 0 first,
        // which completes q columns [0,64) = the first K-half of dV/dK.
        float x[64];
        {
          uint32_t r0[32], r1[32];
          tmem_ld32(tSw + 32 * w, r0);
          tmem_ld32(tSw + 64 + 32 * w, r1);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            x[k] = __uint_as_float(r0[k]);
            x[32 + k] = __uint_as_float(r1[k]);
          }
        }
        const uint64_t sc2 = f2(p.scale_log2, p.scale_log2);
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          const int qb = c.qt * kTile + 64 * ch + 32 * w;
          const int lo = kj - shift - qb;
          const int hi = tk.n_q - qb;
          const bool full = ((un.tile + int(rank)) * kTile + kTile - 1 - shift - qb) <= 0 && hi >= 32;
          float* xc = x + 32 * ch;
          const uint32_t s_l = s_nlse + 4 * (64 * ch + 32 * w);
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            const float4 nl = lds4(s_l + 4 * k);
            float a0, a1, a2, a3;
            f2_split(ffma2(f2(xc[k], xc[k + 1]), sc2, f2(nl.x, nl.y)), a0, a1);
            f2_split(ffma2(f2(xc[k + 2], xc[k + 3]), sc2, f2(nl.z, nl.w)), a2, a3);
            if ((kEmuMask >> (k / 4)) & 1) {
              exp2_fma2(a0, a1);
              exp2_fma2(a2, a3);
              xc[k] = a0;
              xc[k + 1] = a1;
              xc[k + 2] = a2;
              xc[k + 3] = a3;
            } else {
              xc[k] = ex2(a0);
              xc[k + 1] = ex2(a1);
              xc[k + 2] = ex2(a2);
              xc[k + 3] = ex2(a3);
            }
          }
          if (!full) {
#pragma unroll
            for (int k = 0; k < 32; ++k) xc[k] = (k >= lo && k < hi) ? xc[k] : 0.f;
          }
          uint32_t pk[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) pk[k] = pack_bf16(xc[2 * k], xc[2 * k + 1]);
          // P^T (bf16) inside this warpgroup's own S^T columns: K-half ch
          // is the 32 packed columns at 16 + 64 ch (WG0 first, then WG1)
          tmem_st16(tSw + 16 + 64 * ch + 16 * w, pk);
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive_leader(ch ? &bars->p_full : &bars->p_half);
        }
        mbar_wait_warp(&bars->dp_full, dp_ph);
        dp_ph ^= 1;
        mbar_wait_warp(&bars->d_full[it & 1], (it >> 1) & 1);  // the tile's -D rows
        tc_fence_after();
        float y[64];
        {
          uint32_t r0[32], r1[32];
          tmem_ld32(tDPw + 32 * w, r0);
          tmem_ld32(tDPw + 64 + 32 * w, r1);
          tmem_wait_ld();
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            y[k] = __uint_as_float(r0[k]);
            y[32 + k] = __uint_as_float(r1[k]);
          }
        }
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          const int qb = c.qt * kTile + 64 * ch + 32 * w;
          const int lo = kj - shift - qb;
          const int hi = tk.n_q - qb;
          const bool full = ((un.tile + int(rank)) * kTile + kTile - 1 - shift - qb) <= 0 && hi >= 32;
          const float* xc = x + 32 * ch;
          float* yc = y + 32 * ch;
          const uint32_t s_d = s_nd + 4 * (64 * ch + 32 * w);
#pragma unroll
          for (int k = 0; k < 32; k += 4) {
            const float4 nd = lds4(s_d + 4 * k);
            f2_split(fmul2(f2(xc[k], xc[k + 1]), fadd2(f2(yc[k], yc[k + 1]), f2(nd.x, nd.y))), yc[k],
                     yc[k + 1]);
            f2_split(fmul2(f2(xc[k + 2], xc[k + 3]), fadd2(f2(yc[k + 2], yc[k + 3]), f2(nd.z, nd.w))),
                     yc[k + 2], yc[k + 3]);
          }
          if (!full) {
#pragma unroll
            for (int k = 0; k < 32; ++k) yc[k] = (k >= lo && k < hi) ? yc[k] : 0.f;
          }
          uint32_t pk[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) pk[k] = pack_bf16(yc[2 * k], yc[2 * k + 1]);
          // dS^T (bf16) packed into dP^T columns [64, 128): WG w at 64 + 32w,
          // chunk ch at +16ch -- columns this warpgroup has already read
          tmem_st16(tDPw + 64 + 32 * w + 16 * ch, pk);
          // dS into the dQ A operand of CTA ch (q half ch), once the previous
          // iteration's partial has left both CTAs' staging
          if (ch == 0 && !kNoDstWait) mbar_wait_warp(&bars->dst_free[it & 1], ((it >> 1) & 1) ^ 1);
          const uint32_t dsb = (it & 1) * kTileBytes;
          if (kNoXchg || kNoExchange) {
          } else if (uint32_t(ch) == rank) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(ds_local + dsb + (((4 * w + j) ^ (r & 7)) << 4)),
                           "r"(pk[4 * j]), "r"(pk[4 * j + 1]), "r"(pk[4 * j + 2]), "r"(pk[4 * j + 3])
                           : "memory");
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              asm volatile(
                  "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
                      ds_remote + dsb + (((4 * w + j) ^ (r & 7)) << 4)),
                  "r"(pk[4 * j]), "r"(pk[4 * j + 1]), "r"(pk[4 * j + 2]), "r"(pk[4 * j + 3]), "r"(xchg_remote)
                  : "memory");
          }
          tmem_wait_st();
          tc_fence_before();
          if (ch) {
            fence_proxy_async_smem();  // the local dS half -> the tensor core
            mbar_arrive_leader(&bars->ds_full);
          } else {
            mbar_arrive_leader(&bars->ds_half);
          }
        }
      }
      // ---- epilogue: warpgroup w stores d columns [c0, c0+64) of dV and dK
      mbar_wait_warp(&bars->acc_full, acc_ph);
      acc_ph ^= 1;
      tc_fence_after();
      const int row = un.kv_off + kj;
      const bool valid = row < un.kv_end;
      const int64_t off = (int64_t(row) * p.h_kv + un.hk) * kHeadDim + c0;
      tmem_row_to_global(tDV + lsel + c0, 1.f, p.dv + off, valid);
      tmem_row_to_global(tDK + lsel + c0, p.scale, p.dk + off, valid);
      tc_fence_before();
      mbar_arrive_leader(&bars->acc_free);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 9) tmem_free_2sm<512>(tmem);
}

// dQ = scale * accumulator (fp32 -> bf16) over the task rows (the delta
// kernel's row chunks: <= 32 contiguous rows, all heads). HBM-bound.
__global__ void __launch_bounds__(256) dq_convert_kernel(const int2* chunks, const float* acc, __nv_bfloat16* dq,
                                                         int h_q, float scale) {
  const int2 ch = chunks[blockIdx.x];
  const int64_t base = int64_t(ch.x) * h_q * kHeadDim;
  const int64_t n4 = int64_t(ch.y) * h_q * kHeadDim / 4;
  const float4* a4 = reinterpret_cast<const float4*>(acc + base);
  uint2* d2 = reinterpret_cast<uint2*>(dq + base);
  for (int64_t i = threadIdx.x; i < n4; i += 256) {
    const float4 v = __ldcs(a4 + i);
    d2[i] = make_uint2(pack_bf16(v.x * scale, v.y * scale), pack_bf16(v.z * scale, v.w * scale));
  }
}

}  // namespace kvq2

void preload_dkdvq2() {
  set_max_smem(reinterpret_cast<const void*>(kvq2::ca_bwd_dkdvq_pair_kernel), kvq2::kSmemBytes,
               "cudaFuncSetAttribute(dkdvq2)");
  cudaFuncAttributes a;
  cuda_check(cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(kvq2::dq_convert_kernel)), "load dq_convert");
}

bool fused_bwd_enabled() {
  static const bool on = std::getenv("CAD_BWD_FUSED") && std::getenv("CAD_BWD_FUSED")[0] == '1';
  return on;
}

size_t dq_acc_bytes(const cad_ca_shape& sh) {
  return (size_t(sh.q_rows) * sh.h_q * kHeadDim * 4 + 255) / 256 * 256;
}

// Fused pair dK/dV/dQ: zero the accumulator, run the kernel (dK, dV stored,
// dQ partials added into acc). false if the plan has no pair units.
bool launch_dkdvq_pair(const cad_ca_plan* plan, const void* q, const void* k, const void* v, const void* dout,
                       const float* nlse2, const float* ndelta, int64_t pitch, void* dk, void* dv, float* acc,
                       cudaStream_t stream) {
  if (plan->kv2_units.empty()) return false;
  const cad_ca_shape& sh = plan->shape;
  kvq2::Params p;
  make_tile_map(&p.tm_q, q, sh.q_rows, sh.h_q);
  make_tile_map(&p.tm_q64, q, sh.q_rows, sh.h_q, 64);
  make_tile_map(&p.tm_do, dout, sh.q_rows, sh.h_q);
  make_tile_map(&p.tm_do64, dout, sh.q_rows, sh.h_q, 64);
  make_tile_map(&p.tm_k, k, sh.kv_rows, sh.h_kv);
  make_tile_map(&p.tm_v, v, sh.kv_rows, sh.h_kv);
  make_acc_map(&p.tm_dqa, acc, sh.q_rows, sh.h_q);
  p.nlse2 = nlse2;
  p.ndelta = ndelta;
  p.pitch = pitch;
  p.tasks = plan->d_tasks;
  p.units = plan->d_kv2;
  p.segs = plan->d_segs;
  p.n_units = static_cast<int>(plan->kv2_units.size());
  p.sched = plan->sched_kv2.d;
  p.group = sh.h_q / sh.h_kv;
  p.h_kv = sh.h_kv;
  p.dk = static_cast<__nv_bfloat16*>(dk);
  p.dv = static_cast<__nv_bfloat16*>(dv);
  p.scale = sh.softmax_scale;
  p.scale_log2 = sh.softmax_scale * 1.4426950408889634f;
  cuda_check(cudaMemsetAsync(acc, 0, size_t(sh.q_rows) * sh.h_q * kHeadDim * 4, stream), "memset(dq acc)");
  set_max_smem(reinterpret_cast<const void*>(kvq2::ca_bwd_dkdvq_pair_kernel), kvq2::kSmemBytes,
               "cudaFuncSetAttribute(dkdvq2)");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * plan->sched_kv2.G);
  cfg.blockDim = dim3(kvq2::kThreads);
  cfg.dynamicSmemBytes = kvq2::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kvq2::ca_bwd_dkdvq_pair_kernel, p), "ca_bwd_dkdvq_pair launch");
  return true;
}

void launch_dq_convert(const cad_ca_plan* plan, const float* acc, void* dq, cudaStream_t stream) {
  if (plan->row_chunks.empty()) return;
  kvq2::dq_convert_kernel<<<static_cast<unsigned>(plan->row_chunks.size()), 256, 0, stream>>>(
      plan->d_row_chunks, acc, static_cast<__nv_bfloat16*>(dq), plan->shape.h_q, plan->shape.softmax_scale);
  cuda_check(cudaGetLastError(), "dq_convert launch");
}

}  // namespace cad_dev
