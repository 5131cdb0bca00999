// dK/dV on CTA pairs (cta_group::2): a pair runs two consecutive kv tiles
// of one KV group and KV head (CTA r: tile 2t + r) over the q tiles that see
// the first of them (a superset of the second's: the second CTA's extra
// iterations are fully masked). Every MMA is M=256 (kv rows of both tiles)
// issued by the even CTA; each CTA stages half of every B operand:
//   S^T = K Q^T, dP^T = V dO^T: B = Q / dO rows [64r, 64r+64) (K-major),
//   dV += P^T dO, dK += dS^T Q: B = dO / Q columns [64r, 64r+64) of all 128
//   q rows (MN-major),
// so the shared-memory operand traffic per MMA drops by a quarter (the pool's
// B200s are power-capped; the CTA-pair forward and dQ ran 7-9 % faster than
// their single-CTA versions). Element-wise work, TMEM layout and MMA order
// are ca_bwd_dkdv_kernel's (ca_bwd.cu); arrivals go to the even CTA's
// barriers, and each CTA copies the -LSE/-D rows for its own warpgroups.
#define CAD_KERNEL_TAG "ca_dkdv2"  // names this file in the mbarrier-timeout report
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
namespace kv2 {

#ifndef CAD_DKDV_EMU_MASK
#define CAD_DKDV_EMU_MASK 0x1111
#endif
constexpr uint32_t kDkdvEmuMask = CAD_DKDV_EMU_MASK;
constexpr int kThreads = 384;
#ifndef CAD_KV2_QSTAGES
#define CAD_KV2_QSTAGES 2  // 2 measured 1.5 % faster than 3 at config 2 (A/B) and frees the staging below
#endif
#ifndef CAD_KV2_TMA_STORE
#define CAD_KV2_TMA_STORE 1
#endif
#ifndef CAD_KV2_DOSTAGES
#define CAD_KV2_DOSTAGES 2
#endif
constexpr int kQStages = CAD_KV2_QSTAGES, kDOStages = CAD_KV2_DOSTAGES;
static_assert(kQStages >= 2, "the Q ring needs two stages (S^T(i+1) loads while dK(i) reads Q(i))");
constexpr uint32_t kKOff = 0;
constexpr uint32_t kVOff = kTileBytes;
// Q / dO stage (32 KB): [K-major: q rows 64r..64r+63, two 8 KB d-planes |
// MN-major: all 128 q rows, d columns 64r..64r+63 (16 KB)]
constexpr uint32_t kQOff = 2 * kTileBytes;
constexpr uint32_t kDOOff = kQOff + kQStages * kTileBytes;
constexpr uint32_t kLseOff = kDOOff + kDOStages * kTileBytes;
constexpr uint32_t kDOff = kLseOff + kQStages * 512;
// dV/dK staging: one 16 KB SW128 plane per element-wise warpgroup (its 64 d
// columns), used for dV then dK; full tiles leave by TMA stores
constexpr uint32_t kStOff = (kDOff + kDOStages * 512 + 1023) / 1024 * 1024;
constexpr uint32_t kBarOff = CAD_KV2_TMA_STORE ? kStOff + kTileBytes : kDOff + kDOStages * 512;
constexpr uint32_t kSmemBytes = kBarOff + 256;
static_assert(kSmemBytes <= 232448, "dK/dV pair shared memory");

struct Bars {
  uint64_t kv_full, kv_empty;
  uint64_t q_full[kQStages], q_empty[kQStages], lse_full[kQStages];
  uint64_t do_full[kDOStages], do_empty[kDOStages], d_full[kDOStages];
  uint64_t s_full, dp_full, p_half, p_full, ds_half, ds_full, acc_full, acc_free;
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "dK/dV pair barriers");

template <int N>
struct KRing {
  uint32_t i = 0, ph = 0;
  __device__ void next() {
    if (++i == N) { i = 0; ph ^= 1; }
  }
};

struct Params {
  CUtensorMap tm_q, tm_q64, tm_k, tm_v, tm_do, tm_do64, tm_dk, tm_dv;
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
// One K-half (q rows [64h, 64h+64)) of D (M=256, N=128 d) += A (TMEM, packed
// bf16) B, B = this CTA's 64 d columns of all q rows (MN-major, 16 KB).
__device__ __forceinline__ void issue_acc_pair_half(uint32_t d_tmem, uint32_t a_tmem, uint32_t b_smem, int half,
                                                    bool accumulate) {
  constexpr uint32_t idesc = idesc_bf16(256, 128, false, true);
  if (!elect_one()) return;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    umma_ts_2sm(d_tmem, a_tmem + k * 8, sw128_desc(b_smem + (half * 4 + k) * 2048, kTileBytes / 2, 1024), idesc,
                (accumulate || half > 0 || k > 0) ? 1u : 0u);
}
__device__ __forceinline__ void commit_pair(uint64_t* bar) {
  if (elect_one()) umma_commit_pair(bar);
  __syncwarp();
}

__global__ void __launch_bounds__(kThreads, 1) ca_bwd_dkdv_pair_kernel(const __grid_constant__ Params p) {
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
    mbar_init(&bars->kv_full, 2);
    mbar_init(&bars->kv_empty, 1);
    for (int i = 0; i < kQStages; ++i) {
      mbar_init(&bars->q_full[i], 2);
      mbar_init(&bars->lse_full[i], 32);
      mbar_init(&bars->q_empty[i], 1);
    }
    for (int i = 0; i < kDOStages; ++i) {
      mbar_init(&bars->do_full[i], 2);
      mbar_init(&bars->d_full[i], 32);
      mbar_init(&bars->do_empty[i], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->p_half, 512);
    mbar_init(&bars->p_full, 512);
    mbar_init(&bars->ds_half, 512);
    mbar_init(&bars->ds_full, 512);
    mbar_init(&bars->acc_full, 1);
    mbar_init(&bars->acc_free, 512);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc_2sm<512>(&bars->tmem_base);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const uint32_t tS = tmem, tDP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (warp == 8) {
      // ---------------------------------------------------------- producer
      // Lane 0 issues this CTA's halves of the tile loads (2-SM TMA: the
      // bytes complete on the even CTA's q_full / do_full / kv_full); the
      // whole warp copies the tile's 128 -LSE and 128 -D values into this
      // CTA's own rows (cp.async; each lane's arrive lands on the local
      // lse_full / d_full, count 32).
      uint32_t kv_it = 0;
      KRing<kQStages> qr;
      KRing<kDOStages> dr;
      for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
        const int u = sched_unit(p.sched, n_pairs, ui);
        const KvUnit un = p.units[u];
        const int krow = un.kv_off + (un.tile + int(rank)) * kTile;  // this CTA's kv tile
        if (lane == 0) {
          mbar_wait(&bars->kv_empty, (kv_it & 1) ^ 1);
          if (leader) mbar_expect_tx(&bars->kv_full, 4 * kTileBytes);
          else mbar_arrive_leader(&bars->kv_full);
          tma_load_3d_2sm(&p.tm_k, &bars->kv_full, smem + kKOff, 0, krow, un.hk);
          tma_load_3d_2sm(&p.tm_k, &bars->kv_full, smem + kKOff + kTileBytes / 2, 64, krow, un.hk);
          tma_load_3d_2sm(&p.tm_v, &bars->kv_full, smem + kVOff, 0, krow, un.hk);
          tma_load_3d_2sm(&p.tm_v, &bars->kv_full, smem + kVOff + kTileBytes / 2, 64, krow, un.hk);
        }
        ++kv_it;
        Cursor c;
        c.start(un, p.segs);
        for (int i = 0; i < un.n_iter; ++i, c.next(un, p.segs, p.group)) {
          const DevTask tk = p.tasks[p.segs[c.seg].task];
          const int head = un.hk * p.group + c.g;
          const int qrow = tk.q_off + c.qt * kTile;
          const float* nl = p.nlse2 + int64_t(head) * p.pitch;
          const float* nd = p.ndelta + int64_t(head) * p.pitch;
          // rows past the buffer only feed masked columns: clamp the source
          mbar_wait(&bars->q_empty[qr.i], qr.ph ^ 1);
          if (lane == 0) {
            if (leader) mbar_expect_tx(&bars->q_full[qr.i], 2 * kTileBytes);
            else mbar_arrive_leader(&bars->q_full[qr.i]);
            uint8_t* q = smem + kQOff + qr.i * kTileBytes;
            tma_load_3d_2sm(&p.tm_q64, &bars->q_full[qr.i], q, 0, qrow + 64 * int(rank), head);
            tma_load_3d_2sm(&p.tm_q64, &bars->q_full[qr.i], q + kTileBytes / 4, 64, qrow + 64 * int(rank), head);
            tma_load_3d_2sm(&p.tm_q, &bars->q_full[qr.i], q + kTileBytes / 2, 64 * int(rank), qrow, head);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int col = lane + 32 * k;
            cp_async4(lse_rows + qr.i * 128 + col, nl + min(int64_t(qrow) + col, p.pitch - 1));
          }
          cp_async_arrive(&bars->lse_full[qr.i]);
          qr.next();
          mbar_wait(&bars->do_empty[dr.i], dr.ph ^ 1);
          if (lane == 0) {
            if (leader) mbar_expect_tx(&bars->do_full[dr.i], 2 * kTileBytes);
            else mbar_arrive_leader(&bars->do_full[dr.i]);
            uint8_t* d = smem + kDOOff + dr.i * kTileBytes;
            tma_load_3d_2sm(&p.tm_do64, &bars->do_full[dr.i], d, 0, qrow + 64 * int(rank), head);
            tma_load_3d_2sm(&p.tm_do64, &bars->do_full[dr.i], d + kTileBytes / 4, 64, qrow + 64 * int(rank), head);
            tma_load_3d_2sm(&p.tm_do, &bars->do_full[dr.i], d + kTileBytes / 2, 64 * int(rank), qrow, head);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int col = lane + 32 * k;
            cp_async4(d_rows + dr.i * 128 + col, nd + min(int64_t(qrow) + col, p.pitch - 1));
          }
          cp_async_arrive(&bars->d_full[dr.i]);
          dr.next();
        }
      }
    } else if (warp == 9 && leader) {
      // ---------------------------------------------------------- MMA (even CTA)
      uint32_t kv_it = 0, acc_it = 0, p_ph = 0, ds_ph = 0;
      KRing<kQStages> qr;
      KRing<kDOStages> dr;
      const uint32_t sK = sbase + kKOff, sV = sbase + kVOff;
      for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
        const int u = sched_unit(p.sched, n_pairs, ui);
        const KvUnit un = p.units[u];
        const int n = un.n_iter;
        mbar_wait(&bars->kv_full, kv_it & 1);
        ++kv_it;
        mbar_wait(&bars->q_full[qr.i], qr.ph);
        tc_fence_after();
        uint32_t sQ = sbase + kQOff + qr.i * kTileBytes, sDO = sbase + kDOOff + dr.i * kTileBytes;
        issue_kq_pair(tS, sK, sQ);
        commit_pair(&bars->s_full);
        mbar_wait(&bars->do_full[dr.i], dr.ph);
        tc_fence_after();
        issue_kq_pair(tDP, sV, sDO);
        commit_pair(&bars->dp_full);
        if (n == 1) commit_pair(&bars->kv_empty);  // K / V read for the last time
        for (int i = 0; i < n; ++i) {
          const uint32_t qcur = qr.i, dcur = dr.i;
          qr.next();
          dr.next();
          // dV += P^T dO, in two K-halves (q columns [0,64) and [64,128)) as
          // the warpgroups release them
          mbar_wait(&bars->p_half, p_ph);
          if (i == 0) {
            mbar_wait(&bars->acc_free, (acc_it & 1) ^ 1);
            ++acc_it;
          }
          tc_fence_after();
          issue_acc_pair_half(tDV, tS + 16, sDO + kTileBytes / 2, 0, i > 0);
          mbar_wait(&bars->p_full, p_ph);
          p_ph ^= 1;
          tc_fence_after();
          issue_acc_pair_half(tDV, tS + 80, sDO + kTileBytes / 2, 1, true);
          const uint32_t nQ = sbase + kQOff + qr.i * kTileBytes, nDO = sbase + kDOOff + dr.i * kTileBytes;
          if (i + 1 < n) {
            mbar_wait(&bars->q_full[qr.i], qr.ph);
            tc_fence_after();
            issue_kq_pair(tS, sK, nQ);  // S^T(i+1): runs after dV(i) read P^T (in order)
            commit_pair(&bars->s_full);
          }
          mbar_wait(&bars->ds_half, ds_ph);  // dK += dS^T Q, likewise in K-halves
          tc_fence_after();
          issue_acc_pair_half(tDK, tDP + 16, sQ + kTileBytes / 2, 0, i > 0);
          mbar_wait(&bars->ds_full, ds_ph);
          ds_ph ^= 1;
          tc_fence_after();
          issue_acc_pair_half(tDK, tDP + 80, sQ + kTileBytes / 2, 1, true);
          commit_pair(&bars->q_empty[qcur]);   // Q(i): S^T(i), dK(i); its -LSE rows: exps(i)
          commit_pair(&bars->do_empty[dcur]);  // dO(i): dP^T(i), dV(i); its -D rows: dS(i)
          if (i + 1 < n) {
            mbar_wait(&bars->do_full[dr.i], dr.ph);
            tc_fence_after();
            issue_kq_pair(tDP, sV, nDO);  // dP^T(i+1)
            commit_pair(&bars->dp_full);
            // last reads of K / V issued: the next unit's tiles load under
            // this unit's last element-wise phase, dV/dK MMAs and epilogue
            if (i + 2 == n) commit_pair(&bars->kv_empty);
            sQ = nQ;
            sDO = nDO;
          }
        }
        commit_pair(&bars->acc_full);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    // ------------------------------------------------------------ elementwise
    const int w = warp >> 2;                    // q column chunks, see below
    const uint32_t r = (warp & 3) * 32 + lane;  // kv row within the tile
    const uint32_t lsel = ((warp & 3) * 32) << 16;
    const int c0 = 64 * w;
    const uint32_t tSw = tS + lsel, tDPw = tDP + lsel;
    uint32_t s_ph = 0, dp_ph = 0, acc_ph = 0;
    KRing<kQStages> qr;
    KRing<kDOStages> dr;
    for (int ui = sched_begin(p.sched, pair); ui < sched_end(p.sched, pair); ++ui) {
      const int u = sched_unit(p.sched, n_pairs, ui);
      const KvUnit un = p.units[u];
      const int kj = (un.tile + int(rank)) * kTile + r;  // key index relative to kv_off
      Cursor c;
      c.start(un, p.segs);
      for (int i = 0; i < un.n_iter; ++i, c.next(un, p.segs, p.group)) {
        const DevTask tk = p.tasks[p.segs[c.seg].task];
        const int shift = tk.kv_len - tk.n_q;
        mbar_wait_warp(&bars->lse_full[qr.i], qr.ph);  // the tile's -LSE rows (own copy)
        const uint32_t s_nlse = smem_u32(lse_rows + qr.i * 128), s_nd = smem_u32(d_rows + dr.i * 128);
        uint64_t* const do_full = &bars->d_full[dr.i];
        const uint32_t do_ph = dr.ph;
        qr.next();
        dr.next();
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
          // column k of the chunk is visible iff kj <= shift + qb + k and
          // qb + k < n_q; the chunk is mask-free (warp-uniform) when the
          // tile's last kv row is visible from its column 0 and all of its
          // columns are queries.
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
            if ((kDkdvEmuMask >> (k / 4)) & 1) {
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
        mbar_wait_warp(do_full, do_ph);  // the tile's -D rows
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
          tmem_st16(tDPw + 16 + 64 * ch + 16 * w, pk);  // dS^T (bf16), same layout
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive_leader(ch ? &bars->ds_full : &bars->ds_half);
        }
      }
      // ---- epilogue: warpgroup w stores d columns [c0, c0+64) of dV and dK
      mbar_wait_warp(&bars->acc_full, acc_ph);
      acc_ph ^= 1;
      tc_fence_after();
      const int row = un.kv_off + kj;
      const bool valid = row < un.kv_end;
      const int64_t off = (int64_t(row) * p.h_kv + un.hk) * kHeadDim + c0;
      const int row0 = un.kv_off + (un.tile + int(rank)) * kTile;
      if (CAD_KV2_TMA_STORE && row0 + kTile <= un.kv_end) {
        uint8_t* st = smem + kStOff + w * (kTileBytes / 2);
        if (r == 0) bulk_wait_read0();  // the previous unit's dK store has read the staging
        named_sync(1 + w, 128);
        tmem_row_to_smem_sw128(tDV + lsel + c0, 1.f, st, r);
        uint32_t pk[32];  // dK row, packed, while dV leaves
        tmem_row_to_regs_bf16(tDK + lsel + c0, p.scale, pk);
        tc_fence_before();
        mbar_arrive_leader(&bars->acc_free);  // TMEM read out: the next unit may accumulate
        fence_proxy_async_smem();
        named_sync(1 + w, 128);
        if (r == 0) {
          tma_store_3d(&p.tm_dv, st, c0, row0, un.hk);
          bulk_commit();
          bulk_wait_read0();
        }
        named_sync(1 + w, 128);
        regs_to_smem_sw128(pk, st, r);
        fence_proxy_async_smem();
        named_sync(1 + w, 128);
        if (r == 0) {
          tma_store_3d(&p.tm_dk, st, c0, row0, un.hk);
          bulk_commit();
        }
      } else {
        tmem_row_to_global(tDV + lsel + c0, 1.f, p.dv + off, valid);
        tmem_row_to_global(tDK + lsel + c0, p.scale, p.dk + off, valid);
        tc_fence_before();
        mbar_arrive_leader(&bars->acc_free);
      }
    }
  }
  if (CAD_KV2_TMA_STORE && warp < 8 && (warp & 3) == 0 && lane == 0) bulk_wait0();  // stores done
  tc_fence_before();
  cluster_sync_all();
  if (warp == 9) tmem_free_2sm<512>(tmem);
}

}  // namespace kv2

void preload_dkdv2() {
  set_max_smem(reinterpret_cast<const void*>(kv2::ca_bwd_dkdv_pair_kernel), kv2::kSmemBytes,
               "cudaFuncSetAttribute(dkdv2)");
}

// Launch of the pair dK/dV kernel (cluster dims 2); false if the plan has no pair units.
bool launch_dkdv_pair(const cad_ca_plan* plan, const void* q, const void* k, const void* v, const void* dout,
                      const float* nlse2, const float* ndelta, int64_t pitch, void* dk, void* dv,
                      cudaStream_t stream) {
  if (plan->kv2_units.empty()) return false;
  const cad_ca_shape& sh = plan->shape;
  kv2::Params p;
  make_tile_map(&p.tm_q, q, sh.q_rows, sh.h_q);
  make_tile_map(&p.tm_q64, q, sh.q_rows, sh.h_q, 64);
  make_tile_map(&p.tm_do, dout, sh.q_rows, sh.h_q);
  make_tile_map(&p.tm_do64, dout, sh.q_rows, sh.h_q, 64);
  make_tile_map(&p.tm_k, k, sh.kv_rows, sh.h_kv);
  make_tile_map(&p.tm_v, v, sh.kv_rows, sh.h_kv);
  make_tile_map(&p.tm_dk, dk, sh.kv_rows, sh.h_kv);
  make_tile_map(&p.tm_dv, dv, sh.kv_rows, sh.h_kv);
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
  set_max_smem(reinterpret_cast<const void*>(kv2::ca_bwd_dkdv_pair_kernel), kv2::kSmemBytes,
               "cudaFuncSetAttribute(dkdv2)");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * plan->sched_kv2.G);
  cfg.blockDim = dim3(kv2::kThreads);
  cfg.dynamicSmemBytes = kv2::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cuda_check(cudaLaunchKernelEx(&cfg, kv2::ca_bwd_dkdv_pair_kernel, p), "ca_bwd_dkdv_pair launch");
  return true;
}

}  // namespace cad_dev
