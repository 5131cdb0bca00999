// CA backward on sm_100a: dQ, dK, dV of O = softmax(scale Q K^T + mask) V
// over the server's CA-tasks, recomputing P from the forward's LSE (no
// materialised P).
//
// Three launches, all deterministic (no atomics):
//   1. ca_delta:   D[h][row] = sum_d dO * O (fp32).
//   2. ca_bwd_dkdv: one unit per (KV group, kv tile, KV head). For every
//      query head of the GQA group and every 64-row q sub-tile that can see
//      the kv tile (two sub-tiles in flight, one per warpgroup):
//        S^T = K Q^T, dP^T = V dO^T                        (tcgen05 -> TMEM)
//        P^T = exp(S^T - LSE), dS^T = P^T (dP^T - D)      (2 warpgroups, bf16
//                                                          written back to TMEM)
//        dV += P^T dO, dK += dS^T Q                        (A operand in TMEM)
//      dK/dV stay in TMEM for the whole unit and are stored once (bf16).
//   3. ca_bwd_dq: one unit per (task, q tile, query head), walking its kv
//      tiles: S = Q K^T, dP = dO V^T, dS = P (dP - D), dQ += dS K; dQ stays in
//      TMEM and is stored once.
// The dQ pass recomputes S and dP (7 tile GEMMs instead of 5) in exchange for
// no fp32 dQ atomics and exact determinism.
//
// Both main kernels: 12 warps = elementwise warpgroups 0 and 1 (thread =
// TMEM lane = tile row), control warpgroup 2 (warp 8 TMA producer, warp 9
// MMA issuer).
#define CAD_KERNEL_TAG "ca_bwd"  // names this file in the mbarrier-timeout report
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "../host/cad_status.hpp"
#include "ca_common.cuh"
#include "ca_mma.cuh"
#include "ca_rows.cuh"
#include "sm100.cuh"

namespace cad_dev {
namespace bwd {

constexpr int kThreads = 384;
constexpr float kLog2e = 1.4426950408889634f;

// ============================================================== D = rowsum
// One CTA per chunk of <= 32 consecutive query rows of a task, all heads:
// half-warps take (row, head) pairs in memory order (16-byte loads of the
// 256-byte dO and O head rows, fully coalesced), the sums go through shared
// memory, and -D plus the forward's LSE as -LSE*log2(e) are written as
// 128-byte runs of the [h_q][pitch] rows (negated so the consumers fold them
// into one FFMA2/FADD2). HBM-bound: 2 x 256 B read per (row, head).
constexpr int kDeltaThreads = 256;
__global__ void __launch_bounds__(kDeltaThreads) ca_delta_kernel(const int2* chunks, const __nv_bfloat16* o,
                                                                 const __nv_bfloat16* dout, const float* lse,
                                                                 float* delta, float* lse2, int h_q, int64_t q_rows,
                                                                 int64_t pitch) {
  extern __shared__ float dsum[];  // [h_q][32]
  const int2 ch = chunks[blockIdx.x];
  const int hw = threadIdx.x >> 4, l16 = threadIdx.x & 15;
  const int items = ch.y * h_q;
  const uint4* o4 = reinterpret_cast<const uint4*>(o + int64_t(ch.x) * h_q * kHeadDim);
  const uint4* d4 = reinterpret_cast<const uint4*>(dout + int64_t(ch.x) * h_q * kHeadDim);
  constexpr int kU = 4;
  for (int base = hw; base < items; base += kU * (kDeltaThreads / 16)) {
    uint4 a[kU], b[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int it = base + u * (kDeltaThreads / 16);
      if (it < items) {
        a[u] = __ldg(o4 + int64_t(it) * 16 + l16);
        b[u] = __ldg(d4 + int64_t(it) * 16 + l16);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int it = base + u * (kDeltaThreads / 16);
      const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&a[u]);
      const __nv_bfloat162* b2 = reinterpret_cast<const __nv_bfloat162*>(&b[u]);
      float s = 0.f;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 fa = __bfloat1622float2(a2[i]);
        const float2 fb = __bfloat1622float2(b2[i]);
        s += fa.x * fb.x + fa.y * fb.y;
      }
#pragma unroll
      for (int off = 8; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
      if (l16 == 0 && it < items) dsum[(it % h_q) * 32 + it / h_q] = s;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < h_q * 32; i += kDeltaThreads) {
    const int h = i >> 5, r = i & 31;
    if (r < ch.y) {
      const int64_t row = ch.x + r;
      delta[int64_t(h) * pitch + row] = -dsum[i];
      lse2[int64_t(h) * pitch + row] = -lse[int64_t(h) * q_rows + row] * kLog2e;
    }
  }
}

// ============================================================== dK / dV
namespace kv {

// 128-row q tiles; all four GEMMs are M=128, N=128 (the tensor core reads
// its SS operands from shared memory at a fixed rate, so N=64 MMAs ran
// smem-bound).
//   TMEM: S^T [0,128)  dP^T [128,256)  dV [256,384)  dK [384,512)
// Iteration i: S^T(i), dP^T(i) -> both warpgroups. Warpgroup w owns q
// columns [32w, 32w+32) and [64+32w, 64+32w+32), so the two warpgroups
// together finish q columns [0,64) (= the first K-half of dV/dK) halfway
// through: P^T -> p_half, p_full; dS^T -> ds_half, ds_full. The bf16 P^T
// (dS^T) of K-half h is written into the packed columns [16+64h, 48+64h)
// of S^T (dP^T), inside the columns each warpgroup itself read.
// MMA order: dV(i) half 0 | dV(i) half 1 | S^T(i+1) | dK(i) halves |
// dP^T(i+1): the tensor core runs dV(i)+S^T(i+1) while the warpgroups
// compute dS^T(i), and dK(i)+dP^T(i+1) while they exponentiate i+1.
#ifndef CAD_DKDV_EMU_MASK
#define CAD_DKDV_EMU_MASK 0x1111  // 25 %: measured -4 % dK/dV time
#endif
// one bit per group of 4 q columns: 1 = polynomial exp2 on the FMA pipe
constexpr uint32_t kDkdvEmuMask = CAD_DKDV_EMU_MASK;
// Q tiles are staged 3 deep and dO tiles 2 deep: S^T(i+1) needs Q(i+1)
// right after dV(i), while Q(i) still feeds dK(i) and the slot of Q(i-1)
// only frees after dK(i-1) -- with 2 stages the MMA warp waited ~280 cycles
// per iteration for Q(i+1) to land (clock64 trace, scripts/timeline_dkdv.py).
constexpr int kQStages = 3, kDOStages = 2;
constexpr uint32_t kKOff = 0;
constexpr uint32_t kVOff = kTileBytes;
constexpr uint32_t kQOff = 2 * kTileBytes;                    // kQStages x 32 KB
constexpr uint32_t kDOOff = kQOff + kQStages * kTileBytes;    // kDOStages x 32 KB
constexpr uint32_t kLseOff = kDOOff + kDOStages * kTileBytes; // [q stage][128] -LSE*log2e fp32
constexpr uint32_t kDOff = kLseOff + kQStages * 512;          // [dO stage][128] -D fp32
constexpr uint32_t kBarOff = kDOff + kDOStages * 512;
// Dynamic shared memory starts 1024-aligned (no static shared memory in this
// kernel; checked at run time), so the budget carries no alignment slack.
constexpr uint32_t kSmemBytes = kBarOff + 256;
static_assert(kSmemBytes <= 232448, "dK/dV shared memory");

struct Bars {
  uint64_t kv_full, kv_empty;
  uint64_t q_full[kQStages], q_empty[kQStages], do_full[kDOStages], do_empty[kDOStages];
  uint64_t s_full, dp_full, p_half, p_full, ds_half, ds_full, acc_full, acc_free;
  uint32_t tmem_base;
};
static_assert(sizeof(Bars) <= 256, "dK/dV barriers");

// Slot index + phase of a ring of N stages.
template <int N>
struct KRing {
  uint32_t i = 0, ph = 0;
  __device__ void next() {
    if (++i == N) { i = 0; ph ^= 1; }
  }
};

struct Params {
  CUtensorMap tm_q, tm_k, tm_v, tm_do;
  const float* nlse2;   // -LSE * log2(e), [h_q][pitch]
  const float* ndelta;  // -D, [h_q][pitch]
  int64_t pitch;
  const DevTask* tasks;
  const KvUnit* units;
  const KvSeg* segs;
  int n_units;
  const int32_t* sched;  // per-CTA work lists (CtaLists)
  int group;
  int h_kv;
  __nv_bfloat16* dk;
  __nv_bfloat16* dv;
  float scale;       // softmax scale (dK multiplier)
  float scale_log2;  // softmax scale * log2(e)
};

// Iteration cursor over (segment, q tile, head in group) of one unit. q tiles
// are walked from the LAST one down to the first that sees the kv tile, so
// co-running CTAs (consecutive kv tiles of one document) stream the same Q/dO
// rows at the same time; the GQA heads are innermost.
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

__global__ void __launch_bounds__(kThreads, 1) ca_bwd_dkdv_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem[];
  Bars* bars = reinterpret_cast<Bars*>(smem + kBarOff);
  float* lse_rows = reinterpret_cast<float*>(smem + kLseOff);
  float* d_rows = reinterpret_cast<float*>(smem + kDOff);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t warp = warp_id(), lane = lane_id();
  if (sbase & 1023) __trap();  // SW128 tiles need 1024-byte alignment

  if (warp == 8 && lane == 0) {
    tma_prefetch(&p.tm_q);
    tma_prefetch(&p.tm_k);
    tma_prefetch(&p.tm_v);
    tma_prefetch(&p.tm_do);
    mbar_init(&bars->kv_full, 1);
    mbar_init(&bars->kv_empty, 1);
    for (int i = 0; i < kQStages; ++i) {
      mbar_init(&bars->q_full[i], 33);
      mbar_init(&bars->q_empty[i], 1);
    }
    for (int i = 0; i < kDOStages; ++i) {
      mbar_init(&bars->do_full[i], 33);
      mbar_init(&bars->do_empty[i], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->p_half, 256);
    mbar_init(&bars->p_full, 256);
    mbar_init(&bars->ds_half, 256);
    mbar_init(&bars->ds_full, 256);
    mbar_init(&bars->acc_full, 1);
    mbar_init(&bars->acc_free, 256);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const uint32_t tS = tmem, tDP = tmem + 128, tDV = tmem + 256, tDK = tmem + 384;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (warp == 8) {
      // ---------------------------------------------------------- producer
      // Lane 0 issues the TMA tile loads; the whole warp copies the tile's
      // 128 -LSE and 128 -D values (arbitrary, unaligned row offsets, so
      // cp.async rather than TMA); each lane's async arrives land on q_full
      // (-LSE, with Q) and do_full (-D, with dO) when its copies have (count
      // 1 + 32 each).
      uint32_t kv_it = 0;
      KRing<kQStages> qr;
      KRing<kDOStages> dr;
      for (int ui = sched_begin(p.sched, blockIdx.x); ui < sched_end(p.sched, blockIdx.x); ++ui) {
        const int u = sched_unit(p.sched, gridDim.x, ui);
        const KvUnit un = p.units[u];
        const int krow = un.kv_off + un.tile * kTile;
        if (lane == 0) {
          mbar_wait(&bars->kv_empty, (kv_it & 1) ^ 1);
          mbar_expect_tx(&bars->kv_full, 2 * kTileBytes);
          tma_load_3d(&p.tm_k, &bars->kv_full, smem + kKOff, 0, krow, un.hk);
          tma_load_3d(&p.tm_k, &bars->kv_full, smem + kKOff + kTileBytes / 2, 64, krow, un.hk);
          tma_load_3d(&p.tm_v, &bars->kv_full, smem + kVOff, 0, krow, un.hk);
          tma_load_3d(&p.tm_v, &bars->kv_full, smem + kVOff + kTileBytes / 2, 64, krow, un.hk);
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
            mbar_expect_tx(&bars->q_full[qr.i], kTileBytes);
            uint8_t* q = smem + kQOff + qr.i * kTileBytes;
            tma_load_3d(&p.tm_q, &bars->q_full[qr.i], q, 0, qrow, head);
            tma_load_3d(&p.tm_q, &bars->q_full[qr.i], q + kTileBytes / 2, 64, qrow, head);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int col = lane + 32 * k;
            cp_async4(lse_rows + qr.i * 128 + col, nl + min(int64_t(qrow) + col, p.pitch - 1));
          }
          cp_async_arrive(&bars->q_full[qr.i]);
          qr.next();
          mbar_wait(&bars->do_empty[dr.i], dr.ph ^ 1);
          if (lane == 0) {
            mbar_expect_tx(&bars->do_full[dr.i], kTileBytes);
            uint8_t* d = smem + kDOOff + dr.i * kTileBytes;
            tma_load_3d(&p.tm_do, &bars->do_full[dr.i], d, 0, qrow, head);
            tma_load_3d(&p.tm_do, &bars->do_full[dr.i], d + kTileBytes / 2, 64, qrow, head);
          }
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int col = lane + 32 * k;
            cp_async4(d_rows + dr.i * 128 + col, nd + min(int64_t(qrow) + col, p.pitch - 1));
          }
          cp_async_arrive(&bars->do_full[dr.i]);
          dr.next();
        }
      }
    } else if (warp == 9) {
      // ---------------------------------------------------------- MMA
      uint32_t kv_it = 0, acc_it = 0, p_ph = 0, ds_ph = 0;
      KRing<kQStages> qr;
      KRing<kDOStages> dr;
      const uint32_t sK = sbase + kKOff, sV = sbase + kVOff;
      for (int ui = sched_begin(p.sched, blockIdx.x); ui < sched_end(p.sched, blockIdx.x); ++ui) {
        const int u = sched_unit(p.sched, gridDim.x, ui);
        const KvUnit un = p.units[u];
        const int n = un.n_iter;
        mbar_wait(&bars->kv_full, kv_it & 1);
        ++kv_it;
        mbar_wait(&bars->q_full[qr.i], qr.ph);
        tc_fence_after();
        uint32_t sQ = sbase + kQOff + qr.i * kTileBytes, sDO = sbase + kDOOff + dr.i * kTileBytes;
        issue_qk(tS, sK, sQ);
        mma_commit(&bars->s_full);
        mbar_wait(&bars->do_full[dr.i], dr.ph);
        tc_fence_after();
        issue_qk(tDP, sV, sDO);
        mma_commit(&bars->dp_full);
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
          issue_pv_half(tDV, tS + 16, sDO, 0, i > 0);
          mbar_wait(&bars->p_full, p_ph);
          p_ph ^= 1;
          tc_fence_after();
          issue_pv_half(tDV, tS + 80, sDO, 1, true);
          const uint32_t nQ = sbase + kQOff + qr.i * kTileBytes, nDO = sbase + kDOOff + dr.i * kTileBytes;
          if (i + 1 < n) {
            mbar_wait(&bars->q_full[qr.i], qr.ph);
            tc_fence_after();
            issue_qk(tS, sK, nQ);  // S^T(i+1): runs after dV(i) read P^T (in order)
            mma_commit(&bars->s_full);
          }
          mbar_wait(&bars->ds_half, ds_ph);  // dK += dS^T Q, likewise in K-halves
          tc_fence_after();
          issue_pv_half(tDK, tDP + 16, sQ, 0, i > 0);
          mbar_wait(&bars->ds_full, ds_ph);
          ds_ph ^= 1;
          tc_fence_after();
          issue_pv_half(tDK, tDP + 80, sQ, 1, true);
          mma_commit(&bars->q_empty[qcur]);   // Q(i): S^T(i), dK(i); its -LSE rows: exps(i)
          mma_commit(&bars->do_empty[dcur]);  // dO(i): dP^T(i), dV(i); its -D rows: dS(i)
          if (i + 1 < n) {
            mbar_wait(&bars->do_full[dr.i], dr.ph);
            tc_fence_after();
            issue_qk(tDP, sV, nDO);  // dP^T(i+1)
            mma_commit(&bars->dp_full);
            sQ = nQ;
            sDO = nDO;
          }
        }
        mma_commit(&bars->acc_full);
        mma_commit(&bars->kv_empty);
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
    for (int ui = sched_begin(p.sched, blockIdx.x); ui < sched_end(p.sched, blockIdx.x); ++ui) {
      const int u = sched_unit(p.sched, gridDim.x, ui);
      const KvUnit un = p.units[u];
      const int kj = un.tile * kTile + r;  // key index relative to kv_off
      Cursor c;
      c.start(un, p.segs);
      for (int i = 0; i < un.n_iter; ++i, c.next(un, p.segs, p.group)) {
        const DevTask tk = p.tasks[p.segs[c.seg].task];
        const int shift = tk.kv_len - tk.n_q;
        mbar_wait_warp(&bars->q_full[qr.i], qr.ph);  // Q(i) and its -LSE rows
        const uint32_t s_nlse = smem_u32(lse_rows + qr.i * 128), s_nd = smem_u32(d_rows + dr.i * 128);
        uint64_t* const do_full = &bars->do_full[dr.i];
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
          const bool full = (un.tile * kTile + kTile - 1 - shift - qb) <= 0 && hi >= 32;
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
          mbar_arrive(ch ? &bars->p_full : &bars->p_half);
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
          const bool full = (un.tile * kTile + kTile - 1 - shift - qb) <= 0 && hi >= 32;
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
          mbar_arrive(ch ? &bars->ds_full : &bars->ds_half);
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
      mbar_arrive(&bars->acc_free);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_free<512>(tmem);
}

}  // namespace kv

// ============================================================== dQ
namespace dq {

#ifndef CAD_DQ_EMU_MASK
#define CAD_DQ_EMU_MASK 0  // measured: no gain (dQ is not MUFU-bound)
#endif
// one bit per group of 4 kv columns: 1 = polynomial exp2 on the FMA pipe
constexpr uint32_t kDqEmuMask = CAD_DQ_EMU_MASK;
// K tiles are read twice per iteration (S(j) and, later, dQ(j)), V once
// (dP(j)): a 3-deep K ring and a 2-deep V ring, each slot freed as soon as
// its last reader completes.
constexpr int kKStages = 3, kVStages = 2;
constexpr uint32_t kQOff = 0;
constexpr uint32_t kDOOff = kTileBytes;
constexpr uint32_t kKOff = 2 * kTileBytes;
constexpr uint32_t kVOff = kKOff + kKStages * kTileBytes;
constexpr uint32_t kBarOff = kVOff + kVStages * kTileBytes;
constexpr uint32_t kSmemBytes = kBarOff + 256 + 1024;
static_assert(kSmemBytes <= 232448, "dQ shared memory");

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[kKStages], k_empty[kKStages], v_full[kVStages], v_empty[kVStages];
  // ds_full per dS buffer (j & 1), see ca_dq2.cu
  uint64_t s_full, dp_full, p_read, dp_read, ds_full[2], dq_full, dq_free;
  uint32_t tmem_base;
};

// Slot index + phase of a ring of N stages.
template <int N>
struct Ring {
  uint32_t i = 0, ph = 0;
  __device__ void next() {
    if (++i == N) { i = 0; ph ^= 1; }
  }
};

struct Params {
  CUtensorMap tm_q, tm_k, tm_v, tm_do;
  const DevTask* tasks;
  const FwdUnit* units;
  int n_units;
  const int32_t* sched;  // per-CTA work lists (CtaLists)
  int group;
  int h_q;
  const float* lse2;   // -LSE * log2(e), [h_q][pitch]
  const float* delta;  // -D, [h_q][pitch]
  __nv_bfloat16* dq;
  int64_t pitch;
  float scale;
  float scale_log2;
};

__global__ void __launch_bounds__(kThreads, 1) ca_bwd_dq_kernel(const __grid_constant__ Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars* bars = reinterpret_cast<Bars*>(smem + kBarOff);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 8 && lane == 0) {
    tma_prefetch(&p.tm_q);
    tma_prefetch(&p.tm_k);
    tma_prefetch(&p.tm_v);
    tma_prefetch(&p.tm_do);
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&bars->k_full[i], 1);
      mbar_init(&bars->k_empty[i], 1);
    }
    for (int i = 0; i < kVStages; ++i) {
      mbar_init(&bars->v_full[i], 1);
      mbar_init(&bars->v_empty[i], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->p_read, 256);
    mbar_init(&bars->dp_read, 256);
    mbar_init(&bars->ds_full[0], 256);
    mbar_init(&bars->ds_full[1], 256);
    mbar_init(&bars->dq_full, 1);
    mbar_init(&bars->dq_free, 256);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  // TMEM: S [0,128)  dP [128,256)  dQ [256,384)  dS buffers [384,448) [448,512)
  const uint32_t tS = tmem, tDP = tmem + 128, tDQ = tmem + 256, tDS = tmem + 384;

  if (warp >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (warp == 8 && lane == 0) {
      uint32_t q_it = 0;
      Ring<kKStages> kr;
      Ring<kVStages> vr;
      for (int ui = sched_begin(p.sched, blockIdx.x); ui < sched_end(p.sched, blockIdx.x); ++ui) {
        const int u = sched_unit(p.sched, gridDim.x, ui);
        const FwdUnit un = p.units[u];
        const DevTask tk = p.tasks[un.task];
        const int hk = un.head0 / p.group;
        const int qrow = tk.q_off + un.tile * kTile;
        mbar_wait(&bars->q_empty, (q_it & 1) ^ 1);
        ++q_it;
        mbar_expect_tx(&bars->q_full, 2 * kTileBytes);
        tma_load_3d(&p.tm_q, &bars->q_full, smem + kQOff, 0, qrow, un.head0);
        tma_load_3d(&p.tm_q, &bars->q_full, smem + kQOff + kTileBytes / 2, 64, qrow, un.head0);
        tma_load_3d(&p.tm_do, &bars->q_full, smem + kDOOff, 0, qrow, un.head0);
        tma_load_3d(&p.tm_do, &bars->q_full, smem + kDOOff + kTileBytes / 2, 64, qrow, un.head0);
        for (int j = 0; j < un.n_kv; ++j) {
          const int krow = tk.kv_off + j * kTile;
          mbar_wait(&bars->k_empty[kr.i], kr.ph ^ 1);
          mbar_expect_tx(&bars->k_full[kr.i], kTileBytes);
          uint8_t* k = smem + kKOff + kr.i * kTileBytes;
          tma_load_3d(&p.tm_k, &bars->k_full[kr.i], k, 0, krow, hk);
          tma_load_3d(&p.tm_k, &bars->k_full[kr.i], k + kTileBytes / 2, 64, krow, hk);
          kr.next();
          mbar_wait(&bars->v_empty[vr.i], vr.ph ^ 1);
          mbar_expect_tx(&bars->v_full[vr.i], kTileBytes);
          uint8_t* v = smem + kVOff + vr.i * kTileBytes;
          tma_load_3d(&p.tm_v, &bars->v_full[vr.i], v, 0, krow, hk);
          tma_load_3d(&p.tm_v, &bars->v_full[vr.i], v + kTileBytes / 2, 64, krow, hk);
          vr.next();
        }
      }
    } else if (warp == 9) {
      // Per iteration j: S(j+1) as soon as the S(j) rows are in registers,
      // dP(j+1) as soon as the dP(j) rows are, then dQ(j) once dS(j) is in
      // TMEM (dS is double-buffered, so dS(j+1) can be written meanwhile).
      uint32_t q_it = 0, dq_it = 0, pr_ph = 0, dr_ph = 0, ds_ph[2] = {0, 0};
      Ring<kKStages> kr;
      Ring<kVStages> vr;
      for (int ui = sched_begin(p.sched, blockIdx.x); ui < sched_end(p.sched, blockIdx.x); ++ui) {
        const int u = sched_unit(p.sched, gridDim.x, ui);
        const FwdUnit un = p.units[u];
        const int n = un.n_kv;
        mbar_wait(&bars->q_full, q_it & 1);
        ++q_it;
        const uint32_t sQ = sbase + kQOff, sDO = sbase + kDOOff;
        mbar_wait(&bars->k_full[kr.i], kr.ph);
        tc_fence_after();
        issue_qk(tS, sQ, sbase + kKOff + kr.i * kTileBytes);  // S(0)
        mma_commit(&bars->s_full);
        mbar_wait(&bars->v_full[vr.i], vr.ph);
        tc_fence_after();
        issue_qk(tDP, sDO, sbase + kVOff + vr.i * kTileBytes);  // dP(0)
        mma_commit(&bars->dp_full);
        mma_commit(&bars->v_empty[vr.i]);
        vr.next();
        for (int j = 0; j < n; ++j) {
          const uint32_t kcur = kr.i;
          kr.next();
          mbar_wait(&bars->p_read, pr_ph);
          pr_ph ^= 1;
          if (j + 1 < n) {
            mbar_wait(&bars->k_full[kr.i], kr.ph);
            tc_fence_after();
            issue_qk(tS, sQ, sbase + kKOff + kr.i * kTileBytes);  // S(j+1)
            mma_commit(&bars->s_full);
          }
          mbar_wait(&bars->dp_read, dr_ph);
          dr_ph ^= 1;
          if (j + 1 < n) {
            mbar_wait(&bars->v_full[vr.i], vr.ph);
            tc_fence_after();
            issue_qk(tDP, sDO, sbase + kVOff + vr.i * kTileBytes);  // dP(j+1)
            mma_commit(&bars->dp_full);
            mma_commit(&bars->v_empty[vr.i]);
            vr.next();
          }
          mbar_wait(&bars->ds_full[j & 1], ds_ph[j & 1]);
          ds_ph[j & 1] ^= 1;
          if (j == 0) {
            mbar_wait(&bars->dq_free, (dq_it & 1) ^ 1);
            ++dq_it;
          }
          tc_fence_after();
          const uint32_t ds = tDS + (j & 1) * 64;
          issue_pv(tDQ, ds, ds + 32, sbase + kKOff + kcur * kTileBytes, j > 0);  // dQ += dS K
          mma_commit(&bars->k_empty[kcur]);
        }
        mma_commit(&bars->dq_full);
        mma_commit(&bars->q_empty);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    const int w = warp >> 2;                    // kv column half [64w, 64w+64)
    const uint32_t r = (warp & 3) * 32 + lane;  // q row within the tile
    const uint32_t lsel = ((warp & 3) * 32) << 16;
    const int c0 = 64 * w;
    uint32_t s_ph = 0, dp_ph = 0, dq_ph = 0;
    for (int ui = sched_begin(p.sched, blockIdx.x); ui < sched_end(p.sched, blockIdx.x); ++ui) {
      const int u = sched_unit(p.sched, gridDim.x, ui);
      const FwdUnit un = p.units[u];
      const DevTask tk = p.tasks[un.task];
      const int shift = tk.kv_len - tk.n_q;
      const int qi = un.tile * kTile + r;
      const bool valid = qi < tk.n_q;
      const int64_t row = int64_t(tk.q_off) + qi;
      const float lse2 = valid ? -p.lse2[int64_t(un.head0) * p.pitch + row] : 0.f;
      const float dd = valid ? -p.delta[int64_t(un.head0) * p.pitch + row] : 0.f;
      const int pos = valid ? shift + qi : -1;  // invalid rows see nothing
      const bool all_rows = un.tile * kTile + kTile <= tk.n_q;
      for (int j = 0; j < un.n_kv; ++j) {
        mbar_wait_warp(&bars->s_full, s_ph);
        s_ph ^= 1;
        tc_fence_after();
        float x[64];
        load_row64(tS + lsel + c0, x);
        tc_fence_before();
        mbar_arrive(&bars->p_read);
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
        mbar_wait_warp(&bars->dp_full, dp_ph);
        dp_ph ^= 1;
        tc_fence_after();
        float y[64];
        load_row64(tDP + lsel + c0, y);
        tc_fence_before();
        mbar_arrive(&bars->dp_read);
        const uint64_t nd2 = f2(-dd, -dd);
#pragma unroll
        for (int k = 0; k < 64; k += 2)
          f2_split(fmul2(f2(x[k], x[k + 1]), fadd2(f2(y[k], y[k + 1]), nd2)), y[k], y[k + 1]);
        store_bf16_64(tDS + lsel + (j & 1) * 64 + 32 * w, y);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars->ds_full[j & 1]);
      }
      mbar_wait_warp(&bars->dq_full, dq_ph);
      dq_ph ^= 1;
      tc_fence_after();
      tmem_row_to_global(tDQ + lsel + c0, p.scale,
                         p.dq + (row * p.h_q + un.head0) * kHeadDim + c0, valid);
      tc_fence_before();
      mbar_arrive(&bars->dq_free);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_free<512>(tmem);
}

}  // namespace dq
}  // namespace bwd

void preload_bwd() {
  set_max_smem(reinterpret_cast<const void*>(bwd::kv::ca_bwd_dkdv_kernel), bwd::kv::kSmemBytes,
               "cudaFuncSetAttribute(dkdv)");
  set_max_smem(reinterpret_cast<const void*>(bwd::dq::ca_bwd_dq_kernel), bwd::dq::kSmemBytes,
               "cudaFuncSetAttribute(dq)");
  cudaFuncAttributes a;
  cuda_check(cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(bwd::ca_delta_kernel)), "load delta");
}
}  // namespace cad_dev

extern "C" int cad_ca_bwd_parts(const cad_ca_plan* plan, const void* q, const void* k,
                                const void* v, const void* o, const float* lse, const void* dout,
                                void* dq, void* dk, void* dv, void* workspace, size_t ws_bytes,
                                int parts, void* stream) {
  using namespace cad_dev;
  using namespace cad_dev::bwd;
  return cad::guarded([&] {
    if (!plan || !q || !k || !v || !o || !lse || !dout || !dq || !dk || !dv || !workspace)
      throw cad::DomainError("null argument");
    const cad_ca_shape& sh = plan->shape;
    const int64_t pitch = (sh.q_rows + 3) / 4 * 4;
    const size_t need = size_t(2) * pitch * sh.h_q * 4;
    if (ws_bytes < need) throw cad::DomainError("backward workspace too small");
    if (plan->tasks.empty()) return;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    static const bool debug_sync = std::getenv("CAD_DEBUG_SYNC") != nullptr;
    float* delta = static_cast<float*>(workspace);
    float* lse2 = delta + pitch * sh.h_q;
    DeviceGuard dg(plan->device);
    set_max_smem(reinterpret_cast<const void*>(kv::ca_bwd_dkdv_kernel), kv::kSmemBytes, "cudaFuncSetAttribute(dkdv)");
    set_max_smem(reinterpret_cast<const void*>(dq::ca_bwd_dq_kernel), dq::kSmemBytes, "cudaFuncSetAttribute(dq)");
    // 1. D = rowsum(dO * O)
    if ((parts & CAD_BWD_DELTA) && !plan->row_chunks.empty()) {
      ca_delta_kernel<<<static_cast<unsigned>(plan->row_chunks.size()), kDeltaThreads, sh.h_q * 32 * 4, s>>>(
          plan->d_row_chunks, static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), lse,
          delta, lse2, sh.h_q, sh.q_rows, pitch);
      cuda_check(cudaGetLastError(), "ca_delta launch");
      if (debug_sync) cuda_check(cudaStreamSynchronize(s), "ca_delta");
    }
    // 2-3 fused (experimental, CAD_BWD_FUSED=1, when the workspace holds the
    // fp32 dQ accumulator and the plan has pair units): the pair kernel
    // computes dK, dV and adds the dQ partials into the accumulator
    // (CAD_BWD_DKDV), the conversion writes dQ (CAD_BWD_DQ).
    static const bool pair_off = std::getenv("CAD_DKDV_PAIR") && std::getenv("CAD_DKDV_PAIR")[0] == '0';
    if (fused_bwd_enabled() && !pair_off && ws_bytes >= need + dq_acc_bytes(sh) && !plan->kv2_units.empty()) {
      float* acc = reinterpret_cast<float*>(static_cast<char*>(workspace) + need);
      if (parts & CAD_BWD_DKDV) {
        launch_dkdvq_pair(plan, q, k, v, dout, lse2, delta, pitch, dk, dv, acc, s);
        if (debug_sync) cuda_check(cudaStreamSynchronize(s), "ca_bwd_dkdvq_pair");
      }
      if (parts & CAD_BWD_DQ) {
        launch_dq_convert(plan, acc, dq, s);
        if (debug_sync) cuda_check(cudaStreamSynchronize(s), "dq_convert");
      }
      return;
    }
    // 2-3. dK/dV then dQ on `stream`; CAD_BWD_FORK=1 forks dQ onto the plan's
    // side stream (joined back below) so its CTAs take the SMs dK/dV's tail
    // frees -- measured 0.5-1 % slower, hence off by default
    static const bool fork_on = std::getenv("CAD_BWD_FORK") && std::getenv("CAD_BWD_FORK")[0] == '1';
    const bool fork = fork_on && (parts & CAD_BWD_DKDV) && (parts & CAD_BWD_DQ) && plan->side;
    cudaStream_t s_dq = s;
    if (fork) {
      cuda_check(cudaEventRecord(plan->ev_fork, s), "event(fork)");
      cuda_check(cudaStreamWaitEvent(plan->side, plan->ev_fork, 0), "wait(fork)");
      s_dq = plan->side;
    }
    // 2. dK, dV (CTA pairs unless CAD_DKDV_PAIR=0)
    static const bool dkdv_pair_off = std::getenv("CAD_DKDV_PAIR") && std::getenv("CAD_DKDV_PAIR")[0] == '0';
    if ((parts & CAD_BWD_DKDV) && !dkdv_pair_off &&
        launch_dkdv_pair(plan, q, k, v, dout, lse2, delta, pitch, dk, dv, s)) {
      if (debug_sync) cuda_check(cudaStreamSynchronize(s), "ca_bwd_dkdv_pair");
    } else if ((parts & CAD_BWD_DKDV) && !plan->kv_units.empty()) {
      kv::Params p;
      make_tile_map(&p.tm_q, q, sh.q_rows, sh.h_q);
      make_tile_map(&p.tm_do, dout, sh.q_rows, sh.h_q);
      make_tile_map(&p.tm_k, k, sh.kv_rows, sh.h_kv);
      make_tile_map(&p.tm_v, v, sh.kv_rows, sh.h_kv);
      p.nlse2 = lse2;
      p.ndelta = delta;
      p.pitch = pitch;
      p.tasks = plan->d_tasks;
      p.units = plan->d_kv;
      p.segs = plan->d_segs;
      p.n_units = static_cast<int>(plan->kv_units.size());
      p.sched = plan->sched_kv.d;
      p.group = sh.h_q / sh.h_kv;
      p.h_kv = sh.h_kv;
      p.dk = static_cast<__nv_bfloat16*>(dk);
      p.dv = static_cast<__nv_bfloat16*>(dv);
      p.scale = sh.softmax_scale;
      p.scale_log2 = sh.softmax_scale * kLog2e;
      const int grid = plan->sched_kv.G;
      kv::ca_bwd_dkdv_kernel<<<grid, kThreads, kv::kSmemBytes, s>>>(p);
      cuda_check(cudaGetLastError(), "ca_bwd_dkdv launch");
      if (debug_sync) cuda_check(cudaStreamSynchronize(s), "ca_bwd_dkdv");
    }
    // 3. dQ (CTA pairs for even GQA groups unless CAD_DQ_PAIR=0)
    static const bool dq_pair_off = std::getenv("CAD_DQ_PAIR") && std::getenv("CAD_DQ_PAIR")[0] == '0';
    if ((parts & CAD_BWD_DQ) && !dq_pair_off &&
        launch_dq_pair(plan, q, k, v, dout, lse2, delta, pitch, dq, s_dq)) {
      if (debug_sync) cuda_check(cudaStreamSynchronize(s_dq), "ca_bwd_dq_pair");
    } else if (parts & CAD_BWD_DQ) {
      dq::Params p;
      make_tile_map(&p.tm_q, q, sh.q_rows, sh.h_q);
      make_tile_map(&p.tm_do, dout, sh.q_rows, sh.h_q);
      make_tile_map(&p.tm_k, k, sh.kv_rows, sh.h_kv);
      make_tile_map(&p.tm_v, v, sh.kv_rows, sh.h_kv);
      p.tasks = plan->d_tasks;
      p.units = plan->d_dq;
      p.n_units = static_cast<int>(plan->dq_units.size());
      p.sched = plan->sched_dq.d;
      p.group = sh.h_q / sh.h_kv;
      p.h_q = sh.h_q;
      p.lse2 = lse2;
      p.delta = delta;
      p.dq = static_cast<__nv_bfloat16*>(dq);
      p.pitch = pitch;
      p.scale = sh.softmax_scale;
      p.scale_log2 = sh.softmax_scale * kLog2e;
      const int grid = plan->sched_dq.G;
      dq::ca_bwd_dq_kernel<<<grid, kThreads, dq::kSmemBytes, s_dq>>>(p);
      cuda_check(cudaGetLastError(), "ca_bwd_dq launch");
      if (debug_sync) cuda_check(cudaStreamSynchronize(s_dq), "ca_bwd_dq");
    }
    if (fork) {
      cuda_check(cudaEventRecord(plan->ev_join, plan->side), "event(join)");
      cuda_check(cudaStreamWaitEvent(s, plan->ev_join, 0), "wait(join)");
    }
  });
}

extern "C" int cad_ca_bwd(const cad_ca_plan* plan, const void* q, const void* k, const void* v,
                          const void* o, const float* lse, const void* dout, void* dq, void* dk,
                          void* dv, void* workspace, size_t ws_bytes, void* stream) {
  return cad_ca_bwd_parts(plan, q, k, v, o, lse, dout, dq, dk, dv, workspace, ws_bytes,
                          CAD_BWD_ALL, stream);
}
