// Shared definitions of the CA kernels: device task/work-unit records, the
// plan object behind cad_ca_plan, and TMA tensor-map construction.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../../include/cad.h"

namespace cad_dev {

constexpr int kTile = 128;    // q rows and kv rows per tile
constexpr int kHeadDim = 128; // d
constexpr uint32_t kTileBytes = kTile * kHeadDim * 2;  // one bf16 128x128 tile

// One CA task on the device (row offsets into the packed THD buffers).
struct DevTask {
  int32_t q_off, n_q, kv_off, kv_len;
};

// Forward work unit: `nh` query heads starting at head0 (same KV head) on
// q tile `tile` of task `task`; it walks kv tiles 0..n_kv-1.
struct FwdUnit {
  int32_t task, tile;
  int16_t head0, nh;
  int32_t n_kv;
};

constexpr int kSub = 128;  // q rows per dK/dV iteration

// dK/dV work unit: kv tile `tile` of a KV group (the tasks sharing one KV
// row range [kv_off, kv_end), e.g. the shards of one document on this
// server) for KV head hk. It walks, for every query head of hk's GQA group,
// the segments seg_begin..seg_end-1: (task, 64-row q sub-tiles
// qt_lo..qt_hi-1) that can see the tile. One unit owns its dK/dV rows, so no reduction across
// units is needed.
struct KvUnit {
  int32_t kv_off, kv_end, tile;
  int16_t hk, pad;
  int32_t seg_begin, seg_end;
  int32_t n_iter;  // group * sum of segment lengths
};
struct KvSeg {
  int32_t task, qt_lo, qt_hi;
};

// Static per-CTA work lists: CTA (or CTA pair) c runs units
// list[off[c] .. off[c+1]) in order. Stored on the device as one array:
// off[0..G] followed by list.
struct CtaLists {
  int G = 0;
  std::vector<int32_t> host;  // off (G + 1) then list
  int32_t* d = nullptr;
};

__device__ __forceinline__ int32_t sched_begin(const int32_t* sc, int c) { return sc[c]; }
__device__ __forceinline__ int32_t sched_end(const int32_t* sc, int c) { return sc[c + 1]; }
__device__ __forceinline__ int32_t sched_unit(const int32_t* sc, int G, int32_t i) { return sc[G + 1 + i]; }

}  // namespace cad_dev

struct cad_ca_plan {
  cad_ca_shape shape{};
  std::vector<cad_dev::DevTask> tasks;
  std::vector<cad_dev::FwdUnit> fwd_units;
  std::vector<cad_dev::FwdUnit> dq_units;  // nh == 1
  std::vector<cad_dev::FwdUnit> fwd2_units;  // CTA-pair forward: nh == 4 (GQA group % 4 == 0)
  std::vector<cad_dev::FwdUnit> dq2_units;   // CTA-pair dQ: nh == 2 (even GQA group)
  std::vector<cad_dev::KvUnit> kv_units;
  std::vector<cad_dev::KvUnit> kv2_units;  // CTA-pair dK/dV: kv tiles (tile, tile + 1)
  std::vector<cad_dev::KvSeg> kv_segs;
  std::vector<int2> row_chunks;  // (first row, rows <= 32) covering every task's query rows
  cad_dev::DevTask* d_tasks = nullptr;
  int2* d_row_chunks = nullptr;
  cad_dev::FwdUnit* d_fwd = nullptr;
  cad_dev::FwdUnit* d_dq = nullptr;
  cad_dev::FwdUnit* d_fwd2 = nullptr;
  cad_dev::FwdUnit* d_dq2 = nullptr;
  cad_dev::KvUnit* d_kv = nullptr;
  cad_dev::KvUnit* d_kv2 = nullptr;
  cad_dev::KvSeg* d_segs = nullptr;
  int64_t pairs = 0;
  int device = 0;
  int num_sms = 148;
  int max_ctas = 0;  // 0: one persistent CTA per SM
  int grid(int64_t units) const {
    const int cap = max_ctas > 0 ? std::min(max_ctas, num_sms) : num_sms;
    return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(units, cap)));
  }
  // LPT work lists per kernel for the current grid (rebuilt by set_max_ctas)
  cad_dev::CtaLists sched_fwd, sched_fwd2, sched_dq, sched_dq2, sched_kv, sched_kv2;
  // backward fork/join: dQ runs on a side stream next to dK/dV, so dQ's CTAs
  // take the SMs dK/dV's retire from (its LPT tail) instead of waiting for the
  // last dK/dV CTA
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};

namespace cad_dev {

// 3-D tiled map over a packed [rows][heads][128] bf16 buffer: box of
// 64 d-values x 128 rows x 1 head, 128-byte swizzle. A 128x128 tile is two
// boxes (d 0-63 and 64-127), landing as two 16 KB K-major SW128 planes.
void make_tile_map(CUtensorMap* map, const void* base, int64_t rows, int heads, int box_rows = kTile);
// 3-D map over a packed [rows][heads][128] fp32 buffer (the fused backward's
// dQ accumulator): box of 32 d-values x 32 rows x 1 head, 128-byte swizzle.
void make_acc_map(CUtensorMap* map, void* base, int64_t rows, int heads);
// Bytes of that accumulator (256-byte aligned).
size_t dq_acc_bytes(const cad_ca_shape& sh);
// CAD_BWD_FUSED=1: the experimental fused dK/dV/dQ backward (ca_dkdvq2.cu)
// instead of the two-pass one (slower today).
bool fused_bwd_enabled();
// 2-D map over a [heads][rows] fp32 buffer (LSE, D): box of 128 rows x 1 head.
void make_row_map(CUtensorMap* map, const void* base, int64_t rows, int heads);
void cuda_check(cudaError_t e, const char* what);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute belongs to the current device's context, so a process that
// drives several GPUs through the C-ABI needs it on each of them. Thread-safe.
void set_max_smem(const void* kernel, int bytes, const char* what);
// Loads every kernel of the library on the current device (once per device):
// with CUDA's lazy module loading the first launch of a kernel loads its
// module, which can block the host until the device is idle -- a deadlock
// when the device waits on work this host thread has yet to enqueue (several
// ranks' contexts driven from one thread). Called at plan/context creation.
void preload_kernels();
void preload_fwd();
void preload_fwd2();
void preload_bwd();
void preload_dkdv2();
void preload_dkdvq2();
void preload_dq2();
void preload_comm();
// Makes the plan's device current for the duration of a launch (and restores
// the caller's device), so one host thread may drive plans on several GPUs.
struct DeviceGuard {
  int prev = -1, want = -1;
  explicit DeviceGuard(int device);
  ~DeviceGuard();
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};
bool launch_fwd_pair(const cad_ca_plan* plan, const void* q, const void* k, const void* v, void* o, float* lse,
                     cudaStream_t stream);
bool launch_dkdv_pair(const cad_ca_plan* plan, const void* q, const void* k, const void* v, const void* dout,
                      const float* nlse2, const float* ndelta, int64_t pitch, void* dk, void* dv,
                      cudaStream_t stream);
bool launch_dkdvq_pair(const cad_ca_plan* plan, const void* q, const void* k, const void* v, const void* dout,
                       const float* nlse2, const float* ndelta, int64_t pitch, void* dk, void* dv, float* acc,
                       cudaStream_t stream);
void launch_dq_convert(const cad_ca_plan* plan, const float* acc, void* dq, cudaStream_t stream);
bool launch_dq_pair(const cad_ca_plan* plan, const void* q, const void* k, const void* v, const void* dout,
                    const float* lse2, const float* delta, int64_t pitch, void* dq, cudaStream_t stream);

}  // namespace cad_dev
