// cad_ca_plan: the device work list of one CA task set (one server, one
// nano-batch half), built once on the host and reused by every layer's
// forward and backward launch.
//
// Work decomposition. Forward: one unit per (task, 128-row q tile, KV head,
// pair of query heads of that KV head's GQA group); it walks the causal kv
// tiles 0..n_kv-1 (tiles entirely above the diagonal are never visited).
// Backward: one unit per (task, 128-row kv tile, KV head, pair of query
// heads); it walks q tiles from the first one that can see the kv tile.
// Units are sorted by KV head, then by length, longest first, and dealt to
// the persistent CTAs greedily (each unit to the CTA with the least work so
// far, LPT): concurrently running CTAs stay on the same KV head, sharing
// L2-resident tiles, and every CTA ends within about one short unit of the
// others.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <mutex>
#include <type_traits>
#include <numeric>
#include <cstdio>
#include <cstdlib>
#include <queue>
#include <set>
#include <string>

#include "../host/cad_status.hpp"
#include "ca_common.cuh"

namespace cad_dev {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw cad::CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void set_max_smem(const void* kernel, int bytes, const char* what) {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  const std::pair<const void*, int> key{kernel, dev};
  {
    std::lock_guard<std::mutex> g(mu);
    if (done.count(key)) return;
  }
  // idempotent, so a race between two threads only sets it twice
  cuda_check(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes), what);
  std::lock_guard<std::mutex> g(mu);
  done.insert(key);
}

void preload_kernels() {
  int dev = 0;
  cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  static std::mutex mu;
  static std::set<int> done;
  std::lock_guard<std::mutex> g(mu);
  if (done.count(dev)) return;
  preload_fwd();
  preload_fwd2();
  preload_bwd();
  preload_dkdv2();
  preload_dkdvq2();
  preload_dq2();
  preload_comm();
  // the runtime's own memset / device-to-device copy kernels (the executor's
  // cudaMemsetAsync, cudaMemcpyAsync and cudaMemcpy2DAsync)
  char* p = nullptr;
  cuda_check(cudaMalloc(reinterpret_cast<void**>(&p), 4096), "cudaMalloc");
  cuda_check(cudaMemsetAsync(p, 0, 4096, nullptr), "memset");
  cuda_check(cudaMemcpyAsync(p + 2048, p, 1024, cudaMemcpyDeviceToDevice, nullptr), "memcpy");
  cuda_check(cudaMemcpy2DAsync(p + 2048, 64, p, 128, 4, 8, cudaMemcpyDeviceToDevice, nullptr), "memcpy2d");
  cuda_check(cudaStreamSynchronize(nullptr), "sync");
  cudaFree(p);
  done.insert(dev);
}

DeviceGuard::DeviceGuard(int device) : want(device) {
  cuda_check(cudaGetDevice(&prev), "cudaGetDevice");
  if (prev != want) cuda_check(cudaSetDevice(want), "cudaSetDevice");
}

DeviceGuard::~DeviceGuard() {
  if (prev >= 0 && prev != want) cudaSetDevice(prev);
}

namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) throw cad::CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

}  // namespace

void make_tile_map(CUtensorMap* map, const void* base, int64_t rows, int heads, int box_rows) {
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kHeadDim), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(heads)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(heads) * kHeadDim * 2,
                                 static_cast<cuuint64_t>(kHeadDim) * 2};
  const cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cad::CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
}

void make_acc_map(CUtensorMap* map, void* base, int64_t rows, int heads) {
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kHeadDim), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(heads)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(heads) * kHeadDim * 4,
                                 static_cast<cuuint64_t>(kHeadDim) * 4};
  const cuuint32_t box[3] = {32, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cad::CudaError("cuTensorMapEncodeTiled(acc) failed: " + std::to_string(int(r)));
}

void make_row_map(CUtensorMap* map, const void* base, int64_t rows, int heads) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(heads)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(rows) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kTile), 1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base),
                                 dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw cad::CudaError("cuTensorMapEncodeTiled(rows) failed: " + std::to_string(int(r)));
}

static void build_units(cad_ca_plan& P) {
  const int hq = P.shape.h_q, hkv = P.shape.h_kv, group = hq / hkv;
  const int per_unit = (group % 2 == 0) ? 2 : 1;  // query heads sharing one KV tile stream
  const int n_tasks = static_cast<int>(P.tasks.size());
  for (int32_t t = 0; t < n_tasks; ++t) {
    const DevTask& tk = P.tasks[t];
    const int shift = tk.kv_len - tk.n_q;
    const int n_qt = (tk.n_q + kTile - 1) / kTile;
    for (int i = 0; i < n_qt; ++i) {
      const int last_pos = shift + std::min(tk.n_q, (i + 1) * kTile) - 1;
      const int n_kv = last_pos / kTile + 1;
      for (int hk = 0; hk < hkv; ++hk) {
        for (int g = 0; g < group; g += per_unit)
          P.fwd_units.push_back({t, i, static_cast<int16_t>(hk * group + g), static_cast<int16_t>(per_unit), n_kv});
        for (int g = 0; g < group; ++g)
          P.dq_units.push_back({t, i, static_cast<int16_t>(hk * group + g), 1, n_kv});
        if (group % 2 == 0)
          for (int g = 0; g < group; g += 2)
            P.dq2_units.push_back({t, i, static_cast<int16_t>(hk * group + g), 2, n_kv});
        if (group % 4 == 0)
          for (int g = 0; g < group; g += 4)
            P.fwd2_units.push_back({t, i, static_cast<int16_t>(hk * group + g), 4, n_kv});
      }
    }
  }
  // KV groups: tasks sharing kv_off. Groups must own disjoint KV rows and
  // tasks disjoint Q rows, otherwise the backward's plain (non-atomic)
  // stores would race.
  std::vector<int> order(n_tasks);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return P.tasks[a].kv_off < P.tasks[b].kv_off; });
  std::vector<std::pair<int, int>> qspans;
  for (const DevTask& t : P.tasks) qspans.push_back({t.q_off, t.q_off + t.n_q});
  std::sort(qspans.begin(), qspans.end());
  for (size_t i = 1; i < qspans.size(); ++i)
    if (qspans[i].first < qspans[i - 1].second) throw cad::DomainError("CA tasks overlap in Q rows");
  int prev_end = -1;
  for (size_t a = 0; a < order.size();) {
    size_t b = a;
    int kv_off = P.tasks[order[a]].kv_off, kv_end = kv_off;
    while (b < order.size() && P.tasks[order[b]].kv_off == kv_off) {
      kv_end = std::max(kv_end, P.tasks[order[b]].kv_off + P.tasks[order[b]].kv_len);
      ++b;
    }
    if (kv_off < prev_end) throw cad::DomainError("CA task KV ranges overlap without sharing kv_off");
    prev_end = kv_end;
    const int n_kt = (kv_end - kv_off + kTile - 1) / kTile;
    for (int j = 0; j < n_kt; ++j) {
      const int32_t seg_begin = static_cast<int32_t>(P.kv_segs.size());
      int32_t len = 0;
      for (size_t x = a; x < b; ++x) {
        const DevTask& tk = P.tasks[order[x]];
        const int shift = tk.kv_len - tk.n_q;
        const int q_first = std::max(0, j * kTile - shift);  // first query that sees key j*128
        if (q_first >= tk.n_q) continue;
        const int n_qs = (tk.n_q + kSub - 1) / kSub;
        P.kv_segs.push_back({order[x], q_first / kSub, n_qs});
        len += n_qs - q_first / kSub;
      }
      const int32_t seg_end = static_cast<int32_t>(P.kv_segs.size());
      if (len == 0) continue;
      for (int hk = 0; hk < hkv; ++hk)
        P.kv_units.push_back({kv_off, kv_end, j, static_cast<int16_t>(hk), 0, seg_begin, seg_end, len * group});
    }
    a = b;
  }
  // Head-major, then longest first: the ~148 concurrently running CTAs work
  // on the same KV head, so the K/V (fwd, dq) or Q/dO (dkdv) tiles they all
  // stream stay L2-resident; within a head the strided walk is LPT.
  std::stable_sort(P.fwd_units.begin(), P.fwd_units.end(), [group](const FwdUnit& a, const FwdUnit& b) {
    const int ha = a.head0 / group, hb = b.head0 / group;
    return ha != hb ? ha < hb : a.n_kv > b.n_kv;
  });
  std::stable_sort(P.fwd2_units.begin(), P.fwd2_units.end(), [group](const FwdUnit& a, const FwdUnit& b) {
    const int ha = a.head0 / group, hb = b.head0 / group;
    return ha != hb ? ha < hb : a.n_kv > b.n_kv;
  });
  std::stable_sort(P.dq_units.begin(), P.dq_units.end(), [group](const FwdUnit& a, const FwdUnit& b) {
    const int ha = a.head0 / group, hb = b.head0 / group;
    return ha != hb ? ha < hb : a.n_kv > b.n_kv;
  });
  std::stable_sort(P.dq2_units.begin(), P.dq2_units.end(), [group](const FwdUnit& a, const FwdUnit& b) {
    const int ha = a.head0 / group, hb = b.head0 / group;
    return ha != hb ? ha < hb : a.n_kv > b.n_kv;
  });
  // CTA-pair dK/dV: the even kv tiles of every group; the pair's second tile
  // (tile + 1, possibly past kv_end) is seen by a subset of the first one's
  // q tiles, so the first tile's segments and length cover both.
  for (const KvUnit& u : P.kv_units)
    if (u.tile % 2 == 0) P.kv2_units.push_back(u);
  std::stable_sort(P.kv_units.begin(), P.kv_units.end(), [](const KvUnit& a, const KvUnit& b) {
    return a.hk != b.hk ? a.hk < b.hk : a.n_iter > b.n_iter;
  });
  std::stable_sort(P.kv2_units.begin(), P.kv2_units.end(), [](const KvUnit& a, const KvUnit& b) {
    return a.hk != b.hk ? a.hk < b.hk : a.n_iter > b.n_iter;
  });
}

// Greedy LPT deal of units (in their sorted order) over G CTAs.
static void deal(CtaLists& L, const std::vector<int64_t>& cost, int G) {
  G = std::max(1, G);
  std::vector<std::vector<int32_t>> per(G);
  using Slot = std::pair<int64_t, int>;  // (load, cta): ties go to the lower CTA
  std::priority_queue<Slot, std::vector<Slot>, std::greater<Slot>> heap;
  for (int c = 0; c < G; ++c) heap.push({0, c});
  for (size_t u = 0; u < cost.size(); ++u) {
    Slot s = heap.top();
    heap.pop();
    per[s.second].push_back(static_cast<int32_t>(u));
    s.first += cost[u];
    heap.push(s);
  }
  if (std::getenv("CAD_SCHED_STATS")) {
    std::vector<int64_t> load(G, 0);
    int64_t tot = 0, mx = 0;
    for (int c = 0; c < G; ++c) {
      for (int32_t u : per[c]) load[c] += cost[u];
      tot += load[c];
      mx = std::max(mx, load[c]);
    }
    const int64_t umax = cost.empty() ? 0 : *std::max_element(cost.begin(), cost.end());
    std::fprintf(stderr, "sched: %zu units over %d lists: max/mean load %.4f, largest unit %.4f of mean\n",
                 cost.size(), G, tot ? double(mx) * G / double(tot) : 0.0, tot ? double(umax) * G / double(tot) : 0.0);
  }
  L.G = G;
  L.host.assign(1, 0);
  for (int c = 0; c < G; ++c) L.host.push_back(L.host.back() + static_cast<int32_t>(per[c].size()));
  for (int c = 0; c < G; ++c) L.host.insert(L.host.end(), per[c].begin(), per[c].end());
  cudaFree(L.d);
  L.d = nullptr;
  cuda_check(cudaMalloc(reinterpret_cast<void**>(&L.d), L.host.size() * sizeof(int32_t)), "cudaMalloc(sched)");
  cuda_check(cudaMemcpy(L.d, L.host.data(), L.host.size() * sizeof(int32_t), cudaMemcpyHostToDevice),
             "cudaMemcpy(sched)");
}

// Per-unit cost in tile iterations, plus the unit's fixed prologue/epilogue.
static void build_schedules(cad_ca_plan& P) {
  std::vector<int64_t> c;
  // fixed per-unit cost in tile iterations (fill/drain, epilogue);
  // CAD_SCHED_FIXED / CAD_SCHED_KV_FIXED override for experiments
  static const int64_t fixed_q = std::getenv("CAD_SCHED_FIXED") ? std::atoll(std::getenv("CAD_SCHED_FIXED")) : 1;
  static const int64_t fixed_kv = std::getenv("CAD_SCHED_KV_FIXED") ? std::atoll(std::getenv("CAD_SCHED_KV_FIXED")) : -1;
  auto fwd_cost = [&](const std::vector<FwdUnit>& v) {
    c.clear();
    for (const FwdUnit& u : v) c.push_back(int64_t(u.n_kv) + fixed_q);
    return c;
  };
  deal(P.sched_fwd, fwd_cost(P.fwd_units), P.grid(P.fwd_units.size()));
  // CTA pairs: half the grid, one list per pair
  deal(P.sched_fwd2, fwd_cost(P.fwd2_units),
       std::max<int>(1, std::min<int64_t>(P.fwd2_units.size(), P.grid(1 << 30) / 2)));
  deal(P.sched_dq, fwd_cost(P.dq_units), P.grid(P.dq_units.size()));
  deal(P.sched_dq2, fwd_cost(P.dq2_units),
       std::max<int>(1, std::min<int64_t>(P.dq2_units.size(), P.grid(1 << 30) / 2)));
  c.clear();
  const int group = P.shape.h_q / P.shape.h_kv;
  const int64_t kv_fixed = fixed_kv >= 0 ? fixed_kv : 2 * group;
  for (const KvUnit& u : P.kv_units) c.push_back(int64_t(u.n_iter) + kv_fixed);
  deal(P.sched_kv, c, P.grid(P.kv_units.size()));
  c.clear();
  for (const KvUnit& u : P.kv2_units) c.push_back(int64_t(u.n_iter) + kv_fixed);
  deal(P.sched_kv2, c, std::max<int>(1, std::min<int64_t>(P.kv2_units.size(), P.grid(1 << 30) / 2)));
}

}  // namespace cad_dev

using cad_dev::cuda_check;

extern "C" {

int cad_ca_plan_create(const cad_ca_task* tasks, int64_t n_tasks, const cad_ca_shape* shape,
                       cad_ca_plan** plan) {
  return cad::guarded([&] {
    if (!shape || !plan || (n_tasks > 0 && !tasks) || n_tasks < 0) throw cad::DomainError("null argument");
    *plan = nullptr;
    if (shape->head_dim != cad_dev::kHeadDim) throw cad::ConfigError("head_dim must be 128");
    if (shape->h_q < 1 || shape->h_kv < 1 || shape->h_q % shape->h_kv != 0)
      throw cad::ConfigError("h_q must be a positive multiple of h_kv");
    if (shape->q_rows < 0 || shape->kv_rows < 0 || shape->q_rows >= (int64_t(1) << 31) ||
        shape->kv_rows >= (int64_t(1) << 31))
      throw cad::ConfigError("row counts out of range");
    auto P = std::make_unique<cad_ca_plan>();
    P->shape = *shape;
    if (!(P->shape.softmax_scale > 0)) P->shape.softmax_scale = 1.0f / std::sqrt(float(shape->head_dim));
    for (int64_t i = 0; i < n_tasks; ++i) {
      const cad_ca_task& t = tasks[i];
      if (t.n_q < 1 || t.kv_len < t.n_q) throw cad::DomainError("CA task needs kv_len >= n_q >= 1");
      if (t.q_off < 0 || t.q_off + t.n_q > shape->q_rows || t.kv_off < 0 ||
          t.kv_off + t.kv_len > shape->kv_rows)
        throw cad::DomainError("CA task rows outside the buffers");
      P->tasks.push_back({static_cast<int32_t>(t.q_off), static_cast<int32_t>(t.n_q),
                          static_cast<int32_t>(t.kv_off), static_cast<int32_t>(t.kv_len)});
      P->pairs += cad_causal_pairs(t.n_q, t.kv_len);
    }
    cad_dev::build_units(*P);
    cuda_check(cudaGetDevice(&P->device), "cudaGetDevice");
    cad_dev::preload_kernels();
    cuda_check(cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, P->device),
               "cudaDeviceGetAttribute");
    auto upload = [](auto& vec, auto** dst) {
      using T = typename std::decay_t<decltype(vec)>::value_type;
      const size_t bytes = std::max<size_t>(1, vec.size()) * sizeof(T);
      cuda_check(cudaMalloc(reinterpret_cast<void**>(dst), bytes), "cudaMalloc(plan)");
      if (!vec.empty())
        cuda_check(cudaMemcpy(*dst, vec.data(), vec.size() * sizeof(T), cudaMemcpyHostToDevice),
                   "cudaMemcpy(plan)");
    };
    for (const cad_dev::DevTask& t : P->tasks)
      for (int r = 0; r < t.n_q; r += 32) P->row_chunks.push_back(make_int2(t.q_off + r, std::min(32, t.n_q - r)));
    upload(P->tasks, &P->d_tasks);
    upload(P->row_chunks, &P->d_row_chunks);
    upload(P->fwd_units, &P->d_fwd);
    upload(P->dq_units, &P->d_dq);
    upload(P->fwd2_units, &P->d_fwd2);
    upload(P->dq2_units, &P->d_dq2);
    upload(P->kv_units, &P->d_kv);
    upload(P->kv2_units, &P->d_kv2);
    upload(P->kv_segs, &P->d_segs);
    cad_dev::build_schedules(*P);
    cuda_check(cudaStreamCreateWithFlags(&P->side, cudaStreamNonBlocking), "cudaStreamCreate(side)");
    cuda_check(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming), "cudaEventCreate");
    *plan = P.release();
  });
}

int cad_ca_plan_info_get(const cad_ca_plan* plan, cad_ca_plan_info* info) {
  return cad::guarded([&] {
    if (!plan || !info) throw cad::DomainError("null argument");
    info->n_fwd_units = static_cast<int64_t>(plan->fwd_units.size());
    info->n_bwd_units = static_cast<int64_t>(plan->kv_units.size() + plan->dq_units.size());
    info->causal_pairs = plan->pairs;
    const double base = double(plan->shape.head_dim) * double(plan->shape.h_q) * double(plan->pairs);
    info->fwd_flops = 4.0 * base;
    info->bwd_flops = 10.0 * base;
    // D = rowsum(dO * O) and log2-domain LSE per (head, row), fp32, rows
    // padded to a multiple of 4 (16-byte TMA pitch)
    // (+ the experimental fused backward's fp32 dQ accumulator, [rows][h_q]
    // [128], when CAD_BWD_FUSED=1 selects it; see ca_dkdvq2.cu)
    info->workspace_bytes = size_t(2) * ((plan->shape.q_rows + 3) / 4 * 4) * plan->shape.h_q * 4 +
                            (cad_dev::fused_bwd_enabled() ? cad_dev::dq_acc_bytes(plan->shape) : 0);
  });
}

int cad_ca_plan_set_max_ctas(cad_ca_plan* plan, int max_ctas) {
  return cad::guarded([&] {
    if (!plan || max_ctas < 0) throw cad::DomainError("bad argument");
    cad_dev::DeviceGuard dg(plan->device);
    plan->max_ctas = max_ctas;
    cad_dev::build_schedules(*plan);
  });
}

int cad_ca_plan_destroy(cad_ca_plan* plan) {
  return cad::guarded([&] {
    if (!plan) return;
    cad_dev::DeviceGuard dg(plan->device);
    cudaFree(plan->d_tasks);
    cudaFree(plan->d_row_chunks);
    cudaFree(plan->d_fwd);
    cudaFree(plan->d_dq);
    cudaFree(plan->d_fwd2);
    cudaFree(plan->d_dq2);
    cudaFree(plan->d_kv);
    cudaFree(plan->d_kv2);
    cudaFree(plan->d_segs);
    for (cad_dev::CtaLists* L : {&plan->sched_fwd, &plan->sched_fwd2, &plan->sched_dq, &plan->sched_dq2,
                                 &plan->sched_kv, &plan->sched_kv2})
      cudaFree(L->d);
    if (plan->side) cudaStreamDestroy(plan->side);
    if (plan->ev_fork) cudaEventDestroy(plan->ev_fork);
    if (plan->ev_join) cudaEventDestroy(plan->ev_join);
    delete plan;
  });
}

}  // extern "C"
