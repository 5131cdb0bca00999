// The per-layer executor behind cad_layer_ctx: "run this device's layer --
// dispatch, CA, return". The reference only models this step
// (simulate_layer_pingpong over the four windows of layer_windows,
// P/src/sim.cpp:69-125,176-221; per-device served/sent lists and halves,
// P/src/sim.cpp:34-46,129-157). Here it moves real rows and runs the sm_100a
// CA kernels.
//
// Per layer and half h of rank r (row lists from cad_layer_plan, built for
// every rank so each rank knows where its rows land in the peers' buffers):
//   dispatch QKV   Q rows home -> server, K/V rows owner -> server
//   compute fwd    cad_ca_fwd on the half's server buffers
//   return O       O rows + LSE columns server -> home
//   dispatch DO    dO rows home -> server
//   compute bwd    cad_ca_bwd (Q/K/V/O/LSE resident from the forward)
//   return GRAD    dQ rows server -> home, dK/dV partial rows server ->
//                  the owner's staging; finish sums the partials (fp32)
//
// Transports:
//   LOCAL/IPC  every rank PUSHES its rows straight into the peers' buffers
//              (cudaMemcpyAsync runs through CUDA IPC mappings: copy
//              engines, no SM taken from the persistent CA kernels) and
//              signals arrival with cuStreamWriteValue32 on the peer's flag
//              word; consumers wait with cuStreamWaitValue32. Nothing
//              synchronises on the host. LOCAL is the same code with every
//              rank's context in one process (raw pointers instead of IPC
//              mappings), which lets one GPU run a world-W layer.
//   NCCL       gather -> grouped ncclSend/ncclRecv -> scatter, on the stream
//              the transport call is given.
// Flag words (uint32, monotonically increasing within a context): slot
// (kind, half, source rank); the values of one step with L layers starting at
// g0: forward of layer l -> g0+1+l, backward of layer l -> g0+2L-l, done ->
// g0+2L, so every wait is ">= value" and a later signal never under-shoots.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "../host/cad_status.hpp"
#include "ca_common.cuh"

namespace {

using i64 = int64_t;
using cad_dev::cuda_check;

constexpr int kXQ = CAD_XFER_Q, kXKV = CAD_XFER_KV, kXO = CAD_XFER_O_RET, kXKR = CAD_XFER_KV_RET;
enum FlagKind { F_QKV = 0, F_DO = 1, F_O = 2, F_G = 3, F_DONE = 4, kKinds = 5 };
constexpr uint32_t kBlobMagic = 0xCAD1A7E5u;

// CAD_TRACE_HOST=1: every transport/compute call of a context logged on
// stderr before it is issued (host-side debugging of enqueue order)
bool trace_host() {
  static const bool on = std::getenv("CAD_TRACE_HOST") != nullptr;
  return on;
}

void ok(int rc, const char* what) {
  if (trace_host()) std::fprintf(stderr, "[cad] issued %s rc=%d\n", what, rc);
  if (rc == CAD_OK) return;
  const std::string msg = std::string(what) + ": " + cad_last_error();
  switch (rc) {
    case CAD_ERR_CONFIG: throw cad::ConfigError(msg);
    case CAD_ERR_DOMAIN: throw cad::DomainError(msg);
    case CAD_ERR_NCCL: throw cad::NcclError(msg);
    case CAD_ERR_CAPACITY: throw cad::CapacityError(msg);
    default: throw cad::CudaError(msg);
  }
}

struct XferRows {
  std::vector<i64> send_counts, send_idx, recv_counts, recv_idx;
  i64 n_send() const { return send_idx.size(); }
  i64 n_recv() const { return recv_idx.size(); }
};

struct HalfRows {
  i64 q_rows = 0, kv_rows = 0;
  std::vector<cad_ca_task> tasks;
  XferRows x[4];
  i64 wire[4] = {0, 0, 0, 0};
};

struct RankRows {
  i64 home_rows = 0;
  HalfRows half[2];
};

RankRows read_rank(const cad_plan* plan, const cad_item* items, i64 n, int32_t rank, i64 q_row, i64 kv_row,
                   int32_t balance) {
  cad_layer_plan* lp = nullptr;
  ok(cad_layer_plan_create_ex(plan, items, n, rank, q_row, kv_row, balance, &lp), "cad_layer_plan_create_ex");
  std::unique_ptr<cad_layer_plan, void (*)(cad_layer_plan*)> guard(lp, cad_layer_plan_destroy);
  RankRows R;
  for (int h = 0; h < 2; ++h) {
    cad_layer_half_info info;
    ok(cad_layer_plan_info(lp, h, &info), "cad_layer_plan_info");
    R.home_rows = info.home_rows;
    HalfRows& H = R.half[h];
    H.q_rows = info.q_rows;
    H.kv_rows = info.kv_rows;
    H.tasks.assign(info.tasks, info.tasks + info.n_tasks);
    for (int w = 0; w < 4; ++w) {
      cad_xfer x;
      ok(cad_layer_plan_xfer(lp, h, w, &x), "cad_layer_plan_xfer");
      XferRows& X = H.x[w];
      X.send_counts.assign(x.send_counts, x.send_counts + x.n_peers);
      X.recv_counts.assign(x.recv_counts, x.recv_counts + x.n_peers);
      X.send_idx.assign(x.send_idx, x.send_idx + x.n_send);
      X.recv_idx.assign(x.recv_idx, x.recv_idx + x.n_recv);
      H.wire[w] = info.remote_send_bytes[w];
    }
  }
  return R;
}

// Zero-copy own rows. A rank's home buffers live INSIDE its server buffers:
// every Q-like buffer of a layer (Q, O, dO, dQ) is [R0 | HOME | R1] rows --
// HOME = the rank's home rows, R0 / R1 = the rows of the tasks it serves for
// other ranks in the ping / pong half -- and half 0's view starts at row 0,
// half 1's at row R0, so both halves see HOME contiguously next to their
// remote rows. Every task of a rank's own rows then reads Q/dO and writes
// O/dQ in place; a KV group whose prefix [0, need) is entirely home rows in
// order (a document that starts on this rank) reads K/V in place from the
// [KR0 | HOME | KR1] K/V buffers. Only KV groups assembled from several
// ranks and the LSE re-layout still copy own rows. alias_rows rewrites a
// rank's row plan into these view coordinates (every rank does it for every
// rank, so pushes land where the peer's kernels read).
struct Alias {
  i64 home = 0, r[2] = {0, 0}, kr[2] = {0, 0};
  // own rows that still move: (src, dst) pairs per half
  std::vector<std::pair<i64, i64>> lse_self[2];  // O_RET LSE: view q row -> home row
  std::vector<std::pair<i64, i64>> qd_self[2];   // QD: home row -> view q row (forward-state LSE)
};

Alias alias_rows(RankRows& R, int me) {
  Alias A;
  A.home = R.home_rows;
  for (int h = 0; h < 2; ++h) {
    HalfRows& H = R.half[h];
    auto self_block = [&](const std::vector<i64>& counts) {
      i64 o = 0;
      for (int p = 0; p < me; ++p) o += counts[static_cast<size_t>(p)];
      return std::make_pair(o, counts[static_cast<size_t>(me)]);
    };
    // ---- Q rows: own (from the QD self pairs) -> HOME, the rest -> remote region
    XferRows& QD = H.x[kXQ];
    const auto qs = self_block(QD.send_counts), qr = self_block(QD.recv_counts);
    std::vector<i64> own_q(static_cast<size_t>(std::max<i64>(0, H.q_rows)), -1);
    for (i64 j = 0; j < qs.second; ++j)
      own_q[static_cast<size_t>(QD.recv_idx[static_cast<size_t>(qr.first + j)])] =
          QD.send_idx[static_cast<size_t>(qs.first + j)];
    std::vector<i64> qmap(own_q.size());
    i64 nrem = 0;
    for (size_t row = 0; row < own_q.size(); ++row)
      if (own_q[row] < 0) qmap[row] = nrem++;
    A.r[h] = nrem;
    // view rows: half 0 [R0 | HOME], half 1 [HOME | R1]
    for (size_t row = 0; row < own_q.size(); ++row)
      qmap[row] = own_q[row] >= 0 ? (h == 0 ? nrem : 0) + own_q[row] : (h == 0 ? 0 : A.home) + qmap[row];
    // ---- KV groups: aliased iff all of [kv_off, kv_off + need) are own rows, in home order
    XferRows& KD = H.x[kXKV];
    const auto ks = self_block(KD.send_counts), kr = self_block(KD.recv_counts);
    std::vector<i64> own_kv(static_cast<size_t>(std::max<i64>(0, H.kv_rows)), -1);
    for (i64 j = 0; j < ks.second; ++j)
      own_kv[static_cast<size_t>(KD.recv_idx[static_cast<size_t>(kr.first + j)])] =
          KD.send_idx[static_cast<size_t>(ks.first + j)];
    std::map<i64, i64> need;  // kv_off -> rows of the group
    for (const cad_ca_task& t : H.tasks) need[t.kv_off] = std::max(need[t.kv_off], t.kv_len);
    std::vector<i64> kvmap(own_kv.size(), -1);
    std::vector<char> aliased(own_kv.size(), 0);
    i64 nkr = 0;
    for (const auto& g : need) {
      bool ok_alias = true;
      for (i64 j = 0; j < g.second && ok_alias; ++j)
        ok_alias = own_kv[static_cast<size_t>(g.first + j)] == own_kv[static_cast<size_t>(g.first)] + j &&
                   own_kv[static_cast<size_t>(g.first)] >= 0;
      for (i64 j = 0; j < g.second; ++j) {
        const size_t row = static_cast<size_t>(g.first + j);
        aliased[row] = ok_alias;
        kvmap[row] = ok_alias ? own_kv[row] : nkr + j;  // home row / remote index
      }
      if (!ok_alias) nkr += g.second;
    }
    A.kr[h] = nkr;
    for (size_t row = 0; row < kvmap.size(); ++row)
      if (kvmap[row] >= 0)
        kvmap[row] = aliased[row] ? (h == 0 ? nkr : 0) + kvmap[row] : (h == 0 ? 0 : A.home) + kvmap[row];
    // ---- tasks in view coordinates
    for (cad_ca_task& t : H.tasks) {
      const i64 q0 = qmap[static_cast<size_t>(t.q_off)];
      for (i64 j = 1; j < t.n_q; ++j)
        if (qmap[static_cast<size_t>(t.q_off + j)] != q0 + j) throw cad::DomainError("task rows not contiguous");
      t.q_off = q0;
      t.kv_off = kvmap[static_cast<size_t>(t.kv_off)];
    }
    // ---- exchanges: remap server rows, drop the own rows that no longer move
    for (i64 j = 0; j < qs.second; ++j)
      A.qd_self[h].push_back({QD.send_idx[static_cast<size_t>(qs.first + j)],
                              qmap[static_cast<size_t>(QD.recv_idx[static_cast<size_t>(qr.first + j)])]});
    auto filter_self = [&](XferRows& X, bool send_server, bool recv_server, const std::vector<i64>& map,
                           auto keep_self) {
      const auto ss = self_block(X.send_counts), rs = self_block(X.recv_counts);
      std::vector<i64> si, ri;
      i64 kept = 0;
      for (size_t j = 0; j < X.send_idx.size(); ++j) {
        const i64 jj = static_cast<i64>(j);
        const bool self = jj >= ss.first && jj < ss.first + ss.second;
        const i64 v = send_server ? map[static_cast<size_t>(X.send_idx[j])] : X.send_idx[j];
        if (self) {
          const i64 k = jj - ss.first;
          const i64 rv = X.recv_idx[static_cast<size_t>(rs.first + k)];
          if (!keep_self(X.send_idx[j], rv)) continue;
          ++kept;
        }
        si.push_back(v);
      }
      for (size_t j = 0; j < X.recv_idx.size(); ++j) {
        const i64 jj = static_cast<i64>(j);
        const bool self = jj >= rs.first && jj < rs.first + rs.second;
        if (self) {
          const i64 k = jj - rs.first;
          if (!keep_self(X.send_idx[static_cast<size_t>(ss.first + k)], X.recv_idx[j])) continue;
        }
        ri.push_back(recv_server ? map[static_cast<size_t>(X.recv_idx[j])] : X.recv_idx[j]);
      }
      X.send_idx = si;
      X.recv_idx = ri;
      X.send_counts[static_cast<size_t>(me)] = kept;
      X.recv_counts[static_cast<size_t>(me)] = kept;
    };
    // QD (Q, dO): home -> server view; own rows are in place
    filter_self(QD, false, true, qmap, [](i64, i64) { return false; });
    // KVD: home -> server view; own rows of assembled groups still copy
    filter_self(KD, false, true, kvmap, [&](i64, i64 srv) { return !aliased[static_cast<size_t>(srv)]; });
    // O_RET (O, dQ, LSE): server view -> home; own O/dQ in place, own LSE via lse_self
    XferRows& OR = H.x[kXO];
    {
      const auto os = self_block(OR.send_counts), orr = self_block(OR.recv_counts);
      for (i64 j = 0; j < os.second; ++j)
        A.lse_self[h].push_back({qmap[static_cast<size_t>(OR.send_idx[static_cast<size_t>(os.first + j)])],
                                 OR.recv_idx[static_cast<size_t>(orr.first + j)]});
    }
    filter_self(OR, true, false, qmap, [](i64, i64) { return false; });
    // KV_RET: server view -> owner staging; the own block stays (read in place)
    filter_self(H.x[kXKR], true, false, kvmap, [](i64, i64) { return true; });
    H.q_rows = h == 0 ? A.r[0] + A.home : A.home + A.r[1];
    H.kv_rows = h == 0 ? A.kr[0] + A.home : A.home + A.kr[1];
  }
  return A;
}

// Byte offsets of one rank's context-owned device buffers (one allocation,
// so IPC exports a single handle). Every rank computes every peer's layout
// from the peer's row plan.
struct Bufs {  // a half's views
  size_t q, k, v, o, dout, dq, dk, dv, lse, sdk, sdv;
};
struct Homes {  // a layer's home regions (inside its Q-like / K-like buffers)
  size_t q, k, v, o, dout, dq, lse;
};
struct Layout {
  size_t flags = 0;
  std::vector<std::array<Bufs, 2>> b;  // [layer][half]
  std::vector<Homes> home;             // [layer]
  size_t total = 0;
};

Layout layout_of(const RankRows& R, const Alias& A, int layers, int world, i64 q_row, i64 kv_row, i64 lse_row) {
  Layout L;
  size_t off = 0;
  auto take = [&](i64 bytes) {
    const size_t at = off;
    off += (static_cast<size_t>(std::max<i64>(bytes, 16)) + 255) / 256 * 256;
    return at;
  };
  L.flags = take(static_cast<i64>(4) * 2 * kKinds * world);
  L.b.resize(static_cast<size_t>(layers));
  L.home.resize(static_cast<size_t>(layers));
  const i64 qrows = A.r[0] + A.home + A.r[1], kvrows = A.kr[0] + A.home + A.kr[1];
  for (int l = 0; l < layers; ++l) {
    const size_t q = take(qrows * q_row), o = take(qrows * q_row), dout = take(qrows * q_row),
                 dq = take(qrows * q_row), k = take(kvrows * kv_row), v = take(kvrows * kv_row);
    Homes& Hm = L.home[static_cast<size_t>(l)];
    const size_t hq_off = static_cast<size_t>(A.r[0] * q_row), hk_off = static_cast<size_t>(A.kr[0] * kv_row);
    Hm = Homes{q + hq_off, k + hk_off, v + hk_off, o + hq_off, dout + hq_off, dq + hq_off,
               take(A.home * lse_row)};
    for (int h = 0; h < 2; ++h) {
      const HalfRows& H = R.half[h];
      const size_t qb = h == 0 ? 0 : static_cast<size_t>(A.r[0] * q_row);
      const size_t kb = h == 0 ? 0 : static_cast<size_t>(A.kr[0] * kv_row);
      const i64 qr = std::max<i64>(1, H.q_rows), kr = std::max<i64>(1, H.kv_rows);
      const i64 sr = std::max<i64>(1, H.x[kXKR].n_recv());
      Bufs& B = L.b[static_cast<size_t>(l)][static_cast<size_t>(h)];
      B.q = q + qb;
      B.o = o + qb;
      B.dout = dout + qb;
      B.dq = dq + qb;
      B.k = k + kb;
      B.v = v + kb;
      B.dk = take(kr * kv_row);
      B.dv = take(kr * kv_row);
      B.lse = take(qr * lse_row);
      B.sdk = take(sr * kv_row);
      B.sdv = take(sr * kv_row);
    }
  }
  L.total = off;
  return L;
}

// Maximal runs in which both the source and the destination row advance by one.
std::vector<cad_run> make_runs(const i64* src, const i64* dst, i64 n) {
  std::vector<cad_run> out;
  for (i64 i = 0; i < n;) {
    i64 j = i + 1;
    while (j < n && src[j] == src[j - 1] + 1 && dst[j] == dst[j - 1] + 1) ++j;
    out.push_back({src[i], dst[i], j - i});
    i = j;
  }
  return out;
}

struct BlobRef {
  uint8_t handle[64];
  int64_t offset;
  uint64_t raw;
};
struct Blob {
  uint32_t magic;
  int32_t rank, world, transport, layers, pad;
  int64_t home_rows;
  BlobRef ref[4];  // [0] the arena (the others unused)
};

struct Peer {
  char* arena = nullptr;
  i64 home_rows = 0;
  i64 q_pitch[2] = {1, 1};  // rows of the peer's server Q/LSE buffers per half
  Layout layout;
};

// dK/dV at the owner: every home KV row gathers its partials -- one per
// (server, half, layer) that used it, listed in CSR form (off[row] ..
// off[row+1]) as a row of a half's staging (peers' partials) or of its server
// dK/dV buffer (this rank's own) -- sums them in fp32 and writes bf16
// (and fp32 when asked). One warp per row, 16-byte loads; each partial is read
// once and each output written once: no memset, no atomics.
__global__ void __launch_bounds__(256) reduce_partials_kernel(const int64_t* __restrict__ off,
                                                              const int32_t* __restrict__ ent,
                                                              const uint4* const* __restrict__ src,  // [layer][half]
                                                              int n_layers, int64_t rows, int chunks,
                                                              uint4* __restrict__ out_bf16,
                                                              float4* __restrict__ out_f32) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const int64_t e0 = off[row], e1 = off[row + 1];
  for (int c = lane; c < chunks; c += 32) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t e = e0; e < e1; ++e) {
      const int32_t v = ent[e];
      const int slot = v & 3;  // own (server buffer) << 1 | half
      const int64_t srow = v >> 2;
      for (int l = 0; l < n_layers; ++l) {
        const uint4 x = src[l * 4 + slot][srow * chunks + c];
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&x);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __bfloat1622float2(b[i]);
          acc[2 * i] += f.x;
          acc[2 * i + 1] += f.y;
        }
      }
    }
    if (out_bf16) {
      uint4 o;
      __nv_bfloat162* ob = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
      for (int i = 0; i < 4; ++i) ob[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      out_bf16[row * chunks + c] = o;
    }
    if (out_f32) {
      out_f32[(row * chunks + c) * 2] = make_float4(acc[0], acc[1], acc[2], acc[3]);
      out_f32[(row * chunks + c) * 2 + 1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
  }
}

// This rank's own rows (tasks it serves itself) move between its home and
// server buffers in ONE launch per exchange: chunks of <= kChunkRows rows
// (src_row, dst_row, n) dealt to CTAs grid-stride, 16-byte vectors. One
// cudaMemcpyAsync per run instead costs the host microseconds per run --
// thousands per step with short documents -- and the GPU idles behind it.
constexpr int kChunkRows = 32;
__global__ void __launch_bounds__(256) copy_row_chunks_kernel(const int64_t* __restrict__ chunks, int64_t n_chunks,
                                                              const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                              int64_t row_vec) {
  for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int64_t sr = chunks[3 * c], dr = chunks[3 * c + 1], n = chunks[3 * c + 2];
    const uint4* s = src + sr * row_vec;
    uint4* d = dst + dr * row_vec;
    for (int64_t i = threadIdx.x; i < n * row_vec; i += blockDim.x) d[i] = s[i];
  }
}
// The same for the [heads][rows] fp32 LSE.
__global__ void __launch_bounds__(256) copy_col_chunks_kernel(const int64_t* __restrict__ chunks, int64_t n_chunks,
                                                              const float* __restrict__ src, int64_t src_rows,
                                                              float* __restrict__ dst, int64_t dst_rows, int heads) {
  for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
    const int64_t sr = chunks[3 * c], dr = chunks[3 * c + 1], n = chunks[3 * c + 2];
    for (int64_t i = threadIdx.x; i < n * heads; i += blockDim.x) {
      const int64_t h = i / n, j = i - h * n;
      dst[h * dst_rows + dr + j] = src[h * src_rows + sr + j];
    }
  }
}

template <class T>
T* dev_copy(const std::vector<T>& v) {
  T* d = nullptr;
  cuda_check(cudaMalloc(reinterpret_cast<void**>(&d), std::max<size_t>(1, v.size()) * sizeof(T)), "cudaMalloc");
  if (!v.empty()) cuda_check(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy");
  return d;
}

}  // namespace

struct cad_layer_ctx {
  cad_layer_cfg cfg{};
  int device = 0;
  int W = 1, me = 0, NL = 1;
  i64 hq = 0, hkv = 0, d = 128;
  i64 q_row = 0, kv_row = 0, lse_row = 0;
  RankRows mine;  // this rank's row plan
  cad_ca_plan* plan[2] = {nullptr, nullptr};
  void* ws[2] = {nullptr, nullptr};
  size_t ws_bytes[2] = {0, 0};
  i64 pairs = 0;
  Layout layout;
  char* arena = nullptr;
  int32_t* flags = nullptr;
  std::vector<Peer> peer;
  std::vector<void*> opened;  // IPC mappings to close
  std::vector<cad_run> runs[2][4];  // per (half, xfer): runs of all peers, grouped by peer
  std::vector<size_t> run_off[2][4];  // per peer: first run (W + 1 entries)
  int64_t* d_local_chunks[2][4] = {};  // this rank's own rows: device chunk lists
  int64_t n_local_chunks[2][4] = {};
  // NCCL: row lists without this rank's own rows (those move by the local
  // copy kernels), counts with the self entry zeroed, and the original
  // receive offsets (partials land in the staging at their full-order rows)
  struct NcclX {
    std::vector<i64> sc, rc, rd_full;
    i64 n_send = 0, n_recv = 0;
    i64* d_send = nullptr;
    i64* d_recv = nullptr;
  };
  NcclX nx[2][4];
  int64_t* d_red_off = nullptr;  // dK/dV reduction CSR over home rows
  int32_t* d_red_ent = nullptr;  // (row << 2) | (own << 1) | half
  const uint4** d_red_src[2] = {nullptr, nullptr};  // dK, dV bases [layer][own][half]
  Alias alias;  // this rank's zero-copy layout (alias_rows)
  // own rows that still move: LSE re-layout (server view -> home) and the
  // forward state's LSE (home -> server view), device chunk lists per half
  int64_t* d_lse_self[2] = {};
  int64_t n_lse_self[2] = {};
  int64_t* d_qd_self[2] = {};
  int64_t n_qd_self[2] = {};
  bool connected = false;
  cad_comm* comm = nullptr;
  void* xsend = nullptr;
  void* xrecv = nullptr;
  size_t xbytes = 0;
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> ev;
  uint32_t gen = 0, g0 = 0;
  i64 launches = 0;
  bool move_remote = true;  // false: signal mode -- this rank's own rows still
                            // move, the transfers to peers shrink to their flags

  // ------------------------------------------------------------- helpers
  Bufs b(int l, int h) const { return layout.b[static_cast<size_t>(l)][static_cast<size_t>(h)]; }
  template <class T = void>
  T* at(size_t off) const { return reinterpret_cast<T*>(arena + off); }
  template <class T = void>
  T* peer_at(int p, size_t off) const { return reinterpret_cast<T*>(peer[static_cast<size_t>(p)].arena + off); }
  const Bufs& pb(int p, int l, int h) const {
    return peer[static_cast<size_t>(p)].layout.b[static_cast<size_t>(l)][static_cast<size_t>(h)];
  }
  const Homes& hm(int l) const { return layout.home[static_cast<size_t>(l)]; }
  const Homes& phm(int p, int l) const { return peer[static_cast<size_t>(p)].layout.home[static_cast<size_t>(l)]; }
  // copy a caller buffer into (or out of) a home region, unless it IS that region
  void stage(void* dst, const void* src, i64 bytes, cudaStream_t s) const {
    if (!src || !dst || src == dst || bytes <= 0) return;
    cuda_check(cudaMemcpyAsync(dst, src, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice, s), "stage copy");
  }
  void cols(const int64_t* chunks, int64_t n, const float* src, i64 src_rows, float* dst, i64 dst_rows,
            cudaStream_t s) {
    if (n <= 0) return;
    copy_col_chunks_kernel<<<static_cast<unsigned>(std::min<int64_t>(n, 148 * 4)), 256, 0, s>>>(
        chunks, n, src, src_rows, dst, dst_rows, static_cast<int>(hq));
    cuda_check(cudaGetLastError(), "copy_col_chunks launch");
    ++launches;
  }
  void stage_fwd_state(const cad_layer_io* io, int l, cudaStream_t s) const {
    stage(at(hm(l).o), io->o, mine.home_rows * q_row, s);
    stage(at(hm(l).lse), io->lse, mine.home_rows * lse_row, s);
  }
  // the step's inputs into the layers' home regions (a NULL input: the
  // caller wrote the home region itself, cad_layer_ctx_home)
  void stage_inputs(const cad_layer_io* io, bool qkv, bool dout, cudaStream_t s) const {
    const i64 H = mine.home_rows;
    for (int l = 0; l < NL; ++l) {
      if (qkv) {
        stage(at(hm(l).q), io->q, H * q_row, s);
        stage(at(hm(l).k), io->k, H * kv_row, s);
        stage(at(hm(l).v), io->v, H * kv_row, s);
      }
      if (dout) stage(at(hm(l).dout), io->dout, H * q_row, s);
    }
  }
  uint32_t gl(int l) const { return g0 + 1 + static_cast<uint32_t>(l); }
  uint32_t gb(int l) const { return g0 + 2 * static_cast<uint32_t>(NL) - static_cast<uint32_t>(l); }
  uint32_t gdone() const { return g0 + 2 * static_cast<uint32_t>(NL); }
  bool flagged() const { return cfg.transport != CAD_TRANSPORT_NCCL; }
  int32_t* flag_of(int p, int kind, int h, int src) const {
    int32_t* base = p == me ? flags : peer_at<int32_t>(p, peer[static_cast<size_t>(p)].layout.flags);
    return base + (kind * 2 + h) * W + src;
  }
  void signal(int kind, int h, uint32_t value, cudaStream_t s) const {
    if (trace_host()) std::fprintf(stderr, "[cad] rank %d signal kind %d half %d value %u\n", me, kind, h, value);
    for (int p = 0; p < W; ++p) ok(cad_stream_write_u32(flag_of(p, kind, h, me), value, s), "signal");
  }
  void await(int kind, int h, uint32_t value, cudaStream_t s) const {
    if (trace_host()) std::fprintf(stderr, "[cad] rank %d await kind %d half %d value %u\n", me, kind, h, value);
    for (int src = 0; src < W; ++src) ok(cad_stream_wait_u32(flag_of(me, kind, h, src), value, s), "await");
  }
  cudaEvent_t event(int slot) const { return ev[static_cast<size_t>(slot)]; }

  // rows of exchange x (half h) from src into every peer's buffer dst_of(p);
  // this rank's own rows go on `local` (the compute stream in a step: a
  // local copy overlapping a CA kernel crawls and would hold up the remote
  // pushes queued behind it)
  template <class DstOf>
  void push(int h, int x, const void* src, i64 row_bytes, DstOf dst_of, cudaStream_t s, cudaStream_t local) {
    for (int p = 0; p < W; ++p) {
      const size_t a = run_off[h][x][static_cast<size_t>(p)], e = run_off[h][x][static_cast<size_t>(p) + 1];
      if (a == e) continue;
      if (p == me) {
        // own dK/dV partials stay in the server buffers (the reduction reads them there)
        if (x == kXKR) continue;
        const int64_t n = n_local_chunks[h][x];
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(n, 148 * 4));
        copy_row_chunks_kernel<<<grid, 256, 0, local>>>(d_local_chunks[h][x], n, static_cast<const uint4*>(src),
                                                        static_cast<uint4*>(dst_of(p)), row_bytes / 16);
        cuda_check(cudaGetLastError(), "copy_row_chunks launch");
        ++launches;
        continue;
      }
      if (!move_remote) continue;
      if (lanes.empty()) {
        ok(cad_copy_runs(runs[h][x].data() + a, static_cast<i64>(e - a), src, dst_of(p), row_bytes, s),
           "cad_copy_runs");
        continue;
      }
      for (size_t i = a; i < e; ++i) {  // split into <= kLanePiece pieces over the lanes
        const cad_run& r = runs[h][x][i];
        const char* sp = static_cast<const char*>(src) + r.src_row * row_bytes;
        char* dp = static_cast<char*>(dst_of(p)) + r.dst_row * row_bytes;
        for (i64 off = 0, n = r.n_rows * row_bytes; off < n; off += kLanePiece)
          pieces.push_back({sp + off, dp + off, std::min<i64>(kLanePiece, n - off)});
      }
    }
    flush_pieces(s);
  }

  // CAD_PUSH_LANES=k (k > 1): remote pushes spread over k extra streams (forked
  // from and joined back into the pushing stream), so several copy engines
  // drive NVLink at once
  static constexpr i64 kLanePiece = 16 << 20;
  std::vector<cudaStream_t> lanes;
  std::vector<cudaEvent_t> lane_ev;  // [0] fork, [1..k] joins
  struct Piece {
    const char* src;
    char* dst;
    i64 bytes;
  };
  std::vector<Piece> pieces;
  void flush_pieces(cudaStream_t s) {
    if (pieces.empty()) return;
    cuda_check(cudaEventRecord(lane_ev[0], s), "event(fork)");
    std::vector<i64> load(lanes.size(), 0);
    for (size_t k = 0; k < lanes.size(); ++k) cuda_check(cudaStreamWaitEvent(lanes[k], lane_ev[0], 0), "wait");
    for (const Piece& pc : pieces) {
      const size_t k = static_cast<size_t>(std::min_element(load.begin(), load.end()) - load.begin());
      cuda_check(cudaMemcpyAsync(pc.dst, pc.src, static_cast<size_t>(pc.bytes), cudaMemcpyDeviceToDevice, lanes[k]),
                 "cudaMemcpyAsync(lane)");
      load[k] += pc.bytes;
    }
    for (size_t k = 0; k < lanes.size(); ++k) {
      cuda_check(cudaEventRecord(lane_ev[k + 1], lanes[k]), "event(join)");
      cuda_check(cudaStreamWaitEvent(s, lane_ev[k + 1], 0), "wait(join)");
    }
    pieces.clear();
  }
  // [heads][rows] fp32 columns (LSE) of exchange x: dst_of(p) gives the
  // peer's buffer and its row pitch
  template <class DstOf>
  void push_cols(int h, int x, const float* src, i64 src_rows, DstOf dst_of, cudaStream_t s, cudaStream_t local) {
    for (int p = 0; p < W; ++p) {
      const size_t a = run_off[h][x][static_cast<size_t>(p)], e = run_off[h][x][static_cast<size_t>(p) + 1];
      if (a == e) continue;
      const std::pair<float*, i64> dst = dst_of(p);
      if (p == me) {
        const int64_t n = n_local_chunks[h][x];
        const unsigned grid = static_cast<unsigned>(std::min<int64_t>(n, 148 * 4));
        copy_col_chunks_kernel<<<grid, 256, 0, local>>>(d_local_chunks[h][x], n, src, src_rows, dst.first,
                                                        dst.second, static_cast<int>(hq));
        cuda_check(cudaGetLastError(), "copy_col_chunks launch");
        ++launches;
        continue;
      }
      if (!move_remote) continue;
      ok(cad_copy_runs_cols(runs[h][x].data() + a, static_cast<i64>(e - a), src, src_rows, dst.first, dst.second,
                            static_cast<int32_t>(hq), s),
         "cad_copy_runs_cols");
    }
  }
  void push_lse(int l, int h, const float* src, i64 src_rows, cudaStream_t s, cudaStream_t local) {
    push_cols(h, kXO, src, src_rows,
              [&](int p) {
                return std::make_pair(peer_at<float>(p, phm(p, l).lse), peer[static_cast<size_t>(p)].home_rows);
              },
              s, local);
    cols(d_lse_self[h], n_lse_self[h], src, src_rows, at<float>(hm(l).lse), mine.home_rows, local);
  }

  // NCCL: gather, all-to-allv, then scatter (or, with dst_contig, receive
  // straight into a buffer in recv order)
  void nccl_rows(int h, int x, const void* src, i64 row_bytes, void* dst, bool dst_contig, cudaStream_t s,
                 cudaStream_t local) {
    const NcclX& X = nx[h][x];
    ok(cad_gather_rows(src, X.d_send, X.n_send, row_bytes, xsend, s), "cad_gather_rows");
    launches += X.n_send > 0;
    alltoallv(X, row_bytes, dst_contig ? dst : xrecv, dst_contig, s);
    if (!dst_contig) {
      ok(cad_scatter_rows(xrecv, X.d_recv, X.n_recv, row_bytes, dst, s), "cad_scatter_rows");
      launches += X.n_recv > 0;
    }
    // own rows: one local copy kernel (own dK/dV partials are read in place)
    if (x != kXKR && n_local_chunks[h][x] > 0) {
      const int64_t n = n_local_chunks[h][x];
      copy_row_chunks_kernel<<<static_cast<unsigned>(std::min<int64_t>(n, 148 * 4)), 256, 0, local>>>(
          d_local_chunks[h][x], n, static_cast<const uint4*>(src), static_cast<uint4*>(dst), row_bytes / 16);
      cuda_check(cudaGetLastError(), "copy_row_chunks launch");
      ++launches;
    }
  }
  void nccl_cols(int h, int x, const float* src, i64 src_rows, float* dst, i64 dst_rows, cudaStream_t s) {
    const NcclX& X = nx[h][x];
    ok(cad_gather_cols_f32(src, src_rows, static_cast<int32_t>(hq), X.d_send, X.n_send,
                           static_cast<float*>(xsend), s),
       "cad_gather_cols_f32");
    alltoallv(X, lse_row, xrecv, false, s);
    ok(cad_scatter_cols_f32(static_cast<const float*>(xrecv), X.d_recv, X.n_recv, static_cast<int32_t>(hq), dst,
                            dst_rows, s),
       "cad_scatter_cols_f32");
    launches += (X.n_send > 0) + (X.n_recv > 0);
  }
  void alltoallv(const NcclX& X, i64 row_bytes, void* recv, bool full_order, cudaStream_t s) const {
    if (!comm) throw cad::ConfigError("NCCL transport: cad_layer_ctx_set_comm was not called");
    std::vector<i64> sb(static_cast<size_t>(W)), sd(static_cast<size_t>(W)), rb(static_cast<size_t>(W)),
        rd(static_cast<size_t>(W));
    i64 so = 0, ro = 0;
    for (int p = 0; p < W; ++p) {
      const size_t q = static_cast<size_t>(p);
      sb[q] = X.sc[q] * row_bytes;
      rb[q] = X.rc[q] * row_bytes;
      sd[q] = so;
      rd[q] = full_order ? X.rd_full[q] * row_bytes : ro;
      so += sb[q];
      ro += rb[q];
    }
    ok(cad_alltoallv(comm, xsend, sb.data(), sd.data(), recv, rb.data(), rd.data(), s), "cad_alltoallv");
  }

  void check_io(const cad_layer_io* io, bool) const {
    if (!io) throw cad::DomainError("null io");
  }
  void need_ready() const {
    if (flagged() && !connected) throw cad::ConfigError("layer context not connected (cad_layer_ctx_connect)");
    if (!flagged() && !comm) throw cad::ConfigError("NCCL transport: cad_layer_ctx_set_comm was not called");
  }
  void check_lh(int l, int h) const {
    if (l < 0 || l >= NL || h < 0 || h > 1) throw cad::DomainError("layer or half out of range");
  }

  // ------------------------------------------------------------- phases
  int passes = CAD_PASS_BOTH;  // of the current step
  void begin(cudaStream_t s, int passes_ = CAD_PASS_BOTH) {
    need_ready();
    if (passes_ < CAD_PASS_FWD || passes_ > CAD_PASS_BOTH) throw cad::DomainError("passes must be FWD, BWD or BOTH");
    if (passes_ != CAD_PASS_BOTH && NL != 1) throw cad::ConfigError("single-pass steps need layers == 1");
    passes = passes_;
    g0 = gen;
    gen += 2 * static_cast<uint32_t>(NL);
    // every peer finished the previous step: its server buffers are free
    if (flagged()) await(F_DONE, 0, g0, s);
  }

  // Transfers read and write the layers' home regions (the caller's buffers
  // are staged in and out by stage_inputs / finish); a rank's own rows are
  // already in place in its server views.
  void dispatch(int l, int h, int what, const cad_layer_io*, cudaStream_t s, cudaStream_t local) {
    const Bufs& B = b(l, h);
    const Homes& Hm = hm(l);
    if (what == CAD_DISPATCH_QKV) {
      if (flagged()) {
        // identity between stacked layers: layer l's Q/K/V of half h leave
        // home once every server has returned O(h, l-1)
        if (l > 0) await(F_O, h, gl(l - 1), s);
        push(h, kXQ, at(Hm.q), q_row, [&](int p) { return peer_at(p, pb(p, l, h).q); }, s, local);
        push(h, kXKV, at(Hm.k), kv_row, [&](int p) { return peer_at(p, pb(p, l, h).k); }, s, local);
        push(h, kXKV, at(Hm.v), kv_row, [&](int p) { return peer_at(p, pb(p, l, h).v); }, s, local);
        signal(F_QKV, h, gl(l), s);
      } else {
        nccl_rows(h, kXQ, at(Hm.q), q_row, at(B.q), false, s, local);
        nccl_rows(h, kXKV, at(Hm.k), kv_row, at(B.k), false, s, local);
        nccl_rows(h, kXKV, at(Hm.v), kv_row, at(B.v), false, s, local);
      }
    } else if (what == CAD_DISPATCH_FWD_STATE) {
      // O and LSE rows home -> server, for a backward whose forward ran under
      // another plan (a pipeline tick's backward, P/src/sim.cpp:326-353);
      // ordered before the consumer by the DO dispatch's flag that follows.
      // Own O rows are in place; own LSE columns are re-laid out.
      const i64 pitch = std::max<i64>(1, mine.half[h].q_rows);
      if (flagged()) {
        push(h, kXQ, at(Hm.o), q_row, [&](int p) { return peer_at(p, pb(p, l, h).o); }, s, local);
        push_cols(h, kXQ, at<float>(Hm.lse), mine.home_rows,
                  [&](int p) {
                    return std::make_pair(peer_at<float>(p, pb(p, l, h).lse), peer[static_cast<size_t>(p)].q_pitch[h]);
                  },
                  s, local);
      } else {
        nccl_rows(h, kXQ, at(Hm.o), q_row, at(B.o), false, s, local);
        nccl_cols(h, kXQ, at<float>(Hm.lse), mine.home_rows, at<float>(B.lse), pitch, s);
      }
      cols(d_qd_self[h], n_qd_self[h], at<float>(Hm.lse), mine.home_rows, at<float>(B.lse), pitch, local);
    } else if (what == CAD_DISPATCH_DO) {
      if (flagged()) {
        if (l < NL - 1) await(F_G, h, gb(l + 1), s);  // dQ(h, l+1) home -> dO(h, l)
        push(h, kXQ, at(Hm.dout), q_row, [&](int p) { return peer_at(p, pb(p, l, h).dout); }, s, local);
        signal(F_DO, h, gb(l), s);
      } else {
        nccl_rows(h, kXQ, at(Hm.dout), q_row, at(B.dout), false, s, local);
      }
    } else {
      throw cad::DomainError("unknown dispatch kind");
    }
  }

  void compute(int l, int h, bool bwd, cudaStream_t s, bool wait_flags, bool run) {
    if (wait_flags && flagged()) await(bwd ? F_DO : F_QKV, h, bwd ? gb(l) : gl(l), s);
    if (!run || !plan[h]) return;
    const Bufs& B = b(l, h);
    if (!bwd) {
      ok(cad_ca_fwd(plan[h], at(B.q), at(B.k), at(B.v), at(B.o), at<float>(B.lse), s), "cad_ca_fwd");
      launches += 1;
    } else {
      // dK/dV of every KV group's rows are overwritten (rows of a view outside
      // every group are never read)
      ok(cad_ca_bwd(plan[h], at(B.q), at(B.k), at(B.v), at(B.o), at<float>(B.lse), at(B.dout), at(B.dq), at(B.dk),
                    at(B.dv), ws[h], ws_bytes[h], s),
         "cad_ca_bwd");
      launches += 3;
    }
  }

  void ret(int l, int h, int what, const cad_layer_io*, cudaStream_t s, cudaStream_t local) {
    const Bufs& B = b(l, h);
    const Homes& Hm = hm(l);
    const i64 qr = std::max<i64>(1, mine.half[h].q_rows);
    if (what == CAD_RETURN_O) {
      if (flagged()) {
        push(h, kXO, at(B.o), q_row, [&](int p) { return peer_at(p, phm(p, l).o); }, s, local);
        push_lse(l, h, at<float>(B.lse), qr, s, local);
        signal(F_O, h, gl(l), s);
      } else {
        nccl_rows(h, kXO, at(B.o), q_row, at(Hm.o), false, s, local);
        nccl_cols(h, kXO, at<float>(B.lse), qr, at<float>(Hm.lse), mine.home_rows, s);
        cols(d_lse_self[h], n_lse_self[h], at<float>(B.lse), qr, at<float>(Hm.lse), mine.home_rows, local);
      }
    } else if (what == CAD_RETURN_GRAD) {
      if (flagged()) {
        push(h, kXO, at(B.dq), q_row, [&](int p) { return peer_at(p, phm(p, l).dq); }, s, local);
        push(h, kXKR, at(B.dk), kv_row, [&](int p) { return peer_at(p, pb(p, l, h).sdk); }, s, local);
        push(h, kXKR, at(B.dv), kv_row, [&](int p) { return peer_at(p, pb(p, l, h).sdv); }, s, local);
        signal(F_G, h, gb(l), s);
      } else {
        nccl_rows(h, kXO, at(B.dq), q_row, at(Hm.dq), false, s, local);
        nccl_rows(h, kXKR, at(B.dk), kv_row, at(B.sdk), true, s, local);  // partials land in recv order
        nccl_rows(h, kXKR, at(B.dv), kv_row, at(B.sdv), true, s, local);
      }
    } else {
      throw cad::DomainError("unknown return kind");
    }
  }

  void finish(const cad_layer_io* io, cudaStream_t s) {
    if (flagged())
      for (int h = 0; h < 2; ++h) {
        if (passes & CAD_PASS_FWD) await(F_O, h, gl(NL - 1), s);
        if (passes & CAD_PASS_BWD) await(F_G, h, gb(0), s);
      }
    // outputs to the caller's buffers when they are not the home regions:
    // O/LSE of the last layer, dQ of the first (the backward ends there)
    const i64 rows = mine.home_rows;
    if (passes & CAD_PASS_FWD) {
      stage(io->o, at(hm(NL - 1).o), rows * q_row, s);
      stage(io->lse, at(hm(NL - 1).lse), rows * lse_row, s);
    }
    if (!(passes & CAD_PASS_BWD)) {
      if (flagged()) signal(F_DONE, 0, gdone(), s);
      return;
    }
    stage(io->dq, at(hm(0).dq), rows * q_row, s);
    const int chunks = static_cast<int>(hkv * d / 8);
    if (rows > 0 && (io->dk || io->dk_acc || io->dv || io->dv_acc)) {
      const unsigned blocks = static_cast<unsigned>((rows + 7) / 8);
      const int n_layers = NL;
      reduce_partials_kernel<<<blocks, 256, 0, s>>>(d_red_off, d_red_ent, d_red_src[0], n_layers, rows, chunks,
                                                    static_cast<uint4*>(io->dk), reinterpret_cast<float4*>(io->dk_acc));
      reduce_partials_kernel<<<blocks, 256, 0, s>>>(d_red_off, d_red_ent, d_red_src[1], n_layers, rows, chunks,
                                                    static_cast<uint4*>(io->dv), reinterpret_cast<float4*>(io->dv_acc));
      cuda_check(cudaGetLastError(), "reduce_partials launch");
      launches += 2;
    }
    if (flagged()) signal(F_DONE, 0, gdone(), s);
  }

  // ------------------------------------------------------------- one step
  // Event slots: [0] start, [1] comm done, then per (layer, half) 4 slots:
  // QKV arrived, dO arrived, forward done, backward done.
  int slot(int l, int h, int k) const { return 2 + ((l * 2 + h) * 4 + k); }

  void step(const cad_layer_io* io, int mode, cudaStream_t comp, int passes_ = CAD_PASS_BOTH) {
    need_ready();
    // One thread enqueueing a whole step of rank 0 before rank 1's puts GPU
    // waits ahead of the work that releases them; streams of one context can
    // share a hardware queue (CUDA_DEVICE_MAX_CONNECTIONS), so such a wait can
    // hold up the very stream it waits for. LOCAL contexts are therefore
    // driven phase by phase (cad_layer_begin / cad_dispatch / ... in
    // dependency order across ranks), never by cad_layer_step.
    if (cfg.transport == CAD_TRANSPORT_LOCAL && mode != CAD_STEP_COMPUTE)
      throw cad::ConfigError("cad_layer_step needs one process per rank (IPC or NCCL transport); drive LOCAL "
                             "contexts with the per-layer entry points in dependency order");
    if (mode == CAD_STEP_COMPUTE) {
      if (passes_ & CAD_PASS_FWD)
        for (int l = 0; l < NL; ++l)
          for (int h = 0; h < 2; ++h) compute(l, h, false, comp, false, true);
      if (passes_ & CAD_PASS_BWD)
        for (int l = NL - 1; l >= 0; --l)
          for (int h = 0; h < 2; ++h) compute(l, h, true, comp, false, true);
      return;
    }
    if ((mode == CAD_STEP_SIGNAL || mode == CAD_STEP_COMM_LOCAL) && !flagged())
      throw cad::ConfigError("signal modes need the LOCAL or IPC transport");
    if (mode < CAD_STEP_PINGPONG || mode > CAD_STEP_COMM_LOCAL) throw cad::DomainError("unknown step mode");
    check_io(io, true);
    const bool run = mode != CAD_STEP_COMM && mode != CAD_STEP_COMM_LOCAL;
    move_remote = mode != CAD_STEP_SIGNAL && mode != CAD_STEP_COMM_LOCAL;
    cudaStream_t comm = mode == CAD_STEP_SERIAL ? comp : comm_stream;
    struct Restore {
      cad_layer_ctx* c;
      ~Restore() { c->move_remote = true; }
    } restore{this};
    trace_reset(comp);
    // the caller's inputs into the home regions (on the compute stream, before
    // the comm stream forks off it)
    stage_inputs(io, true, (passes_ & CAD_PASS_BWD) != 0, comp);
    if (passes_ == CAD_PASS_BWD) stage_fwd_state(io, 0, comp);
    cuda_check(cudaEventRecord(event(0), comp), "event");
    cuda_check(cudaStreamWaitEvent(comm, event(0), 0), "wait");
    begin(comm, passes_);
    auto disp = [&](int l, int h, int what) {
      const int m0 = tmark(comm);
      dispatch(l, h, what, io, comm, comp);
      trace_add(what == CAD_DISPATCH_QKV ? CAD_TRACE_DISPATCH_QKV : CAD_TRACE_DISPATCH_DO, l, h, m0, m0,
                tmark(comm));
      cuda_check(cudaEventRecord(event(slot(l, h, what == CAD_DISPATCH_QKV ? 0 : 1)), comm), "event");
    };
    auto ca = [&](int l, int h, bool bwd) {
      const int m0 = tmark(comp);
      cuda_check(cudaStreamWaitEvent(comp, event(slot(l, h, bwd ? 1 : 0)), 0), "wait");
      if (flagged()) await(bwd ? F_DO : F_QKV, h, bwd ? gb(l) : gl(l), comp);
      const int m1 = tmark(comp);
      compute(l, h, bwd, comp, false, run);
      trace_add(bwd ? CAD_TRACE_BWD : CAD_TRACE_FWD, l, h, m0, m1, tmark(comp));
      cuda_check(cudaEventRecord(event(slot(l, h, bwd ? 3 : 2)), comp), "event");
    };
    auto back = [&](int l, int h, int what) {
      cuda_check(cudaStreamWaitEvent(comm, event(slot(l, h, what == CAD_RETURN_O ? 2 : 3)), 0), "wait");
      const int m0 = tmark(comm);
      ret(l, h, what, io, comm, comp);
      trace_add(what == CAD_RETURN_O ? CAD_TRACE_RETURN_O : CAD_TRACE_RETURN_GRAD, l, h, m0, m0, tmark(comm));
    };
    if (passes_ != CAD_PASS_BOTH) {  // one pass of one layer (a pipeline tick)
      const bool bwd = passes_ == CAD_PASS_BWD;
      for (int h = 0; h < 2; ++h) {
        disp(0, h, CAD_DISPATCH_QKV);
        if (bwd) {
          disp(0, h, CAD_DISPATCH_FWD_STATE);
          disp(0, h, CAD_DISPATCH_DO);
        }
        ca(0, h, bwd);
      }
      for (int h = 0; h < 2; ++h) back(0, h, bwd ? CAD_RETURN_GRAD : CAD_RETURN_O);
      cuda_check(cudaEventRecord(event(1), comm), "event");
      cuda_check(cudaStreamWaitEvent(comp, event(1), 0), "wait");
      finish(io, comp);
      return;
    }
    // forward: comm D(0,0) D(1,0) dO(.,L-1) | R(0,l) D(0,l+1) | R(1,l) D(1,l+1) ...
    //          comp       F(0,0)    F(1,0)      F(0,l+1)         F(1,l+1)
    // so the return of half h and the next dispatch hide under CA(1-h)
    // (the reference's windows, P/src/sim.cpp:69-72)
    disp(0, 0, CAD_DISPATCH_QKV);
    ca(0, 0, false);
    disp(0, 1, CAD_DISPATCH_QKV);
    disp(NL - 1, 0, CAD_DISPATCH_DO);  // the loss gradient of the top layer
    disp(NL - 1, 1, CAD_DISPATCH_DO);
    ca(0, 1, false);
    for (int l = 0; l < NL; ++l)
      for (int h = 0; h < 2; ++h) {
        back(l, h, CAD_RETURN_O);
        if (l + 1 < NL) {
          disp(l + 1, h, CAD_DISPATCH_QKV);
          ca(l + 1, h, false);
        }
      }
    // backward, top layer first: G(h,l) then dO(h,l-1) under the other half's CA
    ca(NL - 1, 0, true);
    ca(NL - 1, 1, true);
    for (int l = NL - 1; l >= 0; --l)
      for (int h = 0; h < 2; ++h) {
        back(l, h, CAD_RETURN_GRAD);
        if (l > 0) {
          disp(l - 1, h, CAD_DISPATCH_DO);
          ca(l - 1, h, true);
        }
      }
    cuda_check(cudaEventRecord(event(1), comm), "event");
    const int f0 = tmark(comp);
    cuda_check(cudaStreamWaitEvent(comp, event(1), 0), "wait");
    const int f1 = tmark(comp);
    finish(io, comp);
    trace_add(CAD_TRACE_FINISH, 0, 0, f0, f1, tmark(comp));
  }

  // ------------------------------------------------------------- tracing
  // With tracing on, a step records timing events around every phase; the
  // records of the last step are read back with cad_layer_ctx_trace.
  bool tracing = false;
  std::vector<cudaEvent_t> tev;  // timing events, [0] = step start
  int tused = 0;
  struct TraceRow {
    int kind, layer, half, m0, m1, m2;
  };
  std::vector<TraceRow> trows;
  void trace_reset(cudaStream_t s) {
    trows.clear();
    tused = 0;
    if (tracing) tmark(s);
  }
  int tmark(cudaStream_t s) {
    if (!tracing) return -1;
    if (tused == static_cast<int>(tev.size())) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "cudaEventCreate");
      tev.push_back(e);
    }
    cuda_check(cudaEventRecord(tev[static_cast<size_t>(tused)], s), "event");
    return tused++;
  }
  void trace_add(int kind, int l, int h, int m0, int m1, int m2) {
    if (tracing) trows.push_back({kind, l, h, m0, m1, m2});
  }

  ~cad_layer_ctx() {  // runs with the context's device current
    for (void* base : opened) cudaIpcCloseMemHandle(base);
    for (int h = 0; h < 2; ++h) {
      if (plan[h]) cad_ca_plan_destroy(plan[h]);
      cudaFree(ws[h]);
      for (int x = 0; x < 4; ++x) {
        cudaFree(nx[h][x].d_send);
        cudaFree(nx[h][x].d_recv);
        cudaFree(d_local_chunks[h][x]);
      }
      cudaFree(d_lse_self[h]);
      cudaFree(d_qd_self[h]);
      cudaFree(d_red_src[h]);
    }
    cudaFree(arena);
    cudaFree(d_red_off);
    cudaFree(d_red_ent);
    cudaFree(xsend);
    cudaFree(xrecv);
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    for (cudaEvent_t e : tev) cudaEventDestroy(e);
    for (cudaEvent_t e : lane_ev) cudaEventDestroy(e);
    for (cudaStream_t st : lanes) cudaStreamDestroy(st);
    if (comm_stream) cudaStreamDestroy(comm_stream);
  }
};

extern "C" {

int cad_layer_ctx_create(const cad_plan* plan, const cad_item* home_items, int64_t n_items, const cad_layer_cfg* cfg,
                         cad_layer_ctx** out) {
  return cad::guarded([&] {
    if (!plan || !cfg || !out || (n_items > 0 && !home_items)) throw cad::DomainError("null argument");
    *out = nullptr;
    if (cfg->world < 1 || cfg->rank < 0 || cfg->rank >= cfg->world) throw cad::DomainError("rank out of range");
    if (cfg->head_dim != 128) throw cad::ConfigError("head_dim must be 128");
    if (cfg->h_q < 1 || cfg->h_kv < 1 || cfg->h_q % cfg->h_kv) throw cad::ConfigError("h_q must be a multiple of h_kv");
    if (cfg->transport < CAD_TRANSPORT_LOCAL || cfg->transport > CAD_TRANSPORT_NCCL)
      throw cad::ConfigError("unknown transport");
    if (cfg->layers < 1) throw cad::ConfigError("layers must be >= 1");
    cad_plan_stats st;
    ok(cad_plan_get_stats(plan, &st), "cad_plan_get_stats");
    if (st.n_servers != cfg->world) throw cad::ConfigError("plan servers != world");
    auto C = std::make_unique<cad_layer_ctx>();
    C->cfg = *cfg;
    cuda_check(cudaGetDevice(&C->device), "cudaGetDevice");
    cad_dev::preload_kernels();
    for (const void* f : {reinterpret_cast<const void*>(copy_row_chunks_kernel),
                          reinterpret_cast<const void*>(copy_col_chunks_kernel),
                          reinterpret_cast<const void*>(reduce_partials_kernel)}) {
      cudaFuncAttributes a;  // loaded now, not mid-step (see preload_kernels)
      cuda_check(cudaFuncGetAttributes(&a, f), "load executor kernels");
    }
    C->W = cfg->world;
    C->me = cfg->rank;
    C->NL = cfg->layers;
    C->hq = cfg->h_q;
    C->hkv = cfg->h_kv;
    C->q_row = C->hq * C->d * 2;
    C->kv_row = C->hkv * C->d * 2;
    C->lse_row = C->hq * 4;
    // every rank's rows: ours in full, the peers' for where our rows land
    std::vector<RankRows> all;
    std::vector<Alias> aliases;
    for (int r = 0; r < C->W; ++r) {
      all.push_back(read_rank(plan, home_items, n_items, r, C->q_row, C->kv_row, cfg->balance_halves));
      aliases.push_back(alias_rows(all.back(), r));  // zero-copy own rows, every rank's view
    }
    C->mine = all[static_cast<size_t>(C->me)];
    C->alias = aliases[static_cast<size_t>(C->me)];
    C->layout = layout_of(C->mine, C->alias, C->NL, C->W, C->q_row, C->kv_row, C->lse_row);
    C->peer.resize(static_cast<size_t>(C->W));
    for (int p = 0; p < C->W; ++p) {
      Peer& P = C->peer[static_cast<size_t>(p)];
      P.home_rows = all[static_cast<size_t>(p)].home_rows;
      for (int h = 0; h < 2; ++h) P.q_pitch[h] = std::max<i64>(1, all[static_cast<size_t>(p)].half[h].q_rows);
      P.layout = layout_of(all[static_cast<size_t>(p)], aliases[static_cast<size_t>(p)], C->NL, C->W, C->q_row,
                           C->kv_row, C->lse_row);
    }
    // own rows that still move as columns: LSE server view -> home, and the
    // forward state's LSE home -> server view
    auto chunk_pairs = [](const std::vector<std::pair<i64, i64>>& pairs, int64_t* n) {
      std::vector<i64> src, dst;
      for (const auto& pr : pairs) {
        src.push_back(pr.first);
        dst.push_back(pr.second);
      }
      std::vector<int64_t> ch;
      for (const cad_run& r : make_runs(src.data(), dst.data(), static_cast<i64>(src.size())))
        for (i64 a = 0; a < r.n_rows; a += kChunkRows) {
          ch.push_back(r.src_row + a);
          ch.push_back(r.dst_row + a);
          ch.push_back(std::min<i64>(kChunkRows, r.n_rows - a));
        }
      *n = static_cast<int64_t>(ch.size() / 3);
      return dev_copy(ch);
    };
    for (int h = 0; h < 2; ++h) {
      C->d_lse_self[h] = chunk_pairs(C->alias.lse_self[h], &C->n_lse_self[h]);
      C->d_qd_self[h] = chunk_pairs(C->alias.qd_self[h], &C->n_qd_self[h]);
    }
    // push runs: my send rows to p against p's receive rows from me
    for (int h = 0; h < 2; ++h)
      for (int x = 0; x < 4; ++x) {
        const XferRows& M = C->mine.half[h].x[x];
        auto& R = C->runs[h][x];
        auto& off = C->run_off[h][x];
        off.assign(1, 0);
        i64 so = 0;
        for (int p = 0; p < C->W; ++p) {
          const XferRows& PX = all[static_cast<size_t>(p)].half[h].x[x];
          i64 ro = 0;
          for (int q = 0; q < C->me; ++q) ro += PX.recv_counts[static_cast<size_t>(q)];
          const i64 n = M.send_counts[static_cast<size_t>(p)];
          if (PX.recv_counts[static_cast<size_t>(C->me)] != n) throw cad::DomainError("row plans disagree");
          std::vector<i64> dst(static_cast<size_t>(n));
          for (i64 i = 0; i < n; ++i)
            dst[static_cast<size_t>(i)] = x == kXKR ? ro + i : PX.recv_idx[static_cast<size_t>(ro + i)];
          const auto rr = make_runs(M.send_idx.data() + so, dst.data(), n);
          R.insert(R.end(), rr.begin(), rr.end());
          off.push_back(R.size());
          so += n;
          if (p == C->me) {
            std::vector<int64_t> ch;
            for (const cad_run& r : rr)
              for (i64 a = 0; a < r.n_rows; a += kChunkRows) {
                ch.push_back(r.src_row + a);
                ch.push_back(r.dst_row + a);
                ch.push_back(std::min<i64>(kChunkRows, r.n_rows - a));
              }
            C->n_local_chunks[h][x] = static_cast<int64_t>(ch.size() / 3);
            C->d_local_chunks[h][x] = dev_copy(ch);
          }
        }
      }
    // own dK/dV partial rows: server row (in my KV_RET send list to myself) of
    // the j-th staging row I receive from myself
    std::vector<i64> own_src[2];
    for (int h = 0; h < 2; ++h) {
      const XferRows& M = C->mine.half[h].x[kXKR];
      i64 so = 0;
      for (int p = 0; p < C->me; ++p) so += M.send_counts[static_cast<size_t>(p)];
      own_src[h].assign(M.send_idx.begin() + so, M.send_idx.begin() + so + M.send_counts[static_cast<size_t>(C->me)]);
    }
    all.clear();
    // server CA plans and workspaces
    size_t xmax = 16;
    for (int h = 0; h < 2; ++h) {
      const HalfRows& H = C->mine.half[h];
      for (const cad_ca_task& t : H.tasks) C->pairs += cad_causal_pairs(t.n_q, t.kv_len);
      for (int x = 0; x < 4; ++x) {
        if (cfg->transport == CAD_TRANSPORT_NCCL) {
          const XferRows& X = H.x[x];
          cad_layer_ctx::NcclX& N = C->nx[h][x];
          std::vector<i64> si, ri;
          i64 so = 0, ro = 0;
          for (int p = 0; p < C->W; ++p) {
            const size_t q = static_cast<size_t>(p);
            const i64 ns = X.send_counts[q], nr = X.recv_counts[q];
            N.rd_full.push_back(ro);
            if (p != C->me) {
              si.insert(si.end(), X.send_idx.begin() + so, X.send_idx.begin() + so + ns);
              ri.insert(ri.end(), X.recv_idx.begin() + ro, X.recv_idx.begin() + ro + nr);
            }
            N.sc.push_back(p == C->me ? 0 : ns);
            N.rc.push_back(p == C->me ? 0 : nr);
            so += ns;
            ro += nr;
          }
          N.n_send = static_cast<i64>(si.size());
          N.n_recv = static_cast<i64>(ri.size());
          N.d_send = dev_copy(si);
          N.d_recv = dev_copy(ri);
        }
        xmax = std::max(xmax, static_cast<size_t>(std::max(H.x[x].n_send(), H.x[x].n_recv()) * C->q_row));
      }
      if (H.tasks.empty()) continue;
      cad_ca_shape sh{};
      sh.h_q = cfg->h_q;
      sh.h_kv = cfg->h_kv;
      sh.head_dim = 128;
      sh.softmax_scale = cfg->softmax_scale;
      sh.q_rows = std::max<i64>(1, H.q_rows);
      sh.kv_rows = std::max<i64>(1, H.kv_rows);
      ok(cad_ca_plan_create(H.tasks.data(), static_cast<i64>(H.tasks.size()), &sh, &C->plan[h]), "cad_ca_plan_create");
      if (cfg->reserve_sms > 0) {
        int sms = 148;
        cuda_check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, C->device), "sm count");
        ok(cad_ca_plan_set_max_ctas(C->plan[h], std::max(2, sms - cfg->reserve_sms)), "set_max_ctas");
      }
      cad_ca_plan_info info;
      ok(cad_ca_plan_info_get(C->plan[h], &info), "cad_ca_plan_info_get");
      C->ws_bytes[h] = std::max<size_t>(16, info.workspace_bytes);
      cuda_check(cudaMalloc(&C->ws[h], C->ws_bytes[h]), "cudaMalloc(workspace)");
    }
    cuda_check(cudaMalloc(reinterpret_cast<void**>(&C->arena), C->layout.total), "cudaMalloc(server buffers)");
    C->flags = C->at<int32_t>(C->layout.flags);
    cuda_check(cudaMemset(C->flags, 0, static_cast<size_t>(4) * 2 * kKinds * C->W), "memset flags");
    {  // dK/dV reduction CSR: home row -> (half, staging row) of every partial
      std::vector<std::vector<int32_t>> per(static_cast<size_t>(std::max<i64>(1, C->mine.home_rows)));
      for (int h = 0; h < 2; ++h) {
        const XferRows& X = C->mine.half[h].x[kXKR];
        const auto& ri = X.recv_idx;
        if (static_cast<i64>(ri.size()) >= (i64(1) << 29) || C->mine.half[h].kv_rows >= (i64(1) << 29))
          throw cad::ConfigError("too many partial rows");
        i64 own0 = 0;
        for (int p = 0; p < C->me; ++p) own0 += X.recv_counts[static_cast<size_t>(p)];
        const i64 own1 = own0 + X.recv_counts[static_cast<size_t>(C->me)];
        for (size_t j = 0; j < ri.size(); ++j) {
          const i64 jj = static_cast<i64>(j);
          const bool own = jj >= own0 && jj < own1;  // my own partial: read in my server buffer
          const i64 row = own ? own_src[h][static_cast<size_t>(jj - own0)] : jj;
          per[static_cast<size_t>(ri[j])].push_back(static_cast<int32_t>(row << 2 | (own ? 2 : 0) | h));
        }
      }
      std::vector<int64_t> off(1, 0);
      std::vector<int32_t> ent;
      for (const auto& v : per) {
        ent.insert(ent.end(), v.begin(), v.end());
        off.push_back(static_cast<int64_t>(ent.size()));
      }
      C->d_red_off = dev_copy(off);
      C->d_red_ent = dev_copy(ent);
      for (int t = 0; t < 2; ++t) {
        std::vector<const uint4*> src;
        for (int l = 0; l < C->NL; ++l)
          for (int own = 0; own < 2; ++own)
            for (int h = 0; h < 2; ++h) {
              const Bufs& B = C->b(l, h);
              src.push_back(C->at<const uint4>(own ? (t == 0 ? B.dk : B.dv) : (t == 0 ? B.sdk : B.sdv)));
            }
        C->d_red_src[t] = dev_copy(src);
      }
    }
    if (cfg->transport == CAD_TRANSPORT_NCCL) {
      C->xbytes = xmax;
      cuda_check(cudaMalloc(&C->xsend, xmax), "cudaMalloc(send)");
      cuda_check(cudaMalloc(&C->xrecv, xmax), "cudaMalloc(recv)");
    }
    cuda_check(cudaStreamCreateWithFlags(&C->comm_stream, cudaStreamNonBlocking), "cudaStreamCreate");
    if (const char* e = std::getenv("CAD_PUSH_LANES")) {
      const int k = std::atoi(e);
      for (int i = 0; k > 1 && i < k; ++i) {
        cudaStream_t st;
        cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate(lane)");
        C->lanes.push_back(st);
      }
      C->lane_ev.resize(C->lanes.empty() ? 0 : C->lanes.size() + 1);
      for (cudaEvent_t& ev : C->lane_ev)
        cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate(lane)");
    }
    C->ev.resize(static_cast<size_t>(2 + 8 * C->NL));
    for (cudaEvent_t& e : C->ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
    *out = C.release();
  });
}

int cad_layer_ctx_info_get(const cad_layer_ctx* ctx, cad_layer_ctx_info* info) {
  return cad::guarded([&] {
    if (!ctx || !info) throw cad::DomainError("null argument");
    *info = cad_layer_ctx_info{};
    info->home_rows = ctx->mine.home_rows;
    for (int h = 0; h < 2; ++h) {
      info->q_rows[h] = ctx->mine.half[h].q_rows;
      info->kv_rows[h] = ctx->mine.half[h].kv_rows;
      info->n_tasks[h] = static_cast<int64_t>(ctx->mine.half[h].tasks.size());
      for (int x = 0; x < 4; ++x) info->wire_bytes[h][x] = ctx->mine.half[h].wire[x];
    }
    info->served_pairs = ctx->pairs;
    info->blob_bytes = sizeof(Blob);
    info->launches = ctx->launches;
  });
}

int cad_layer_ctx_bind_outputs(cad_layer_ctx* ctx, void* o, float* lse, void* dq) {
  // The home outputs live in the context (cad_layer_ctx_home); caller buffers
  // in cad_layer_io receive copies. Kept for callers of the earlier contract.
  return cad::guarded([&] {
    if (!ctx || !o || !lse || !dq) throw cad::DomainError("null argument");
  });
}

int cad_layer_ctx_home(const cad_layer_ctx* ctx, int32_t layer, cad_layer_io* io) {
  return cad::guarded([&] {
    if (!ctx || !io) throw cad::DomainError("null argument");
    if (layer < 0 || layer >= ctx->NL) throw cad::DomainError("layer out of range");
    const Homes& H = ctx->hm(layer);
    *io = cad_layer_io{};
    io->q = ctx->at(H.q);
    io->k = ctx->at(H.k);
    io->v = ctx->at(H.v);
    io->dout = ctx->at(H.dout);
    io->o = ctx->at(H.o);
    io->lse = ctx->at<float>(H.lse);
    io->dq = ctx->at(H.dq);
  });
}

int cad_layer_ctx_export(cad_layer_ctx* ctx, void* blob, size_t cap, size_t* need) {
  return cad::guarded([&] {
    if (!ctx || !need) throw cad::DomainError("null argument");
    *need = sizeof(Blob);
    if (!blob || cap < sizeof(Blob)) throw cad::CapacityError("blob buffer too small");
    if (ctx->cfg.transport == CAD_TRANSPORT_NCCL) throw cad::ConfigError("NCCL transport has nothing to export");
    cad_dev::DeviceGuard dg(ctx->device);
    Blob B{};
    B.magic = kBlobMagic;
    B.rank = ctx->me;
    B.world = ctx->W;
    B.transport = ctx->cfg.transport;
    B.layers = ctx->NL;
    B.home_rows = ctx->mine.home_rows;
    B.ref[0].raw = reinterpret_cast<uint64_t>(ctx->arena);  // every buffer a peer writes is in the arena
    if (ctx->cfg.transport == CAD_TRANSPORT_IPC) ok(cad_ipc_handle(ctx->arena, B.ref[0].handle, &B.ref[0].offset), "ipc");
    std::memcpy(blob, &B, sizeof(B));
  });
}

int cad_layer_ctx_connect(cad_layer_ctx* ctx, const void* blobs, size_t blob_bytes) {
  return cad::guarded([&] {
    if (!ctx || !blobs) throw cad::DomainError("null argument");
    if (ctx->cfg.transport == CAD_TRANSPORT_NCCL) throw cad::ConfigError("NCCL transport: use cad_layer_ctx_set_comm");
    if (blob_bytes != sizeof(Blob)) throw cad::DomainError("blob size mismatch");
    if (ctx->connected) throw cad::ConfigError("already connected");
    cad_dev::DeviceGuard dg(ctx->device);
    for (int p = 0; p < ctx->W; ++p) {
      Blob B;
      std::memcpy(&B, static_cast<const char*>(blobs) + static_cast<size_t>(p) * sizeof(Blob), sizeof(Blob));
      if (B.magic != kBlobMagic || B.rank != p || B.world != ctx->W || B.layers != ctx->NL ||
          B.transport != ctx->cfg.transport)
        throw cad::DomainError("blob of rank " + std::to_string(p) + " does not match this context");
      Peer& P = ctx->peer[static_cast<size_t>(p)];
      if (B.home_rows != P.home_rows) throw cad::DomainError("peer home rows disagree with the row plan");
      if (p == ctx->me || ctx->cfg.transport == CAD_TRANSPORT_LOCAL) {
        P.arena = reinterpret_cast<char*>(B.ref[0].raw);
        continue;
      }
      void* base = nullptr;
      ok(cad_ipc_open(B.ref[0].handle, &base), "cad_ipc_open");
      ctx->opened.push_back(base);
      P.arena = static_cast<char*>(base) + B.ref[0].offset;
    }
    ctx->connected = true;
  });
}

int cad_layer_ctx_set_comm(cad_layer_ctx* ctx, cad_comm* comm) {
  return cad::guarded([&] {
    if (!ctx || !comm) throw cad::DomainError("null argument");
    if (ctx->cfg.transport != CAD_TRANSPORT_NCCL) throw cad::ConfigError("not an NCCL-transport context");
    ctx->comm = comm;
  });
}

int cad_layer_ctx_destroy(cad_layer_ctx* ctx) {
  return cad::guarded([&] {
    if (!ctx) return;
    cad_dev::DeviceGuard dg(ctx->device);
    delete ctx;
  });
}

int cad_layer_begin(cad_layer_ctx* ctx, void* stream) {
  return cad_layer_begin_ex(ctx, CAD_PASS_BOTH, stream);
}

int cad_layer_begin_ex(cad_layer_ctx* ctx, int32_t passes, void* stream) {
  return cad::guarded([&] {
    if (!ctx) throw cad::DomainError("null argument");
    cad_dev::DeviceGuard dg(ctx->device);
    ctx->begin(static_cast<cudaStream_t>(stream), passes);
  });
}

int cad_dispatch(cad_layer_ctx* ctx, int32_t layer, int32_t half, int32_t what, const cad_layer_io* io, void* stream) {
  return cad_dispatch_ex(ctx, layer, half, what, io, stream, stream);
}

int cad_dispatch_ex(cad_layer_ctx* ctx, int32_t layer, int32_t half, int32_t what, const cad_layer_io* io,
                    void* stream, void* local_stream) {
  return cad::guarded([&] {
    if (!ctx) throw cad::DomainError("null argument");
    ctx->check_lh(layer, half);
    ctx->check_io(io, false);
    ctx->need_ready();
    cad_dev::DeviceGuard dg(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (half == 0) {  // the caller's buffers into the layer's home regions, once per layer
      const i64 H = ctx->mine.home_rows;
      if (what == CAD_DISPATCH_QKV) {
        ctx->stage(ctx->at(ctx->hm(layer).q), io->q, H * ctx->q_row, s);
        ctx->stage(ctx->at(ctx->hm(layer).k), io->k, H * ctx->kv_row, s);
        ctx->stage(ctx->at(ctx->hm(layer).v), io->v, H * ctx->kv_row, s);
      } else if (what == CAD_DISPATCH_DO) {
        ctx->stage(ctx->at(ctx->hm(layer).dout), io->dout, H * ctx->q_row, s);
      } else if (what == CAD_DISPATCH_FWD_STATE) {
        ctx->stage_fwd_state(io, layer, s);
      }
      if (static_cast<cudaStream_t>(local_stream) != s) {  // own rows read on local_stream
        cuda_check(cudaEventRecord(ctx->event(0), s), "event");
        cuda_check(cudaStreamWaitEvent(static_cast<cudaStream_t>(local_stream), ctx->event(0), 0), "wait");
      }
    }
    ctx->dispatch(layer, half, what, io, s, static_cast<cudaStream_t>(local_stream));
  });
}

int cad_layer_compute(cad_layer_ctx* ctx, int32_t layer, int32_t half, int32_t backward, void* stream) {
  return cad::guarded([&] {
    if (!ctx) throw cad::DomainError("null argument");
    ctx->check_lh(layer, half);
    ctx->need_ready();
    cad_dev::DeviceGuard dg(ctx->device);
    ctx->compute(layer, half, backward != 0, static_cast<cudaStream_t>(stream), true, true);
  });
}

int cad_return(cad_layer_ctx* ctx, int32_t layer, int32_t half, int32_t what, const cad_layer_io* io, void* stream) {
  return cad::guarded([&] {
    if (!ctx) throw cad::DomainError("null argument");
    ctx->check_lh(layer, half);
    ctx->check_io(io, true);
    ctx->need_ready();
    cad_dev::DeviceGuard dg(ctx->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ctx->ret(layer, half, what, io, s, s);
  });
}

int cad_layer_finish(cad_layer_ctx* ctx, const cad_layer_io* io, void* stream) {
  return cad::guarded([&] {
    if (!ctx) throw cad::DomainError("null argument");
    ctx->check_io(io, false);
    ctx->need_ready();
    cad_dev::DeviceGuard dg(ctx->device);
    ctx->finish(io, static_cast<cudaStream_t>(stream));
  });
}

int cad_layer_ctx_set_trace(cad_layer_ctx* ctx, int32_t on) {
  return cad::guarded([&] {
    if (!ctx) throw cad::DomainError("null argument");
    ctx->tracing = on != 0;
  });
}

int cad_layer_ctx_trace(cad_layer_ctx* ctx, cad_trace_rec* recs, int64_t cap, int64_t* n) {
  return cad::guarded([&] {
    if (!ctx || !n) throw cad::DomainError("null argument");
    cad_dev::DeviceGuard dg(ctx->device);
    *n = static_cast<int64_t>(ctx->trows.size());
    if (cap < *n || (*n > 0 && !recs)) throw cad::CapacityError("trace buffer too small");
    if (*n > 0) cuda_check(cudaEventSynchronize(ctx->tev[ctx->tused - 1]), "trace sync");
    auto at = [&](int m) {
      float ms = 0.0f;
      if (m >= 0) cuda_check(cudaEventElapsedTime(&ms, ctx->tev[0], ctx->tev[static_cast<size_t>(m)]), "elapsed");
      return ms;
    };
    for (size_t i = 0; i < ctx->trows.size(); ++i) {
      const auto& r = ctx->trows[i];
      recs[i] = cad_trace_rec{r.kind, r.layer, r.half, 0, at(r.m0), at(r.m1), at(r.m2), 0.0f};
    }
  });
}

int cad_layer_step(cad_layer_ctx* ctx, const cad_layer_io* io, int32_t mode, void* stream) {
  return cad_layer_step_ex(ctx, io, mode, CAD_PASS_BOTH, stream);
}

int cad_layer_step_ex(cad_layer_ctx* ctx, const cad_layer_io* io, int32_t mode, int32_t passes, void* stream) {
  return cad::guarded([&] {
    if (!ctx) throw cad::DomainError("null argument");
    if (passes < CAD_PASS_FWD || passes > CAD_PASS_BOTH) throw cad::DomainError("passes must be FWD, BWD or BOTH");
    if (passes != CAD_PASS_BOTH && ctx->NL != 1) throw cad::ConfigError("single-pass steps need layers == 1");
    cad_dev::DeviceGuard dg(ctx->device);
    ctx->step(io, mode, static_cast<cudaStream_t>(stream), passes);
  });
}

}  // extern "C"
