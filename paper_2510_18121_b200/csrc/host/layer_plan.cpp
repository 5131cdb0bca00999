// Per-rank data movement of one CA layer: the real counterpart of the
// reference's per-device served/sent lists and ping-pong windows
// (device_plans_from_schedule / assign_halves / layer_windows,
// P/src/sim.cpp:34-46,69-157), which only count bytes.
//
// Buffers of rank r:
//   home   Q/K/V/O/dO/dQ/dK/dV rows of r's chunk (place_sequential: tokens
//          [r*T/G, (r+1)*T/G) of the concatenated documents), in item order.
//   server for each half h (ping/pong), the CA-tasks r serves in h:
//          Q rows packed task by task (server order), and one KV group per
//          document holding rows [0, need) where need = max kv_extent of the
//          half's tasks of that document -- KV is shipped once per
//          (document, server, half) and only the rows the server does not
//          already hold are sent over the wire (residency-aware, deduplicated:
//          SURVEY.md 8f next #1; the reference charges the full prefix per
//          remote task and nothing for home-served straddling documents,
//          P/src/scheduler.cpp:342-345).
// head_tail items (per-document CP layouts, P/include/cadsim/types.hpp:101-111)
// are served as two CA-tasks sharing the document's KV group: the head
// [q_begin, q_end) over keys [0, q_end) and the tail
// [M - q_end, M - q_begin) over keys [0, M - q_begin), M = ht_mirror (the
// reference's two sub-calls, P/src/sim.cpp:22-30, P/src/cost.cpp:40-43). A
// head_tail home item holds its head rows, then its tail rows (the chunk
// segment order of P/src/experiment.cpp:120-130).
// Exchanges (per half, row granularity, every rank including itself):
//   QD  Q (and dO in backward) home -> server     KVD K/V home -> server
//   OR  O/LSE (and dQ in backward) server -> home  KVR dK/dV server -> owner
//       (partials of one row from several servers are summed at the owner).
#include <algorithm>
#include <cmath>
#include <map>
#include <memory>
#include <vector>

#include "../../../include/cad.h"
#include "cad_host.hpp"
#include "cad_status.hpp"

struct cad_plan;  // opaque (capi_host.cpp)
const cad::Plan& cad_plan_ref(const cad_plan* p);
const std::vector<cad::DevicePlan>& cad_plan_devices(const cad_plan* p);

namespace {

using cad::i64;

// Owner map of one document: token ranges per home device with home rows.
struct Seg {
  i64 begin, end;  // document positions
  int32_t device;
  i64 home_row;  // row of `begin` in the device's home buffers
};

struct Xfer {  // one exchange as seen by one rank
  std::vector<i64> send_counts, send_idx, recv_counts, recv_idx;
};

struct Half {
  std::vector<cad_ca_task> tasks;
  std::vector<i64> task_index;  // plan task of each server task
  i64 q_rows = 0, kv_rows = 0;
  Xfer x[4];
  i64 remote_bytes[4] = {0, 0, 0, 0};
};

}  // namespace

struct cad_layer_plan {
  int32_t rank = 0, world = 1;
  i64 home_rows = 0;
  Half half[2];
};

namespace {

const Seg& owner_of(const std::vector<Seg>& segs, i64 pos) {
  // segments are sorted by begin
  auto it = std::upper_bound(segs.begin(), segs.end(), pos,
                             [](i64 p, const Seg& s) { return p < s.begin; });
  if (it == segs.begin()) throw cad::DomainError("position before the first segment");
  --it;
  if (pos >= it->end) throw cad::DomainError("position not owned by any device");
  return *it;
}

// Emits rows [a, b) of document `doc` from their owners into a transfer
// whose destination rows start at dst_row, for server `server`.
struct Builder {
  int32_t world;
  // per (src device, dst device): list of (src_row, dst_row)
  std::vector<std::vector<std::vector<std::pair<i64, i64>>>> pairs;
  explicit Builder(int32_t w) : world(w), pairs(w, std::vector<std::vector<std::pair<i64, i64>>>(w)) {}
  void add(int32_t src, int32_t dst, i64 src_row, i64 dst_row) {
    pairs[static_cast<size_t>(src)][static_cast<size_t>(dst)].push_back({src_row, dst_row});
  }
  // The view of `rank`: sends (src == rank) grouped by dst, receives
  // (dst == rank) grouped by src, both in emission order.
  Xfer view(int32_t rank) const {
    Xfer x;
    for (int32_t p = 0; p < world; ++p) {
      const auto& out = pairs[static_cast<size_t>(rank)][static_cast<size_t>(p)];
      x.send_counts.push_back(static_cast<i64>(out.size()));
      for (const auto& e : out) x.send_idx.push_back(e.first);
      const auto& in = pairs[static_cast<size_t>(p)][static_cast<size_t>(rank)];
      x.recv_counts.push_back(static_cast<i64>(in.size()));
      for (const auto& e : in) x.recv_idx.push_back(e.second);
    }
    return x;
  }
  i64 remote_rows(int32_t rank, bool as_sender) const {
    i64 n = 0;
    for (int32_t p = 0; p < world; ++p) {
      if (p == rank) continue;
      n += static_cast<i64>(as_sender ? pairs[static_cast<size_t>(rank)][static_cast<size_t>(p)].size()
                                      : pairs[static_cast<size_t>(p)][static_cast<size_t>(rank)].size());
    }
    return n;
  }
};

// One CA-task as served: query positions [qb, qe) of a plan task's document
// over keys [0, kv) (kv = qe for contiguous items), in half `half`.
struct Part {
  i64 task, qb, qe, kv;
  int half;
  bool splittable;  // contiguous item part (head_tail parts keep the reference's pairing)
};

i64 part_pairs(const Part& p) { return cad::causal_pairs(p.qe - p.qb, p.kv); }

// The CA-tasks of server s: the reference's served list and halves
// (assign_halves, P/src/sim.cpp:34-46) -- and, with `balance`, the halves
// evened out in causal pairs by moving the query tail of the heavier half's
// largest contiguous task (a query shard with its causal prefix is itself a
// CA-task) to the lighter half. The reference balances cores per server but
// not per half; the halves of one server can differ several-fold (one long
// document), and every half of every rank waits for its peers' previous
// returns, so the per-half maximum over ranks sets the step time.
std::vector<Part> server_parts(const cad::Plan& P, const cad::DevicePlan& dev, int balance) {
  std::vector<Part> parts;
  for (const cad::Served& sv : dev.served) {
    const cad::Item& it = P.tasks[static_cast<size_t>(sv.task)].item;
    const bool ht = it.layout == cad::Layout::head_tail;
    // balance 2: one half (every task in the ping half; the pong half is empty)
    const int half = balance == 2 ? 0 : sv.half;
    parts.push_back({sv.task, it.q_begin, it.q_end, it.q_end, half, !ht});
    if (ht) parts.push_back({sv.task, it.ht_mirror - it.q_end, it.ht_mirror - it.q_begin,
                             it.ht_mirror - it.q_begin, half, false});
  }
  if (balance != 1) return parts;
  for (int round = 0; round < 4; ++round) {
    i64 load[2] = {0, 0};
    for (const Part& p : parts) load[p.half] += part_pairs(p);
    const int heavy = load[1] > load[0] ? 1 : 0;
    const i64 delta = (load[heavy] - load[1 - heavy]) / 2;
    if (delta <= (load[0] + load[1]) / 200) break;  // within 1 %
    int best = -1;
    for (size_t i = 0; i < parts.size(); ++i)
      if (parts[i].half == heavy && parts[i].splittable &&
          (best < 0 || part_pairs(parts[i]) > part_pairs(parts[static_cast<size_t>(best)])))
        best = static_cast<int>(i);
    if (best < 0) break;
    Part& b = parts[static_cast<size_t>(best)];
    if (part_pairs(b) <= delta) {
      b.half = 1 - heavy;
      continue;
    }
    // c with pairs of queries [c, qe) ~ delta: sum_{p=c}^{qe-1} (p+1) =
    // (qe(qe+1) - c(c+1)) / 2, c rounded to a 128-row tile of the task
    const double t = double(b.qe) * double(b.qe + 1) - 2.0 * double(delta);
    i64 c = static_cast<i64>(std::sqrt(std::max(0.0, t)));
    c = b.qb + (c - b.qb + 64) / 128 * 128;
    if (c <= b.qb || c >= b.qe) break;
    Part tail = b;
    tail.qb = c;
    tail.half = 1 - heavy;
    b.qe = c;
    b.kv = c;
    parts.push_back(tail);
  }
  return parts;
}

}  // namespace

extern "C" {

int cad_layer_plan_create(const cad_plan* plan, const cad_item* home_items, int64_t n_items,
                          int32_t rank, int64_t q_row_bytes, int64_t kv_row_bytes,
                          cad_layer_plan** out) {
  return cad_layer_plan_create_ex(plan, home_items, n_items, rank, q_row_bytes, kv_row_bytes, 0, out);
}

int cad_layer_plan_create_ex(const cad_plan* plan, const cad_item* home_items, int64_t n_items,
                             int32_t rank, int64_t q_row_bytes, int64_t kv_row_bytes, int32_t balance,
                             cad_layer_plan** out) {
  return cad::guarded([&] {
    if (!plan || !out || (n_items > 0 && !home_items)) throw cad::DomainError("null argument");
    *out = nullptr;
    const cad::Plan& P = cad_plan_ref(plan);
    const auto& devs = cad_plan_devices(plan);
    const int32_t world = static_cast<int32_t>(P.servers.size());
    if (rank < 0 || rank >= world) throw cad::DomainError("rank out of range");
    // Token ownership from the pre-schedule home items (chunk order).
    std::map<i64, std::vector<Seg>> owners;
    std::vector<i64> rows_of(static_cast<size_t>(world), 0);
    for (int64_t i = 0; i < n_items; ++i) {
      const cad_item& it = home_items[i];
      if (it.home_device < 0 || it.home_device >= world) throw cad::DomainError("home device out of range");
      i64& r = rows_of[static_cast<size_t>(it.home_device)];
      owners[it.doc].push_back({it.q_begin, it.q_end, it.home_device, r});
      r += it.q_end - it.q_begin;
      if (it.layout == CAD_LAYOUT_HEAD_TAIL) {
        owners[it.doc].push_back({it.ht_mirror - it.q_end, it.ht_mirror - it.q_begin, it.home_device, r});
        r += it.q_end - it.q_begin;
      }
    }
    for (auto& kv : owners)
      std::sort(kv.second.begin(), kv.second.end(), [](const Seg& a, const Seg& b) { return a.begin < b.begin; });

    auto L = std::make_unique<cad_layer_plan>();
    L->rank = rank;
    L->world = world;
    L->home_rows = rows_of[static_cast<size_t>(rank)];
    std::vector<std::vector<Part>> parts_of;
    if (balance < 0 || balance > 2) throw cad::DomainError("balance must be 0, 1 or 2");
    for (int32_t s = 0; s < world; ++s) parts_of.push_back(server_parts(P, devs[static_cast<size_t>(s)], balance));
    for (int h = 0; h < 2; ++h) {
      Builder qd(world), kvd(world);
      std::vector<Half> all(static_cast<size_t>(world));  // server-side layouts of every rank
      for (int32_t s = 0; s < world; ++s) {
        Half& H = all[static_cast<size_t>(s)];
        std::map<i64, std::pair<i64, i64>> group;  // doc -> (kv_off, need)
        std::vector<i64> doc_order;
        // KV need per document over this half's tasks
        for (const Part& pt : parts_of[static_cast<size_t>(s)]) {
          if (pt.half != h) continue;
          const cad::Item& it = P.tasks[static_cast<size_t>(pt.task)].item;
          const i64 need = pt.kv;
          auto g = group.find(it.doc);
          if (g == group.end()) {
            group[it.doc] = {0, need};
            doc_order.push_back(it.doc);
          } else {
            g->second.second = std::max(g->second.second, need);
          }
        }
        i64 kv_off = 0;
        for (i64 d : doc_order) {
          group[d].first = kv_off;
          kv_off += group[d].second;
        }
        H.kv_rows = kv_off;
        for (const Part& pt : parts_of[static_cast<size_t>(s)]) {
          if (pt.half != h) continue;
          const cad::Item& it = P.tasks[static_cast<size_t>(pt.task)].item;
          const auto& segs = owners.at(it.doc);
          const i64 qb = pt.qb, qe = pt.qe;
          cad_ca_task ct;
          ct.q_off = H.q_rows;
          ct.n_q = qe - qb;
          ct.kv_off = group[it.doc].first;
          ct.kv_len = pt.kv;
          H.tasks.push_back(ct);
          H.task_index.push_back(pt.task);
          // Q rows come from the task's home device
          for (i64 pos = qb; pos < qe; ++pos) {
            const Seg& o = owner_of(segs, pos);
            if (o.device != it.home) throw cad::DomainError("task rows not on its home device");
            qd.add(o.device, s, o.home_row + (pos - o.begin), H.q_rows + (pos - qb));
          }
          H.q_rows += qe - qb;
        }
        for (i64 d : doc_order) {
          const auto& segs = owners.at(d);
          const i64 off = group[d].first, need = group[d].second;
          for (const Seg& o : segs) {
            const i64 a = std::max<i64>(o.begin, 0), b = std::min(o.end, need);
            for (i64 pos = a; pos < b; ++pos) kvd.add(o.device, s, o.home_row + (pos - o.begin), off + pos);
          }
        }
      }
      Half& mine = L->half[h];
      mine = all[static_cast<size_t>(rank)];
      mine.x[0] = qd.view(rank);
      mine.x[1] = kvd.view(rank);
      // Return paths are the transposes: server rows back to the owners.
      Xfer& ret_q = mine.x[2];
      Xfer& ret_kv = mine.x[3];
      const Xfer q_all = qd.view(rank), kv_all = kvd.view(rank);
      ret_q.send_counts = q_all.recv_counts;
      ret_q.send_idx = q_all.recv_idx;
      ret_q.recv_counts = q_all.send_counts;
      ret_q.recv_idx = q_all.send_idx;
      ret_kv.send_counts = kv_all.recv_counts;
      ret_kv.send_idx = kv_all.recv_idx;
      ret_kv.recv_counts = kv_all.send_counts;
      ret_kv.recv_idx = kv_all.send_idx;
      mine.remote_bytes[0] = qd.remote_rows(rank, true) * q_row_bytes;
      mine.remote_bytes[1] = kvd.remote_rows(rank, true) * kv_row_bytes;
      mine.remote_bytes[2] = qd.remote_rows(rank, false) * q_row_bytes;
      mine.remote_bytes[3] = kvd.remote_rows(rank, false) * kv_row_bytes;
    }
    *out = L.release();
  });
}

int cad_layer_plan_info(const cad_layer_plan* lp, int32_t half, cad_layer_half_info* info) {
  return cad::guarded([&] {
    if (!lp || !info || half < 0 || half > 1) throw cad::DomainError("bad argument");
    const Half& H = lp->half[half];
    info->home_rows = lp->home_rows;
    info->q_rows = H.q_rows;
    info->kv_rows = H.kv_rows;
    info->n_tasks = static_cast<int64_t>(H.tasks.size());
    info->tasks = H.tasks.data();
    info->task_index = H.task_index.data();
    for (int k = 0; k < 4; ++k) info->remote_send_bytes[k] = H.remote_bytes[k];
  });
}

int cad_layer_plan_xfer(const cad_layer_plan* lp, int32_t half, int32_t which, cad_xfer* x) {
  return cad::guarded([&] {
    if (!lp || !x || half < 0 || half > 1 || which < 0 || which > 3) throw cad::DomainError("bad argument");
    const Xfer& X = lp->half[half].x[which];
    x->n_peers = lp->world;
    x->send_counts = X.send_counts.data();
    x->send_idx = X.send_idx.data();
    x->recv_counts = X.recv_counts.data();
    x->recv_idx = X.recv_idx.data();
    i64 ns = 0, nr = 0;
    for (i64 c : X.send_counts) ns += c;
    for (i64 c : X.recv_counts) nr += c;
    x->n_send = ns;
    x->n_recv = nr;
  });
}

void cad_layer_plan_destroy(cad_layer_plan* lp) { delete lp; }

}  // extern "C"
