// Communication-aware greedy CA-task scheduler (DistCA section 4.2).
//
// Bit-exact restatement of the reference scheduler:
//   core_of          P/src/cost.cpp:32-44
//   bytes_of         P/src/scheduler.cpp:53-60 (= shard_bytes, comm.cpp:35-42)
//   target_load      P/src/scheduler.cpp:13-19
//   classify         P/src/scheduler.cpp:21-34
//   one_tile_slack   P/src/scheduler.cpp:36-49
//   v_min_comm       P/src/comm.cpp:75-178
//   propose          P/src/scheduler.cpp:70-194
//   schedule         P/src/scheduler.cpp:196-357
//   schedule_pp_tick P/src/scheduler.cpp:359-373
//   plan_text        P/src/scheduler.cpp:375-385
//   device_plans     P/src/sim.cpp:34-46,129-157
// "Bit-exact" covers the emitted task order, every integer field and the
// IEEE-double loads: the floating-point expressions below are evaluated in
// the reference's operand order and the file is built with -ffp-contract=off.
#include <algorithm>
#include <cmath>
#include <limits>
#include <sstream>
#include <tuple>

#include "cad_host.hpp"

namespace cad {

void check_item(const Item& it) {
  if (it.q_end <= it.q_begin) throw DomainError("item query range is empty");
  if (it.q_begin < 0) throw DomainError("item query range is negative");
  if (it.kv_extent != it.q_end) throw DomainError("item kv_extent must equal q_end");
  if (it.layout == Layout::head_tail && it.ht_mirror < 2 * it.q_end)
    throw DomainError("head_tail halves overlap (ht_mirror < 2*q_end)");
}

i64 core_of(const Item& it) {
  check_item(it);
  const i64 n = it.n_q(), kv = it.kv_extent;
  const i64 head = n * (2 * kv - n);
  if (it.layout == Layout::contiguous) return head;
  const i64 mirror_kv = it.ht_mirror - (kv - n);
  return head + n * (2 * mirror_kv - n);
}

static i64 shard_bytes(Layout layout, i64 n_q, i64 n_kv, i64 sq, i64 skv, i64 mirror,
                       bool double_q) {
  if (layout == Layout::contiguous) return n_q * sq + n_kv * skv;
  return (double_q ? 2 * n_q : n_q) * sq + (mirror - (n_kv - n_q)) * skv;
}

i64 bytes_of(const Item& it, const SchedCfg& cfg) {
  return shard_bytes(it.layout, it.n_q(), it.kv_extent, cfg.size_q, cfg.size_kv, it.ht_mirror,
                     cfg.double_query_ht);
}

double target_load(const std::vector<Item>& items, i64 n_servers, double alpha) {
  if (n_servers < 1) throw DomainError("n_servers must be >= 1");
  i64 total = 0;
  for (const Item& it : items) total += core_of(it);
  return alpha * static_cast<double>(total) / static_cast<double>(n_servers);
}

void classify(const std::vector<double>& loads, double target,
              std::vector<std::pair<std::int32_t, double>>& surplus,
              std::vector<std::pair<std::int32_t, double>>& deficit) {
  surplus.clear();
  deficit.clear();
  for (std::size_t i = 0; i < loads.size(); ++i) {
    const double gap = loads[i] - target;
    if (gap > 0)
      surplus.emplace_back(static_cast<std::int32_t>(i), gap);
    else if (gap < 0)
      deficit.emplace_back(static_cast<std::int32_t>(i), -gap);
  }
  // Largest gap first, lower device id on ties: a strict total order.
  auto by_gap = [](const std::pair<std::int32_t, double>& a,
                   const std::pair<std::int32_t, double>& b) {
    if (a.second != b.second) return a.second > b.second;
    return a.first < b.first;
  };
  std::sort(surplus.begin(), surplus.end(), by_gap);
  std::sort(deficit.begin(), deficit.end(), by_gap);
}

double one_tile_slack(const std::vector<Item>& items, const SchedCfg& cfg) {
  const i64 t = std::max<i64>(1, cfg.tile);
  i64 worst = 0;
  for (const Item& it : items) {
    const i64 c = it.layout == Layout::head_tail ? 2 * t * it.ht_mirror
                                                 : t * (2 * it.kv_extent - t);
    if (c > worst) worst = c;
  }
  return cfg.alpha * static_cast<double>(worst);
}

static inline i64 round_up(i64 x, i64 t) { return t <= 1 ? x : ((x + t - 1) / t) * t; }
static inline i64 round_down(i64 x, i64 t) { return t <= 1 ? x : (x / t) * t; }

// ---------------------------------------------------------------------------
// Minimal-communication shard (P/src/comm.cpp:75-178).

namespace {

struct Probe {
  ShardChoice s;
  bool ok = false;
};

// For a fixed query count, the lowest kv end (tile-aligned unless clipped by
// the box) whose work reaches `need` (P/src/comm.cpp:75-94).
Probe probe_kv(const CommQuery& q, i64 tile, i64 n_q, i64 need) {
  Probe p;
  if (n_q < 1 || n_q > q.L_q) return p;
  const i64 kv_floor = n_q + q.L_kv - q.L_q;
  const i64 kv_need = (need + n_q * n_q + 2 * n_q - 1) / (2 * n_q);
  const i64 kv = std::max(kv_need, kv_floor);
  if (kv > q.L_kv) return p;
  const i64 aligned = std::min(round_up(kv, tile), q.L_kv);
  p.s.n_q = n_q;
  p.s.n_kv = std::max(aligned, kv);
  p.s.core = n_q * (2 * p.s.n_kv - n_q);
  p.s.bytes = shard_bytes(q.layout, n_q, p.s.n_kv, q.size_q, q.size_kv, q.ht_mirror, false);
  p.ok = true;
  return p;
}

}  // namespace

ShardChoice v_min_comm(const CommQuery& q, i64 tile_size) {
  if (q.L_q < 1 || q.L_kv < q.L_q) throw DomainError("v_min_comm: bad extents");
  if (q.size_q < 1 || q.size_kv < 1) throw DomainError("v_min_comm: bad sizes");
  if (!(q.f_item > 0) || !(q.delta_f_max > 0))
    throw DomainError("v_min_comm: flops must be positive");
  if (q.delta_f_max > q.f_item * (1.0 + 1e-12))
    throw DomainError("v_min_comm: delta_f_max exceeds the item's flops");
  if (q.layout == Layout::head_tail && q.ht_mirror < 2 * q.L_kv)
    throw DomainError("v_min_comm: head_tail mirror too small");
  const i64 tile = std::max<i64>(1, tile_size);

  const i64 whole_core = q.L_q * (2 * q.L_kv - q.L_q);
  const double G = static_cast<double>(q.L_q) * static_cast<double>(2 * q.L_kv - q.L_q);
  const double frac = std::min(1.0, q.delta_f_max / q.f_item);
  ShardChoice whole{q.L_q, q.L_kv,
                    shard_bytes(q.layout, q.L_q, q.L_kv, q.size_q, q.size_kv, q.ht_mirror, false),
                    whole_core};
  i64 need = static_cast<i64>(std::ceil(frac * G - 1e-9));
  need = std::clamp<i64>(need, 1, whole_core);
  if (need >= whole_core) return whole;

  // Continuous feasible range of the query count for the kv box, and the
  // closed-form byte optimum (boundary optimum for head_tail).
  const double Lkv = static_cast<double>(q.L_kv);
  const double gap = static_cast<double>(q.L_kv - q.L_q);
  const double lo = Lkv - std::sqrt(std::max(0.0, Lkv * Lkv - frac * G));
  const double hi = -gap + std::sqrt(gap * gap + frac * G);
  double opt = lo;
  if (q.layout == Layout::contiguous) {
    const double beta = static_cast<double>(q.size_kv) / static_cast<double>(q.size_q);
    opt = std::sqrt(frac * beta * G / (beta + 2.0));
  }
  const double x = std::clamp(opt, lo, hi);
  const i64 up = round_up(static_cast<i64>(std::ceil(x)), tile);
  const i64 cands[6] = {round_down(static_cast<i64>(x), tile),
                        up,
                        up + tile,
                        round_up(static_cast<i64>(std::ceil(lo)), tile),
                        round_down(static_cast<i64>(hi), tile),
                        q.L_q};
  Probe best;
  for (i64 n : cands) {
    if (n < 1 || n > q.L_q) continue;
    if (n != q.L_q && n % tile != 0) continue;
    const Probe c = probe_kv(q, tile, n, need);
    if (!c.ok) continue;
    bool take = !best.ok;
    if (!take) {
      const i64 over_c = c.s.core - need, over_b = best.s.core - need;
      take = c.s.bytes < best.s.bytes ||
             (c.s.bytes == best.s.bytes &&
              (over_c < over_b || (over_c == over_b && c.s.n_q < best.s.n_q)));
    }
    if (take) best = c;
  }
  return best.ok ? best.s : whole;
}

// ---------------------------------------------------------------------------
// One candidate move (P/src/scheduler.cpp:70-194).

namespace {

// Cut `it` so the shard holds queries [n_kv - n_q, n_kv); what is left of the
// query range stays as up to two items (prefix first, then suffix).
void cut(const Item& it, i64 n_q, i64 n_kv, Item& shard, std::vector<Item>& rest) {
  const i64 lo = n_kv - n_q, hi = n_kv;
  shard = it;
  shard.q_begin = lo;
  shard.q_end = hi;
  shard.kv_extent = hi;
  rest.clear();
  if (lo > it.q_begin) {
    Item pre = it;
    pre.q_end = lo;
    pre.kv_extent = lo;
    rest.push_back(pre);
  }
  if (hi < it.q_end) {
    Item post = it;
    post.q_begin = hi;
    rest.push_back(post);
  }
}

// Smallest shard a split can mint (P/src/scheduler.cpp:94-101).
i64 smallest_shard_core(const Item& it, i64 t) {
  const i64 kv = it.q_begin + t;
  i64 c = t * (2 * kv - t);
  if (it.layout == Layout::head_tail) c += t * (2 * (it.ht_mirror - (kv - t)) - t);
  return c;
}

}  // namespace

bool propose(const Server& src, const Server& dst, const Item& item, double target,
             const SchedCfg& cfg, Proposal& p) {
  const double surplus = src.flops - target;
  const double deficit = target - dst.flops;
  if (!(surplus > 0) || !(deficit > 0)) return false;
  const double f_item = cfg.alpha * static_cast<double>(core_of(item));
  const double delta = std::min({f_item, surplus, deficit});
  if (!(delta > 0)) return false;

  const bool at_home = dst.device == item.home;
  auto finish = [&](i64 bytes) {
    p.v_comm = at_home ? 0 : bytes;
    p.priority = p.v_comm > 0 ? delta / static_cast<double>(p.v_comm)
                              : std::numeric_limits<double>::infinity();
  };
  auto move_whole = [&]() {
    p.delta = delta;
    p.shard = item;
    p.rest.clear();
    p.whole = true;
    finish(bytes_of(item, cfg));
    return true;
  };
  p.delta = delta;
  if (delta >= f_item * (1.0 - 1e-12)) return move_whole();

  const i64 tile = std::max<i64>(1, cfg.tile);
  const i64 L_q = item.n_q();
  if (L_q <= tile) return delta >= 0.9 * f_item ? move_whole() : false;

  double ask = delta;
  const double min_core = cfg.alpha * static_cast<double>(smallest_shard_core(item, tile));
  if (delta < min_core) {
    if (delta >= 0.9 * f_item) return move_whole();
    if (min_core >= 2.0 * delta) return false;
    ask = min_core;
  }

  CommQuery q;
  q.delta_f_max = ask;
  q.f_item = f_item;
  q.L_q = L_q;
  q.L_kv = item.kv_extent;
  q.size_q = cfg.size_q;
  q.size_kv = cfg.size_kv;
  q.layout = item.layout;
  q.ht_mirror = item.ht_mirror;
  ShardChoice s = v_min_comm(q, tile);
  if (s.n_q >= L_q) return delta >= 0.9 * f_item ? move_whole() : false;

  // Over-delivery after tile rounding: one aligned kv step down is taken when
  // it lands closer to the request from below.
  const double over = cfg.alpha * static_cast<double>(s.core) - delta;
  if (over > 0) {
    const i64 kv_min = s.n_q + item.kv_extent - L_q;
    const i64 kv_down = std::max(kv_min, round_down(s.n_kv - 1, tile));
    if (kv_down < s.n_kv) {
      const i64 core_down = s.n_q * (2 * kv_down - s.n_q);
      const double under = delta - cfg.alpha * static_cast<double>(core_down);
      if (core_down > 0 && under >= 0 && under < over) {
        s.n_kv = kv_down;
        s.core = core_down;
      }
    }
  }
  cut(item, s.n_q, s.n_kv, p.shard, p.rest);
  p.whole = false;
  finish(bytes_of(p.shard, cfg));
  return true;
}

// ---------------------------------------------------------------------------
// The greedy loop (P/src/scheduler.cpp:196-357).

namespace {

struct Balancer {
  const SchedCfg& cfg;
  std::vector<Server> sv;
  double fbar = 0, eps_abs = 0, avg_bytes = 1.0;

  explicit Balancer(const SchedCfg& c) : cfg(c) {}

  double worst_dev() const {
    double d = 0;
    for (const Server& s : sv) d = std::max(d, std::abs(s.flops - fbar));
    return d;
  }
  double worst_over() const {
    double d = 0;
    for (const Server& s : sv) d = std::max(d, s.flops - fbar);
    return d;
  }
  void reload(Server& s) const { s.flops = cfg.alpha * static_cast<double>(s.core); }

  // Candidate order: highest priority, then larger delta, then lower item
  // identity (doc, q_begin, q_end, layout), then lower source index.
  static bool better(const Proposal& a, const Item& ia, std::size_t sa, const Proposal& b,
                     const Item& ib, std::size_t sb) {
    const auto ka = std::make_tuple(-a.priority, -a.delta, ia.doc, ia.q_begin, ia.q_end,
                                    static_cast<int>(ia.layout), sa);
    const auto kb = std::make_tuple(-b.priority, -b.delta, ib.doc, ib.q_begin, ib.q_end,
                                    static_cast<int>(ib.layout), sb);
    return ka < kb;
  }

  // Best move toward destination d, or false.
  bool best_move(std::size_t d, Plan& plan, Proposal& best, std::size_t& bs,
                 std::size_t& bi) const {
    bool have = false;
    Proposal cand;
    for (std::size_t s = 0; s < sv.size(); ++s) {
      if (s == d || !(sv[s].flops > fbar)) continue;
      const std::vector<Item>& items = sv[s].items;
      for (std::size_t i = 0; i < items.size(); ++i) {
        if (!propose(sv[s], sv[d], items[i], fbar, cfg, cand)) {
          ++plan.rejected_small;
          continue;
        }
        if (cand.priority * avg_bytes / std::max(fbar, 1.0) < cfg.e_threshold) continue;
        if (!have || better(cand, items[i], s, best, sv[bs].items[bi], bs)) {
          best = cand;
          bs = s;
          bi = i;
          have = true;
        }
      }
    }
    return have;
  }

  void apply(const Proposal& m, std::size_t s, std::size_t i, std::size_t d) {
    const i64 moved = core_of(m.shard);
    Server& src = sv[s];
    Server& dst = sv[d];
    src.items.erase(src.items.begin() + static_cast<std::ptrdiff_t>(i));
    src.items.insert(src.items.end(), m.rest.begin(), m.rest.end());
    src.core -= moved;
    dst.items.push_back(m.shard);
    dst.core += moved;
    reload(src);
    reload(dst);
  }
};

}  // namespace

Plan schedule(const std::vector<Item>& items, i64 n_servers, const SchedCfg& cfg) {
  if (n_servers < 1) throw DomainError("n_servers must be >= 1");
  for (const Item& it : items) {
    check_item(it);
    if (it.home < 0 || it.home >= n_servers)
      throw DomainError("item home_device outside the server range");
  }
  Plan plan;
  plan.epsilon_used = cfg.epsilon;
  Balancer b(cfg);
  b.sv.resize(static_cast<std::size_t>(n_servers));
  for (i64 s = 0; s < n_servers; ++s) b.sv[static_cast<std::size_t>(s)].device = static_cast<std::int32_t>(s);

  i64 total_core = 0, total_bytes = 0;
  for (const Item& it : items) {
    Server& home = b.sv[static_cast<std::size_t>(it.home)];
    home.items.push_back(it);
    const i64 c = core_of(it);
    home.core += c;
    total_core += c;
    total_bytes += bytes_of(it, cfg);
  }
  for (Server& s : b.sv) b.reload(s);
  b.fbar = cfg.alpha * static_cast<double>(total_core) / static_cast<double>(n_servers);
  plan.target = b.fbar;
  b.eps_abs = cfg.epsilon * b.fbar;
  if (!items.empty())
    b.avg_bytes = std::max(1.0, static_cast<double>(total_bytes) / static_cast<double>(items.size()));
  const double slack = one_tile_slack(items, cfg);

  i64 moves = 0;
  bool moved_any = true;
  std::vector<std::pair<std::int32_t, double>> over, under;
  std::vector<double> loads;
  while (moved_any && b.worst_dev() > b.eps_abs && moves < cfg.max_moves) {
    moved_any = false;
    loads.clear();
    for (const Server& s : b.sv) loads.push_back(s.flops);
    classify(loads, b.fbar, over, under);  // deficit order fixed for the pass
    for (const auto& entry : under) {
      const std::size_t d = static_cast<std::size_t>(entry.first);
      while (moves < cfg.max_moves) {
        const double deficit = b.fbar - b.sv[d].flops;
        if (!(deficit > 0)) break;
        if (deficit <= b.eps_abs && b.worst_over() <= b.eps_abs) break;
        Proposal m;
        std::size_t s = 0, i = 0;
        if (!b.best_move(d, plan, m, s, i)) break;
        b.apply(m, s, i, d);
        ++plan.migrations;
        if (!m.whole) ++plan.splits;
        ++moves;
        moved_any = true;
      }
    }
  }

  plan.tolerance_met = b.worst_dev() <= b.eps_abs + slack;
  plan.servers = std::move(b.sv);
  if (!plan.servers.empty()) {
    plan.max_load = -std::numeric_limits<double>::infinity();
    plan.min_load = std::numeric_limits<double>::infinity();
  }
  for (const Server& s : plan.servers) {
    plan.max_load = std::max(plan.max_load, s.flops);
    plan.min_load = std::min(plan.min_load, s.flops);
  }
  // Tasks in per-server item order (P/src/scheduler.cpp:336-355).
  for (std::size_t s = 0; s < plan.servers.size(); ++s) {
    for (const Item& it : plan.servers[s].items) {
      Task t;
      t.item = it;
      t.source = it.home;
      t.server = static_cast<std::int32_t>(s);
      if (t.server != t.source) {
        t.comm_bytes = bytes_of(it, cfg);
        t.output_bytes = it.n_q() * cfg.size_q;
      }
      plan.total_comm_bytes += t.comm_bytes;
      plan.total_output_bytes += t.output_bytes;
      plan.servers[s].received_bytes += t.comm_bytes;
      if (t.comm_bytes > 0) plan.servers[static_cast<std::size_t>(it.home)].sent_bytes += t.comm_bytes;
      plan.tasks.push_back(t);
    }
  }
  return plan;
}

Plan schedule_pp_tick(const std::vector<std::vector<Item>>& per_stage, i64 n_servers,
                      const SchedCfg& cfg) {
  if (static_cast<i64>(per_stage.size()) > n_servers)
    throw DomainError("more stages than servers in a tick");
  std::vector<Item> pooled;
  for (std::size_t st = 0; st < per_stage.size(); ++st)
    for (Item it : per_stage[st]) {
      it.home = static_cast<std::int32_t>(st);
      pooled.push_back(it);
    }
  return schedule(pooled, n_servers, cfg);
}

std::string plan_text(const Plan& plan) {
  std::ostringstream os;
  os << "# plan v1\n"
     << "# doc q_begin q_end kv_extent ht_mirror layout source server core bytes\n";
  for (const Task& t : plan.tasks) {
    const Item& it = t.item;
    os << it.doc << ' ' << it.q_begin << ' ' << it.q_end << ' ' << it.kv_extent << ' '
       << it.ht_mirror << ' ' << (it.layout == Layout::head_tail ? "head_tail" : "contiguous")
       << ' ' << t.source << ' ' << t.server << ' ' << core_of(it) << ' ' << t.comm_bytes
       << '\n';
  }
  return os.str();
}

// ---------------------------------------------------------------------------
// Per-device served/sent lists with ping/pong halves (P/src/sim.cpp:34-46,
// 129-157): each server splits its served tasks into two halves by LPT on
// core (stable, heaviest first onto the lighter half, ties to half 0); a task
// served away from home is also listed as "sent" on its home device, in
// server order, carrying the server's half.
std::vector<DevicePlan> device_plans(const Plan& plan) {
  std::vector<DevicePlan> out(plan.servers.size());
  for (std::size_t t = 0; t < plan.tasks.size(); ++t) {
    const Task& task = plan.tasks[t];
    Served s;
    s.task = static_cast<i64>(t);
    s.in_bytes = task.comm_bytes;
    s.out_bytes = task.output_bytes;
    out.at(static_cast<std::size_t>(task.server)).served.push_back(s);
  }
  for (DevicePlan& dp : out) {
    std::vector<std::size_t> order(dp.served.size());
    for (std::size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::vector<i64> core(dp.served.size());
    for (std::size_t i = 0; i < core.size(); ++i)
      core[i] = core_of(plan.tasks[static_cast<std::size_t>(dp.served[i].task)].item);
    std::stable_sort(order.begin(), order.end(),
                     [&](std::size_t a, std::size_t b) { return core[a] > core[b]; });
    i64 load[2] = {0, 0};
    for (std::size_t i : order) {
      const int h = load[1] < load[0] ? 1 : 0;
      dp.served[i].half = h;
      load[h] += core[i];
    }
  }
  for (std::size_t d = 0; d < out.size(); ++d)
    for (const Served& s : out[d].served) {
      const std::int32_t home = plan.tasks[static_cast<std::size_t>(s.task)].item.home;
      if (home != static_cast<std::int32_t>(d)) out.at(static_cast<std::size_t>(home)).sent.push_back(s);
    }
  return out;
}

}  // namespace cad
