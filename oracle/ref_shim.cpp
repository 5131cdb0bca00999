// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// C wrappers around the UNMODIFIED reference scheduler (`cadsim`, compiled
// from its own sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libcadsim_ref.so). tests/ and bench.py's cpu_baseline leg load
// it through ctypes to check the product scheduler bit-for-bit and to time
// the reference's CPU path. Struct layouts are the ones of include/cad.h so
// both sides share one Python marshalling layer.
#include <chrono>
#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include "../include/cad.h"
#include "cadsim/comm.hpp"
#include "cadsim/cost.hpp"
#include "cadsim/scheduler.hpp"
#include "cadsim/sim.hpp"
#include "cadsim/types.hpp"
#include "cadsim/workload.hpp"

namespace {

thread_local std::string g_err;

cadsim::Item to_ref(const cad_item& c) {
  cadsim::Item it;
  it.doc = c.doc;
  it.q_begin = c.q_begin;
  it.q_end = c.q_end;
  it.kv_extent = c.kv_extent;
  it.ht_mirror = c.ht_mirror;
  it.home_device = c.home_device;
  it.layout = c.layout == CAD_LAYOUT_HEAD_TAIL ? cadsim::Layout::head_tail
                                               : cadsim::Layout::contiguous;
  return it;
}

cad_item from_ref(const cadsim::Item& it) {
  cad_item c;
  std::memset(&c, 0, sizeof(c));
  c.doc = it.doc;
  c.q_begin = it.q_begin;
  c.q_end = it.q_end;
  c.kv_extent = it.kv_extent;
  c.ht_mirror = it.ht_mirror;
  c.home_device = it.home_device;
  c.layout = it.layout == cadsim::Layout::head_tail ? CAD_LAYOUT_HEAD_TAIL : CAD_LAYOUT_CONTIGUOUS;
  return c;
}

cadsim::SchedulerConfig to_ref(const cad_sched_cfg& c) {
  cadsim::SchedulerConfig s;
  s.epsilon = c.epsilon;
  s.e_threshold = c.e_threshold;
  s.tile_size = c.tile_size;
  s.alpha_ca = c.alpha_ca;
  s.size_q = c.size_q;
  s.size_kv = c.size_kv;
  s.double_query_head_tail = c.double_query_head_tail != 0;
  s.max_moves = c.max_moves;
  return s;
}

std::vector<cadsim::Item> items_to_ref(const cad_item* items, int64_t n) {
  std::vector<cadsim::Item> v;
  for (int64_t i = 0; i < n; ++i) v.push_back(to_ref(items[i]));
  return v;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const cadsim::ConfigError& e) {
    g_err = e.what();
    return -1;
  } catch (const cadsim::DomainError& e) {
    g_err = e.what();
    return -2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -2;
  }
}

// A reference plan flattened for comparison: the plan_to_stream text, the
// scalar stats, per-server loads and per-device served/sent lists with
// halves, all produced by the reference's own functions.
struct RefPlan {
  std::string text;
  cad_plan_stats stats{};
  std::vector<double> server_flops;
  std::vector<int64_t> server_core, server_sent, server_recv;
  std::vector<cad_task> tasks;
  std::string devices;  // "d served|sent doc q_begin q_end half in out\n"
};

void flatten(const cadsim::SchedulePlan& p, RefPlan& r) {
  std::ostringstream os;
  cadsim::plan_to_stream(p, os);
  r.text = os.str();
  std::memset(&r.stats, 0, sizeof(r.stats));
  r.stats.target = p.target;
  r.stats.max_load = p.max_load;
  r.stats.min_load = p.min_load;
  r.stats.epsilon_used = p.epsilon_used;
  r.stats.total_comm_bytes = p.total_comm_bytes;
  r.stats.total_output_bytes = p.total_output_bytes;
  r.stats.migrations = p.migrations;
  r.stats.splits = p.splits;
  r.stats.rejected_small = p.rejected_small;
  r.stats.n_tasks = static_cast<int64_t>(p.tasks.size());
  r.stats.n_servers = static_cast<int64_t>(p.per_server.size());
  r.stats.tolerance_met = p.tolerance_met ? 1 : 0;
  for (const auto& s : p.per_server) {
    r.server_flops.push_back(s.assigned_flops);
    r.server_core.push_back(s.assigned_core);
    r.server_sent.push_back(s.sent_bytes);
    r.server_recv.push_back(s.received_bytes);
  }
  for (const auto& t : p.tasks) {
    cad_task c;
    std::memset(&c, 0, sizeof(c));
    c.item = from_ref(t.item);
    c.source_device = t.source_device;
    c.assigned_server = t.assigned_server;
    c.comm_bytes = t.comm_bytes;
    c.output_bytes = t.output_bytes;
    r.tasks.push_back(c);
  }
  const auto dps = cadsim::device_plans_from_schedule(p, {}, cadsim::CostCoefficients{});
  std::ostringstream ds;
  for (const auto& dp : dps) {
    for (const auto& st : dp.served)
      ds << dp.device << " served " << st.item.doc << ' ' << st.item.q_begin << ' '
         << st.item.q_end << ' ' << st.half << ' ' << st.in_bytes << ' ' << st.out_bytes << '\n';
    for (const auto& st : dp.sent)
      ds << dp.device << " sent " << st.item.doc << ' ' << st.item.q_begin << ' '
         << st.item.q_end << ' ' << st.half << ' ' << st.in_bytes << ' ' << st.out_bytes << '\n';
  }
  r.devices = ds.str();
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_sample_batch(const cad_length_dist* d, int64_t total, int64_t* lengths, int64_t cap,
                     int64_t* n) {
  return guard([&] {
    cadsim::LengthDistribution dist;
    dist.kind = static_cast<cadsim::DistKind>(d->kind);
    dist.max_doc_len = d->max_doc_len;
    dist.min_len_threshold = d->min_len_threshold;
    dist.seed = d->seed;
    dist.log_mu = d->log_mu;
    dist.log_sigma = d->log_sigma;
    dist.upsample_drop_prob = d->upsample_drop_prob;
    dist.long_mix_weight = d->long_mix_weight;
    dist.long_log_mu = d->long_log_mu;
    dist.long_log_sigma = d->long_log_sigma;
    dist.fixed_len = d->fixed_len;
    dist.uniform_min = d->uniform_min;
    for (int64_t i = 0; i < d->hist_n; ++i) dist.histogram.emplace_back(d->hist_len[i], d->hist_p[i]);
    const auto docs = cadsim::sample_batch(dist, total);
    *n = static_cast<int64_t>(docs.size());
    if (!lengths) return;
    for (std::size_t i = 0; i < docs.size() && static_cast<int64_t>(i) < cap; ++i)
      lengths[i] = docs[i].length;
  });
}

int ref_place_sequential(const int64_t* lengths, int64_t n_docs, int64_t devices,
                         int64_t per_device, cad_item* items, int64_t cap, int64_t* n_items) {
  return guard([&] {
    std::vector<cadsim::Document> docs;
    for (int64_t i = 0; i < n_docs; ++i) docs.push_back({i, lengths[i]});
    const auto chunks = cadsim::place_sequential(docs, devices, per_device);
    const auto v = cadsim::chunk_items(chunks);
    *n_items = static_cast<int64_t>(v.size());
    if (!items) return;
    for (std::size_t i = 0; i < v.size() && static_cast<int64_t>(i) < cap; ++i)
      items[i] = from_ref(v[i]);
  });
}

int ref_ca_flops_core(const cad_item* it, int64_t* core) {
  return guard([&] { *core = cadsim::ca_flops_core(to_ref(*it)); });
}

int ref_one_tile_slack(const cad_item* items, int64_t n, const cad_sched_cfg* cfg, double* out) {
  return guard([&] { *out = cadsim::one_tile_slack(items_to_ref(items, n), to_ref(*cfg)); });
}

int ref_target_load(const cad_item* items, int64_t n, int64_t servers, double alpha, double* out) {
  return guard([&] { *out = cadsim::target_load(items_to_ref(items, n), servers, alpha); });
}

int ref_v_min_comm(const cad_comm_query* q, int64_t tile, cad_shard_choice* out) {
  return guard([&] {
    cadsim::CommQuery c;
    c.delta_f_max = q->delta_f_max;
    c.f_item = q->f_item;
    c.L_q = q->L_q;
    c.L_kv = q->L_kv;
    c.size_q = q->size_q;
    c.size_kv = q->size_kv;
    c.layout = q->layout == CAD_LAYOUT_HEAD_TAIL ? cadsim::Layout::head_tail
                                                 : cadsim::Layout::contiguous;
    c.ht_mirror = q->ht_mirror;
    const auto s = cadsim::v_min_comm(c, tile);
    out->n_q = s.n_q;
    out->n_kv = s.n_kv;
    out->bytes = s.bytes;
    out->core = s.core;
  });
}

int ref_propose_migration(const cad_server_load* src, const cad_server_load* dst,
                          const cad_item* item, double target, const cad_sched_cfg* cfg,
                          cad_proposal* out, int32_t* has) {
  return guard([&] {
    cadsim::ServerLoad s, d;
    s.device = src->device;
    s.assigned_flops = src->assigned_flops;
    s.assigned_core = src->assigned_core;
    d.device = dst->device;
    d.assigned_flops = dst->assigned_flops;
    d.assigned_core = dst->assigned_core;
    const auto p = cadsim::propose_migration(s, d, to_ref(*item), target, to_ref(*cfg));
    std::memset(out, 0, sizeof(*out));
    *has = p.has_value() ? 1 : 0;
    if (!p) return;
    out->delta_f_max = p->delta_f_max;
    out->shard = from_ref(p->shard);
    out->n_remainders = static_cast<int32_t>(p->remainders.size());
    for (std::size_t i = 0; i < p->remainders.size() && i < 2; ++i)
      out->remainders[i] = from_ref(p->remainders[i]);
    out->whole_item = p->whole_item ? 1 : 0;
    out->v_comm = p->v_comm;
    out->priority = p->priority;
  });
}

void* ref_schedule(const cad_item* items, int64_t n, int64_t n_servers, const cad_sched_cfg* cfg,
                   const int32_t* stage_of, int64_t n_stages) {
  RefPlan* r = new RefPlan;
  const int rc = guard([&] {
    cadsim::SchedulePlan p;
    if (stage_of) {
      std::vector<std::vector<cadsim::Item>> per(static_cast<std::size_t>(n_stages));
      for (int64_t i = 0; i < n; ++i) per[static_cast<std::size_t>(stage_of[i])].push_back(to_ref(items[i]));
      p = cadsim::schedule_pp_tick(per, n_servers, to_ref(*cfg));
    } else {
      p = cadsim::schedule(items_to_ref(items, n), n_servers, to_ref(*cfg));
    }
    flatten(p, *r);
  });
  if (rc != 0) {
    delete r;
    return nullptr;
  }
  return r;
}

const char* ref_plan_text(void* h) { return static_cast<RefPlan*>(h)->text.c_str(); }
const char* ref_plan_devices(void* h) { return static_cast<RefPlan*>(h)->devices.c_str(); }
void ref_plan_stats(void* h, cad_plan_stats* st) { *st = static_cast<RefPlan*>(h)->stats; }
const cad_task* ref_plan_tasks(void* h, int64_t* n) {
  auto* r = static_cast<RefPlan*>(h);
  *n = static_cast<int64_t>(r->tasks.size());
  return r->tasks.data();
}
void ref_plan_servers(void* h, double* flops, int64_t* core, int64_t* sent, int64_t* recv) {
  auto* r = static_cast<RefPlan*>(h);
  for (std::size_t i = 0; i < r->server_flops.size(); ++i) {
    flops[i] = r->server_flops[i];
    core[i] = r->server_core[i];
    sent[i] = r->server_sent[i];
    recv[i] = r->server_recv[i];
  }
}
void ref_plan_free(void* h) { delete static_cast<RefPlan*>(h); }

// Loads a profiler-grid CSV with the reference's own parser
// (grid_from_csv, P/src/cost.cpp:215-262) and returns profile_lookup at
// (n_q, n_kv); -1 on a parse/validation error.
double ref_grid_lookup(const char* csv, double peak, double alpha, int64_t tile, int64_t n_q,
                       int64_t n_kv) {
  try {
    std::istringstream in(csv);
    const auto g = cadsim::grid_from_csv(in, peak, alpha, tile);
    return cadsim::profile_lookup(g, n_q, n_kv);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}

// Wall time of `reps` calls of the reference schedule() (CPU baseline).
double ref_schedule_seconds(const cad_item* items, int64_t n, int64_t n_servers,
                            const cad_sched_cfg* cfg, int64_t reps) {
  const auto v = items_to_ref(items, n);
  const auto c = to_ref(*cfg);
  const auto t0 = std::chrono::steady_clock::now();
  std::int64_t sink = 0;
  for (int64_t r = 0; r < reps; ++r) sink += cadsim::schedule(v, n_servers, c).migrations;
  const auto t1 = std::chrono::steady_clock::now();
  if (sink < 0) g_err = "unreachable";
  return std::chrono::duration<double>(t1 - t0).count();
}

// simulate_pp_iteration (P/src/sim.cpp:297-485) on microbatches given as
// items (mb_of[i] = microbatch of item i, tokens[m] = its tokens), an
// 8B-like model with num_layers = stages (one layer per stage, so the wire
// bytes stay integral) and the test suite's 8-GPU cluster shape: the tick
// count, the total wire bytes, and per stage the kinds of its events
// (0 forward, 1 backward; 1F1B) in time order.
int ref_pp_iteration(const cad_item* items, const int64_t* mb_of, int64_t n_items, const int64_t* tokens,
                     int64_t M, int64_t S, int32_t kind, const cad_sched_cfg* cfg, int64_t* ticks,
                     int64_t* wire_bytes, int32_t* ev_kinds, int64_t ev_cap, int64_t* ev_count) {
  return guard([&] {
    std::vector<cadsim::Microbatch> mbs(static_cast<std::size_t>(M));
    for (int64_t m = 0; m < M; ++m) mbs[static_cast<std::size_t>(m)].tokens = tokens[m];
    for (int64_t i = 0; i < n_items; ++i) mbs[static_cast<std::size_t>(mb_of[i])].items.push_back(to_ref(items[i]));
    cadsim::ModelConfig model;
    model.num_layers = S;
    model.hidden = 4096;
    model.kv_hidden = 1024;
    model.ffn_intermediate = 14336;
    model.head_dim = 128;
    model.num_heads = 32;
    model.gqa_groups = 8;
    model = cadsim::derive_sizes(model);
    cadsim::ClusterConfig cluster;
    cluster.num_gpus = S;
    cluster.dp = S;
    cluster.interconnect_bandwidth = 50.0 * (1ull << 30);
    cluster.peak_flops = 990e12;
    cluster.tile_size = 128;
    const auto coeff = cadsim::derive_coefficients(model);
    const auto grid = cadsim::synth_grid(model, cluster, 1 << 16);
    cadsim::SimConfig sim;
    sim.record_events = true;
    const auto rep = cadsim::simulate_pp_iteration(
        mbs, S, kind == CAD_PP_1F1B ? cadsim::PPSchedule::vanilla_1f1b : cadsim::PPSchedule::cad_phase_sync, model,
        cluster, coeff, grid, sim, to_ref(*cfg));
    *ticks = rep.ticks;
    *wire_bytes = rep.total_wire_bytes;
    for (int64_t s = 0; s < S; ++s) {
      const auto& ev = rep.per_device[static_cast<std::size_t>(s)].events;
      ev_count[s] = static_cast<int64_t>(ev.size());
      for (std::size_t e = 0; e < ev.size() && static_cast<int64_t>(e) < ev_cap; ++e)
        ev_kinds[s * ev_cap + static_cast<int64_t>(e)] =
            (ev[e].kind == "backward" || ev[e].kind == "tick_backward") ? 1 : 0;
    }
  });
}

}  // extern "C"
