// extern "C" host entry points of include/cad.h: descriptors, workload and
// scheduler. Exceptions never cross the ABI; they become status codes with
// the message kept per thread for cad_last_error().
#include <cstring>
#include <exception>
#include <new>
#include <string>

#include "../../../include/cad.h"
#include "cad_host.hpp"
#include "cad_status.hpp"

struct cad_plan {
  cad::Plan plan;
  std::vector<cad_task> tasks;                 // C mirror of plan.tasks
  std::vector<std::vector<cad_item>> items;    // C mirror of per-server items
  std::vector<cad::DevicePlan> devices;        // built once, read-only after
};

namespace {

cad::Item from_c(const cad_item& c) {
  cad::Item it;
  it.doc = c.doc;
  it.q_begin = c.q_begin;
  it.q_end = c.q_end;
  it.kv_extent = c.kv_extent;
  it.ht_mirror = c.ht_mirror;
  it.home = c.home_device;
  it.layout = c.layout == CAD_LAYOUT_HEAD_TAIL ? cad::Layout::head_tail : cad::Layout::contiguous;
  return it;
}

cad_item to_c(const cad::Item& it) {
  cad_item c;
  std::memset(&c, 0, sizeof(c));
  c.doc = it.doc;
  c.q_begin = it.q_begin;
  c.q_end = it.q_end;
  c.kv_extent = it.kv_extent;
  c.ht_mirror = it.ht_mirror;
  c.home_device = it.home;
  c.layout = static_cast<uint8_t>(it.layout);
  return c;
}

cad::SchedCfg from_c(const cad_sched_cfg& c) {
  cad::SchedCfg s;
  s.epsilon = c.epsilon;
  s.e_threshold = c.e_threshold;
  s.tile = c.tile_size;
  s.alpha = c.alpha_ca;
  s.size_q = c.size_q;
  s.size_kv = c.size_kv;
  s.double_query_ht = c.double_query_head_tail != 0;
  s.max_moves = c.max_moves;
  return s;
}

std::vector<cad::Item> items_from_c(const cad_item* items, int64_t n) {
  if (n < 0 || (n > 0 && !items)) throw cad::DomainError("bad item array");
  std::vector<cad::Item> v;
  v.reserve(static_cast<std::size_t>(n));
  for (int64_t i = 0; i < n; ++i) v.push_back(from_c(items[i]));
  return v;
}

cad_plan* wrap(cad::Plan&& p) {
  auto* out = new cad_plan;
  out->plan = std::move(p);
  for (const cad::Task& t : out->plan.tasks) {
    cad_task c;
    std::memset(&c, 0, sizeof(c));
    c.item = to_c(t.item);
    c.source_device = t.source;
    c.assigned_server = t.server;
    c.comm_bytes = t.comm_bytes;
    c.output_bytes = t.output_bytes;
    out->tasks.push_back(c);
  }
  for (const cad::Server& s : out->plan.servers) {
    std::vector<cad_item> v;
    for (const cad::Item& it : s.items) v.push_back(to_c(it));
    out->items.push_back(std::move(v));
  }
  out->devices = cad::device_plans(out->plan);
  return out;
}

}  // namespace

const cad::Plan& cad_plan_ref(const cad_plan* p) { return p->plan; }
const std::vector<cad::DevicePlan>& cad_plan_devices(const cad_plan* p) { return p->devices; }

extern "C" {

const char* cad_last_error(void) { return cad::last_error().c_str(); }
const char* cad_version(void) { return "cad-b200 0.1 (sm_100a)"; }

void cad_sched_cfg_default(cad_sched_cfg* cfg) {
  if (!cfg) return;
  std::memset(cfg, 0, sizeof(*cfg));
  const cad::SchedCfg d;
  cfg->epsilon = d.epsilon;
  cfg->e_threshold = d.e_threshold;
  cfg->tile_size = d.tile;
  cfg->alpha_ca = d.alpha;
  cfg->size_q = d.size_q;
  cfg->size_kv = d.size_kv;
  cfg->double_query_head_tail = d.double_query_ht ? 1 : 0;
  cfg->max_moves = d.max_moves;
}

void cad_length_dist_default(cad_length_dist* out) {
  if (!out) return;
  std::memset(out, 0, sizeof(*out));
  const cad::LengthDist d;
  out->kind = CAD_DIST_FIXED;
  out->max_doc_len = d.max_doc_len;
  out->min_len_threshold = d.min_len_threshold;
  out->seed = d.seed;
  out->log_mu = d.log_mu;
  out->log_sigma = d.log_sigma;
  out->upsample_drop_prob = d.drop_prob;
  out->long_mix_weight = d.long_weight;
  out->long_log_mu = d.long_log_mu;
  out->long_log_sigma = d.long_log_sigma;
  out->fixed_len = d.fixed_len;
  out->uniform_min = d.uniform_min;
}

int cad_validate_item(const cad_item* item) {
  return cad::guarded([&] {
    if (!item) throw cad::DomainError("null item");
    cad::check_item(from_c(*item));
  });
}

int cad_ca_flops_core(const cad_item* item, int64_t* core) {
  return cad::guarded([&] {
    if (!item || !core) throw cad::DomainError("null argument");
    *core = cad::core_of(from_c(*item));
  });
}

int64_t cad_causal_pairs(int64_t n_q, int64_t n_kv) { return cad::causal_pairs(n_q, n_kv); }

int cad_item_bytes(const cad_item* item, const cad_sched_cfg* cfg, int64_t* bytes) {
  return cad::guarded([&] {
    if (!item || !cfg || !bytes) throw cad::DomainError("null argument");
    *bytes = cad::bytes_of(from_c(*item), from_c(*cfg));
  });
}

int cad_sample_batch(const cad_length_dist* dist, int64_t total_tokens, int64_t* lengths,
                     int64_t cap, int64_t* n_docs) {
  return cad::guarded([&] {
    if (!dist || !n_docs) throw cad::DomainError("null argument");
    cad::LengthDist d;
    switch (dist->kind) {
      case CAD_DIST_PRETRAIN_UPSAMPLED: d.kind = cad::Dist::pretrain_upsampled; break;
      case CAD_DIST_PROLONG_LIKE: d.kind = cad::Dist::prolong_like; break;
      case CAD_DIST_UNIFORM: d.kind = cad::Dist::uniform; break;
      case CAD_DIST_FIXED: d.kind = cad::Dist::fixed; break;
      case CAD_DIST_CUSTOM_HISTOGRAM: d.kind = cad::Dist::histogram; break;
      default: throw cad::ConfigError("unknown distribution kind");
    }
    d.max_doc_len = dist->max_doc_len;
    d.min_len_threshold = dist->min_len_threshold;
    d.seed = dist->seed;
    d.log_mu = dist->log_mu;
    d.log_sigma = dist->log_sigma;
    d.drop_prob = dist->upsample_drop_prob;
    d.long_weight = dist->long_mix_weight;
    d.long_log_mu = dist->long_log_mu;
    d.long_log_sigma = dist->long_log_sigma;
    d.fixed_len = dist->fixed_len;
    d.uniform_min = dist->uniform_min;
    for (int64_t i = 0; i < dist->hist_n; ++i) d.histogram.emplace_back(dist->hist_len[i], dist->hist_p[i]);
    const std::vector<int64_t> v = cad::sample_lengths(d, total_tokens);
    *n_docs = static_cast<int64_t>(v.size());
    if (!lengths) return;
    if (cap < *n_docs) throw cad::CapacityError("length buffer too small");
    std::memcpy(lengths, v.data(), v.size() * sizeof(int64_t));
  });
}

int cad_place_sequential(const int64_t* lengths, int64_t n_docs, int64_t n_devices,
                         int64_t tokens_per_device, cad_item* items, int64_t cap,
                         int64_t* n_items) {
  return cad::guarded([&] {
    if ((!lengths && n_docs > 0) || !n_items || n_docs < 0) throw cad::DomainError("null argument");
    std::vector<int64_t> l(lengths, lengths + n_docs);
    const std::vector<cad::Item> v = cad::sequential_items(l, n_devices, tokens_per_device);
    *n_items = static_cast<int64_t>(v.size());
    if (!items) return;
    if (cap < *n_items) throw cad::CapacityError("item buffer too small");
    for (std::size_t i = 0; i < v.size(); ++i) items[i] = to_c(v[i]);
  });
}

int cad_target_load(const cad_item* items, int64_t n, int64_t n_servers, double alpha_ca,
                    double* target) {
  return cad::guarded([&] {
    if (!target) throw cad::DomainError("null argument");
    *target = cad::target_load(items_from_c(items, n), n_servers, alpha_ca);
  });
}

int cad_classify_servers(const double* loads, int64_t n, double target, int32_t* surplus_dev,
                         double* surplus_gap, int64_t* n_surplus, int32_t* deficit_dev,
                         double* deficit_gap, int64_t* n_deficit) {
  return cad::guarded([&] {
    if ((!loads && n > 0) || !n_surplus || !n_deficit) throw cad::DomainError("null argument");
    std::vector<double> l(loads, loads + n);
    std::vector<std::pair<int32_t, double>> s, d;
    cad::classify(l, target, s, d);
    *n_surplus = static_cast<int64_t>(s.size());
    *n_deficit = static_cast<int64_t>(d.size());
    for (std::size_t i = 0; i < s.size(); ++i) {
      if (surplus_dev) surplus_dev[i] = s[i].first;
      if (surplus_gap) surplus_gap[i] = s[i].second;
    }
    for (std::size_t i = 0; i < d.size(); ++i) {
      if (deficit_dev) deficit_dev[i] = d[i].first;
      if (deficit_gap) deficit_gap[i] = d[i].second;
    }
  });
}

int cad_one_tile_slack(const cad_item* items, int64_t n, const cad_sched_cfg* cfg, double* slack) {
  return cad::guarded([&] {
    if (!cfg || !slack) throw cad::DomainError("null argument");
    *slack = cad::one_tile_slack(items_from_c(items, n), from_c(*cfg));
  });
}

int cad_v_min_comm(const cad_comm_query* q, int64_t tile, cad_shard_choice* out) {
  return cad::guarded([&] {
    if (!q || !out) throw cad::DomainError("null argument");
    cad::CommQuery c;
    c.delta_f_max = q->delta_f_max;
    c.f_item = q->f_item;
    c.L_q = q->L_q;
    c.L_kv = q->L_kv;
    c.size_q = q->size_q;
    c.size_kv = q->size_kv;
    c.layout = q->layout == CAD_LAYOUT_HEAD_TAIL ? cad::Layout::head_tail : cad::Layout::contiguous;
    c.ht_mirror = q->ht_mirror;
    const cad::ShardChoice s = cad::v_min_comm(c, tile);
    out->n_q = s.n_q;
    out->n_kv = s.n_kv;
    out->bytes = s.bytes;
    out->core = s.core;
  });
}

int cad_propose_migration(const cad_server_load* source, const cad_server_load* dest,
                          const cad_item* item, double target, const cad_sched_cfg* cfg,
                          cad_proposal* out, int32_t* has_value) {
  return cad::guarded([&] {
    if (!source || !dest || !item || !cfg || !out || !has_value)
      throw cad::DomainError("null argument");
    cad::Server s, d;
    s.device = source->device;
    s.flops = source->assigned_flops;
    s.core = source->assigned_core;
    d.device = dest->device;
    d.flops = dest->assigned_flops;
    d.core = dest->assigned_core;
    cad::Proposal p;
    std::memset(out, 0, sizeof(*out));
    *has_value = cad::propose(s, d, from_c(*item), target, from_c(*cfg), p) ? 1 : 0;
    if (!*has_value) return;
    out->delta_f_max = p.delta;
    out->shard = to_c(p.shard);
    out->n_remainders = static_cast<int32_t>(p.rest.size());
    for (std::size_t i = 0; i < p.rest.size() && i < 2; ++i) out->remainders[i] = to_c(p.rest[i]);
    out->whole_item = p.whole ? 1 : 0;
    out->v_comm = p.v_comm;
    out->priority = p.priority;
  });
}

int cad_schedule(const cad_item* items, int64_t n, int64_t n_servers, const cad_sched_cfg* cfg,
                 cad_plan** plan) {
  return cad::guarded([&] {
    if (!cfg || !plan) throw cad::DomainError("null argument");
    *plan = nullptr;
    *plan = wrap(cad::schedule(items_from_c(items, n), n_servers, from_c(*cfg)));
  });
}

int cad_schedule_pp_tick(const cad_item* items, const int32_t* stage_of, int64_t n,
                         int64_t n_stages, int64_t n_servers, const cad_sched_cfg* cfg,
                         cad_plan** plan) {
  return cad::guarded([&] {
    if (!cfg || !plan || (n > 0 && !stage_of) || n_stages < 0) throw cad::DomainError("null argument");
    *plan = nullptr;
    std::vector<cad::Item> flat = items_from_c(items, n);
    std::vector<std::vector<cad::Item>> per_stage(static_cast<std::size_t>(n_stages));
    for (int64_t i = 0; i < n; ++i) {
      if (stage_of[i] < 0 || stage_of[i] >= n_stages) throw cad::DomainError("stage index out of range");
      per_stage[static_cast<std::size_t>(stage_of[i])].push_back(flat[static_cast<std::size_t>(i)]);
    }
    *plan = wrap(cad::schedule_pp_tick(per_stage, n_servers, from_c(*cfg)));
  });
}

int cad_plan_get_stats(const cad_plan* plan, cad_plan_stats* st) {
  return cad::guarded([&] {
    if (!plan || !st) throw cad::DomainError("null argument");
    std::memset(st, 0, sizeof(*st));
    const cad::Plan& p = plan->plan;
    st->target = p.target;
    st->max_load = p.max_load;
    st->min_load = p.min_load;
    st->epsilon_used = p.epsilon_used;
    st->total_comm_bytes = p.total_comm_bytes;
    st->total_output_bytes = p.total_output_bytes;
    st->migrations = p.migrations;
    st->splits = p.splits;
    st->rejected_small = p.rejected_small;
    st->n_tasks = static_cast<int64_t>(p.tasks.size());
    st->n_servers = static_cast<int64_t>(p.servers.size());
    st->tolerance_met = p.tolerance_met ? 1 : 0;
  });
}

int cad_plan_tasks(const cad_plan* plan, const cad_task** tasks, int64_t* n) {
  return cad::guarded([&] {
    if (!plan || !tasks || !n) throw cad::DomainError("null argument");
    *tasks = plan->tasks.data();
    *n = static_cast<int64_t>(plan->tasks.size());
  });
}

int cad_plan_server(const cad_plan* plan, int64_t server, cad_server_load* load,
                    const cad_item** items) {
  return cad::guarded([&] {
    if (!plan || !load) throw cad::DomainError("null argument");
    if (server < 0 || server >= static_cast<int64_t>(plan->plan.servers.size()))
      throw cad::DomainError("server index out of range");
    const cad::Server& s = plan->plan.servers[static_cast<std::size_t>(server)];
    std::memset(load, 0, sizeof(*load));
    load->device = s.device;
    load->assigned_flops = s.flops;
    load->assigned_core = s.core;
    load->n_items = static_cast<int64_t>(s.items.size());
    load->sent_bytes = s.sent_bytes;
    load->received_bytes = s.received_bytes;
    if (items) *items = plan->items[static_cast<std::size_t>(server)].data();
  });
}

int cad_plan_to_text(const cad_plan* plan, char* buf, size_t cap, size_t* needed) {
  return cad::guarded([&] {
    if (!plan || !needed) throw cad::DomainError("null argument");
    const std::string s = cad::plan_text(plan->plan);
    *needed = s.size() + 1;
    if (!buf) return;
    if (cap < s.size() + 1) throw cad::CapacityError("text buffer too small");
    std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

void cad_plan_free(cad_plan* plan) { delete plan; }

int cad_device_plan(const cad_plan* plan, int32_t device, cad_served_task* served,
                    int64_t cap_served, int64_t* n_served, cad_served_task* sent, int64_t cap_sent,
                    int64_t* n_sent) {
  return cad::guarded([&] {
    if (!plan || !n_served || !n_sent) throw cad::DomainError("null argument");
    if (device < 0 || device >= static_cast<int32_t>(plan->devices.size()))
      throw cad::DomainError("device index out of range");
    const cad::DevicePlan& dp = plan->devices[static_cast<std::size_t>(device)];
    *n_served = static_cast<int64_t>(dp.served.size());
    *n_sent = static_cast<int64_t>(dp.sent.size());
    auto fill = [](const std::vector<cad::Served>& v, cad_served_task* dst, int64_t cap) {
      if (!dst) return;
      if (cap < static_cast<int64_t>(v.size())) throw cad::CapacityError("served buffer too small");
      for (std::size_t i = 0; i < v.size(); ++i) {
        std::memset(&dst[i], 0, sizeof(dst[i]));
        dst[i].task_index = v[i].task;
        dst[i].in_bytes = v[i].in_bytes;
        dst[i].out_bytes = v[i].out_bytes;
        dst[i].half = v[i].half;
      }
    };
    fill(dp.served, served, cap_served);
    fill(dp.sent, sent, cap_sent);
  });
}

}  // extern "C"
