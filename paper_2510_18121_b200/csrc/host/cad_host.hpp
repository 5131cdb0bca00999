// Host-side CA-task model: descriptors, workload placement and the
// communication-aware greedy scheduler of DistCA (paper section 4.2).
//
// Re-implemented from the reference's documented behaviour; every function
// cites the reference function it must match bit-for-bit
// (P = /root/reference/proj). Integer extents/bytes are int64, loads and
// priorities IEEE double in the same operation order as the reference, and
// this translation unit is compiled with -ffp-contract=off.
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace cad {

using i64 = std::int64_t;

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DomainError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum class Layout : std::uint8_t { contiguous = 0, head_tail = 1 };

// P/include/cadsim/types.hpp:112-124
struct Item {
  i64 doc = 0, q_begin = 0, q_end = 0, kv_extent = 0, ht_mirror = 0;
  std::int32_t home = 0;
  Layout layout = Layout::contiguous;
  i64 n_q() const { return q_end - q_begin; }
};

// P/include/cadsim/types.hpp:131-137
struct Task {
  Item item;
  std::int32_t source = 0, server = 0;
  i64 comm_bytes = 0, output_bytes = 0;
};

// P/include/cadsim/scheduler.hpp:12-21
struct SchedCfg {
  double epsilon = 0.0;
  double e_threshold = 0.01;
  i64 tile = 128;
  double alpha = 1.0;
  i64 size_q = 2, size_kv = 2;
  bool double_query_ht = false;
  i64 max_moves = i64(1) << 20;
};

// P/include/cadsim/scheduler.hpp:23-30
struct Server {
  std::int32_t device = 0;
  double flops = 0;
  i64 core = 0;
  std::vector<Item> items;
  i64 sent_bytes = 0, received_bytes = 0;
};

// P/include/cadsim/scheduler.hpp:32-45
struct Plan {
  std::vector<Task> tasks;
  std::vector<Server> servers;
  double target = 0, max_load = 0, min_load = 0;
  i64 total_comm_bytes = 0, total_output_bytes = 0;
  double epsilon_used = 0;
  bool tolerance_met = false;
  i64 migrations = 0, splits = 0, rejected_small = 0;
};

// P/include/cadsim/scheduler.hpp:60-67
struct Proposal {
  double delta = 0;
  Item shard;
  std::vector<Item> rest;
  i64 v_comm = 0;
  double priority = 0;
  bool whole = false;
};

// P/include/cadsim/comm.hpp:41-60
struct CommQuery {
  double delta_f_max = 0, f_item = 0;
  i64 L_q = 0, L_kv = 0, size_q = 0, size_kv = 0;
  Layout layout = Layout::contiguous;
  i64 ht_mirror = 0;
};
struct ShardChoice {
  i64 n_q = 0, n_kv = 0, bytes = 0, core = 0;
};

enum class Dist : std::uint8_t { pretrain_upsampled, prolong_like, uniform, fixed, histogram };

// P/include/cadsim/workload.hpp:28-43
struct LengthDist {
  Dist kind = Dist::fixed;
  i64 max_doc_len = i64(1) << 20;
  i64 min_len_threshold = 0;
  std::uint64_t seed = 0;
  double log_mu = std::log(2048.0);
  double log_sigma = 1.4;
  double drop_prob = 0.8;
  double long_weight = 0.3;
  double long_log_mu = std::log(65536.0);
  double long_log_sigma = 0.7;
  i64 fixed_len = 1024;
  i64 uniform_min = 1;
  std::vector<std::pair<i64, double>> histogram;
};

struct Served {
  i64 task = 0;  // index into Plan::tasks
  i64 in_bytes = 0, out_bytes = 0;
  int half = 0;
};
struct DevicePlan {
  std::vector<Served> served, sent;
};

// --- cost / bytes ---------------------------------------------------------
void check_item(const Item& it);                      // P/src/types.cpp:58-74
i64 core_of(const Item& it);                          // P/src/cost.cpp:32-44
i64 bytes_of(const Item& it, const SchedCfg& cfg);    // P/src/scheduler.cpp:53-60
inline i64 causal_pairs(i64 n_q, i64 n_kv) { return n_q * (2 * n_kv - n_q + 1) / 2; }

// --- workload ---------------------------------------------------------------
std::vector<i64> sample_lengths(const LengthDist& d, i64 total);          // workload.cpp:67-84
std::vector<Item> sequential_items(const std::vector<i64>& lengths, i64 devices,
                                   i64 per_device);                        // workload.cpp:86-124

// --- scheduler --------------------------------------------------------------
double target_load(const std::vector<Item>& items, i64 n_servers, double alpha);
void classify(const std::vector<double>& loads, double target,
              std::vector<std::pair<std::int32_t, double>>& surplus,
              std::vector<std::pair<std::int32_t, double>>& deficit);
double one_tile_slack(const std::vector<Item>& items, const SchedCfg& cfg);
ShardChoice v_min_comm(const CommQuery& q, i64 tile);
bool propose(const Server& src, const Server& dst, const Item& item, double target,
             const SchedCfg& cfg, Proposal& out);
Plan schedule(const std::vector<Item>& items, i64 n_servers, const SchedCfg& cfg);
Plan schedule_pp_tick(const std::vector<std::vector<Item>>& per_stage, i64 n_servers,
                      const SchedCfg& cfg);
std::string plan_text(const Plan& plan);
std::vector<DevicePlan> device_plans(const Plan& plan);

}  // namespace cad
