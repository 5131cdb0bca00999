// Synthetic packed batches and home placement.
//
// sample_lengths follows P/src/workload.cpp:20-84 (draw order, libstdc++
// distributions on a mt19937_64 seeded with the distribution seed, final
// document truncated to hit the total). sequential_items is
// place_sequential + chunk_items (P/src/workload.cpp:86-124,
// P/src/types.cpp:117-132): device k owns tokens [k*T, (k+1)*T) of the
// concatenated documents and every document segment on a device becomes one
// contiguous item homed there.
#include <algorithm>
#include <random>

#include "cad_host.hpp"

namespace cad {
namespace {

i64 clip_length(double x, i64 cap) {
  if (!(x >= 1.0)) return 1;
  if (x >= static_cast<double>(cap)) return cap;
  return static_cast<i64>(x);
}

i64 draw_length(const LengthDist& d, std::mt19937_64& gen) {
  switch (d.kind) {
    case Dist::fixed:
      return std::min(d.fixed_len, d.max_doc_len);
    case Dist::uniform: {
      std::uniform_int_distribution<i64> pick(std::max<i64>(1, d.uniform_min), d.max_doc_len);
      return pick(gen);
    }
    case Dist::histogram: {
      double mass = 0;
      for (const auto& bin : d.histogram) mass += bin.second;
      std::uniform_real_distribution<double> pick(0.0, mass);
      double r = pick(gen);
      for (const auto& bin : d.histogram) {
        r -= bin.second;
        if (r <= 0) return std::clamp<i64>(bin.first, 1, d.max_doc_len);
      }
      return std::clamp<i64>(d.histogram.back().first, 1, d.max_doc_len);
    }
    case Dist::pretrain_upsampled:
    case Dist::prolong_like: {
      // The three distribution objects are constructed per draw exactly as
      // the reference does; libstdc++'s lognormal keeps a cached normal
      // deviate inside each object, so their lifetime matters.
      std::lognormal_distribution<double> body(d.log_mu, d.log_sigma);
      std::lognormal_distribution<double> tail(d.long_log_mu, d.long_log_sigma);
      std::uniform_real_distribution<double> coin(0.0, 1.0);
      const bool mixed = d.kind == Dist::prolong_like;
      for (int tries = 0; tries < 4096; ++tries) {
        const double x = (mixed && coin(gen) < d.long_weight) ? tail(gen) : body(gen);
        if (x > static_cast<double>(d.max_doc_len)) continue;
        const i64 len = clip_length(x, d.max_doc_len);
        if (len < d.min_len_threshold && coin(gen) < d.drop_prob) continue;
        return len;
      }
      return d.max_doc_len;
    }
  }
  throw ConfigError("unknown distribution kind");
}

}  // namespace

std::vector<i64> sample_lengths(const LengthDist& d, i64 total) {
  if (total < 1) throw DomainError("total_tokens must be >= 1");
  if (d.kind == Dist::histogram && d.histogram.empty())
    throw ConfigError("custom_histogram distribution has no entries");
  std::mt19937_64 gen(d.seed);
  std::vector<i64> out;
  i64 filled = 0;
  while (filled < total) {
    const i64 len = std::min(draw_length(d, gen), total - filled);
    out.push_back(len);
    filled += len;
  }
  return out;
}

std::vector<Item> sequential_items(const std::vector<i64>& lengths, i64 devices,
                                   i64 per_device) {
  if (per_device < 1 || devices < 1) throw ConfigError("pack_fixed: chunk shape must be positive");
  i64 sum = 0;
  for (i64 l : lengths) sum += l;
  if (sum != per_device * devices)
    throw ConfigError("pack_fixed: token total does not match chunk layout");
  // Walk the concatenation once, cutting at device boundaries; items come
  // out grouped by device in ascending order, as chunk_items emits them.
  std::vector<Item> items;
  i64 dev = 0, room = per_device;
  for (std::size_t doc = 0; doc < lengths.size(); ++doc) {
    i64 at = 0;
    while (at < lengths[doc]) {
      if (room == 0) {
        ++dev;
        room = per_device;
      }
      const i64 take = std::min(room, lengths[doc] - at);
      Item it;
      it.doc = static_cast<i64>(doc);
      it.q_begin = at;
      it.q_end = at + take;
      it.kv_extent = at + take;
      it.home = static_cast<std::int32_t>(dev);
      items.push_back(it);
      at += take;
      room -= take;
    }
  }
  return items;
}

}  // namespace cad
