// The pipeline-parallel tick table: per tick, what every stage works on
// (restates the table construction of simulate_pp_iteration,
// P/src/sim.cpp:297-353). A CA runtime drives one tick at a time: the
// attention of every stage active in the tick is pooled and scheduled with
// schedule_pp_tick (P/src/scheduler.cpp:359-373) and executed as one layer
// pass (cad_layer_step_ex with CAD_PASS_FWD or CAD_PASS_BWD).
//   vanilla 1F1B:    stage s runs forward m at tick s + 2m and backward m at
//                    tick 2S - 1 - s + 2m; 2 (M + S - 1) ticks.
//   phase-synced:    S - 1 forward warm-up phases, then forward/backward
//                    alternating over the M microbatches, then S - 1
//                    backward drain phases; in forward phase f stage s runs
//                    microbatch f - s, in backward phase b microbatch
//                    b - (S - 1 - s) -- every stage of a tick does the same
//                    pass, which is what makes the pooling legal.
#include <vector>

#include "../../../include/cad.h"
#include "cad_host.hpp"
#include "cad_status.hpp"

namespace {

using cad::i64;

std::vector<cad_tick_work> tick_table(i64 M, i64 S, int kind) {
  if (S < 1) throw cad::ConfigError("stages must be >= 1");
  if (M < S) throw cad::ConfigError("1F1B needs at least as many microbatches as stages");
  std::vector<cad_tick_work> t;
  auto at = [&](i64 tick, i64 s) -> cad_tick_work& { return t[static_cast<size_t>(tick * S + s)]; };
  if (kind == CAD_PP_1F1B) {
    const i64 ticks = 2 * (M + S - 1);
    t.assign(static_cast<size_t>(ticks * S), cad_tick_work{0, 0, 0});
    for (i64 s = 0; s < S; ++s)
      for (i64 m = 0; m < M; ++m) {
        at(s + 2 * m, s) = cad_tick_work{1, 0, m};
        at(2 * S - 1 - s + 2 * m, s) = cad_tick_work{1, 1, m};
      }
    return t;
  }
  if (kind != CAD_PP_PHASE_SYNC) throw cad::ConfigError("unknown pipeline schedule");
  struct Phase {
    bool backward;
    i64 index;
  };
  std::vector<Phase> phases;
  for (i64 f = 0; f < S - 1; ++f) phases.push_back({false, f});
  for (i64 k = 0; k < M; ++k) {
    phases.push_back({false, S - 1 + k});
    phases.push_back({true, k});
  }
  for (i64 b = M; b < M + S - 1; ++b) phases.push_back({true, b});
  t.assign(phases.size() * static_cast<size_t>(S), cad_tick_work{0, 0, 0});
  for (size_t k = 0; k < phases.size(); ++k)
    for (i64 s = 0; s < S; ++s) {
      const i64 m = phases[k].backward ? phases[k].index - (S - 1 - s) : phases[k].index - s;
      if (m >= 0 && m < M) at(static_cast<i64>(k), s) = cad_tick_work{1, phases[k].backward ? 1 : 0, m};
    }
  return t;
}

}  // namespace

extern "C" int cad_pp_tick_table(int64_t n_microbatches, int64_t n_stages, int32_t kind, cad_tick_work* out,
                                 int64_t cap, int64_t* n_ticks) {
  return cad::guarded([&] {
    if (!n_ticks) throw cad::DomainError("null argument");
    const auto t = tick_table(n_microbatches, n_stages, kind);
    *n_ticks = static_cast<int64_t>(t.size()) / n_stages;
    if (cap < static_cast<int64_t>(t.size()) || !out) throw cad::CapacityError("tick table buffer too small");
    for (size_t i = 0; i < t.size(); ++i) out[i] = t[i];
  });
}
