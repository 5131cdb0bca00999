"""BASELINE config 5 on the host: max/mean causal-pair load across 8 GPUs for
naive per-chunk placement (place_sequential, = the reference's assign_fixed,
P/src/baselines.cpp:29-43) vs the bit-exact scheduler (P/src/scheduler.cpp:
196-357), 8B shape, 512K tokens, per distribution and seed.
Also config 4 (34B, 1M tokens) at 2/4/8 GPUs. Writes profiles/r1_imbalance_sweep.json.
Usage: imbalance_sweep.py [out.json]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_18121_b200 import configs as CF  # noqa: E402
from paper_2510_18121_b200 import scheduler as S  # noqa: E402


def pairs_per_server(plan, n):
    load = [0] * n
    for t in plan.tasks:
        it = t.item
        load[t.assigned_server] += S.exact_causal_pairs(it.q_end - it.q_begin, it.q_end)
    return load


def naive_pairs(items, n):
    load = [0] * n
    for it in items:
        load[it.home_device] += S.exact_causal_pairs(it.q_end - it.q_begin, it.q_end)
    return load


def ratio(load):
    return max(load) / (sum(load) / len(load))


def case(shape, dist, total, n):
    lengths = S.sample_batch(dist, total)
    items = S.place_sequential(lengths, n, total // n)
    t0 = time.perf_counter()
    plan = S.schedule(items, n, CF.sched_config(shape))
    ms = (time.perf_counter() - t0) * 1e3
    return {"docs": len(lengths), "tasks": len(plan.tasks), "migrations": plan.migrations,
            "naive_max_over_mean_pairs": round(ratio(naive_pairs(items, n)), 4),
            "scheduled_max_over_mean_pairs": round(ratio(pairs_per_server(plan, n)), 4),
            "schedule_ms": round(ms, 3), "total_comm_bytes_ref": plan.total_comm_bytes}


def main():
    out = {"what": "max/mean causal pairs per GPU, naive placement vs scheduler (config 5: 8B, 512K, 8 GPUs; "
                   "config 4: 34B, 1M tokens)", "cfg5": {}, "cfg4": {}}
    for kind, seeds in (("pretrain", range(1, 31)), ("uniform", range(1, 6)), ("fixed", range(1, 3)),
                        ("lognormal", range(1, 6)), ("prolong", range(1, 6))):
        rows = {s: case(CF.LLAMA8B, CF.length_dist(kind, s), 524288, 8) for s in seeds}
        out["cfg5"][kind] = rows
        nv = [r["naive_max_over_mean_pairs"] for r in rows.values()]
        sc = [r["scheduled_max_over_mean_pairs"] for r in rows.values()]
        print(f"cfg5 {kind:9s} seeds {min(seeds)}-{max(seeds)}: naive {min(nv):.3f}-{max(nv):.3f} "
              f"-> scheduled {min(sc):.4f}-{max(sc):.4f}")
    for n in (2, 4, 8):
        rows = {s: case(CF.LLAMA34B, CF.length_dist("pretrain", s, max_doc_len=262144), 1 << 20, n) for s in (1, 2, 3)}
        out["cfg4"][n] = rows
        print(f"cfg4 {n} GPUs: " + ", ".join(f"seed {s}: {r['naive_max_over_mean_pairs']:.3f} -> "
                                            f"{r['scheduled_max_over_mean_pairs']:.4f}" for s, r in rows.items()))
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "profiles", "r1_imbalance_sweep.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
