#!/usr/bin/env python
"""Benchmark of the B200-native DistCA core-attention (CA) hot path.

Metric (BASELINE.json): CA fwd+bwd TFLOP/s per GPU at 1/2/4/8 B200 (% BF16
peak); max/mean CA load imbalance. A step is one layer of CA forward +
backward over one synthetic packed batch:
  N=1  config 2: Llama-3-8B CA (32 Q / 8 KV heads, d=128), 131072 packed
       tokens, pretrain_upsampled doc lengths (seed 1), bf16.
  N>1  config 3 shape, weak scaling: 65536 tokens per GPU placed
       sequentially, CA-tasks sharded by the (reference-exact) scheduler,
       Q/KV dispatch + O return (forward) and dO dispatch + dQ/dK/dV return
       (backward) over NCCL all-to-allv, ping-pong across two nano-batches.
FLOPs are algorithmic: 14 * d * H_q * sum(causal pairs).

`value` is the whole-job TFLOP/s (all ranks), timed with CUDA events on the
launching stream, max over ranks. `e2e` is the same metric through the
public API with host (pinned) inputs copied in and gradients copied out
inside the timed region. `--impl reference` times the reference CPU path
(the CA numerics only exist as our C oracle port, oracle/ca_oracle.c, since
the reference is an analytical simulator) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("CA fwd+bwd TFLOP/s per GPU at 1/2/4/8 B200 (% BF16 peak); "
          "max/mean CA load imbalance")
SEED = 1


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk["bf16_tflops"], pk.get("bf16_tflops_sustained") or pk["bf16_tflops"], "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.rows[0][2]) if self.rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------------------- CPU legs
def cpu_sample_tasks():
    """Bounded CPU sample of the config-2 workload: one KV-head group (4 query
    heads of one KV head) of the batch's first documents, cut to 6144 tokens."""
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import scheduler as S
    lengths = S.sample_batch(CF.length_dist("pretrain", SEED), 131072)
    cut, out = 6144, []
    for l in lengths:
        take = min(l, cut - sum(out))
        if take <= 0:
            break
        out.append(take)
    return out


def run_cpu_oracle(lengths, h_q=4, h_kv=1, threads=0, reps=1):
    """Times the oracle fwd+bwd; returns (TFLOP/s, seconds, threads)."""
    import numpy as np
    import oracle
    T = sum(lengths)
    tasks, off = [], 0
    for l in lengths:
        tasks.append((off, l, off, l))
        off += l
    rng = np.random.default_rng(0)
    q = rng.standard_normal((T, h_q, 128), dtype=np.float32)
    k = rng.standard_normal((T, h_kv, 128), dtype=np.float32)
    v = rng.standard_normal((T, h_kv, 128), dtype=np.float32)
    do = rng.standard_normal((T, h_q, 128), dtype=np.float32)
    nthreads = threads or oracle.num_lib().oracle_max_threads()
    t0 = time.perf_counter()
    for _ in range(reps):
        o, _lse = oracle.ca_forward(tasks, q, k, v, threads=nthreads)
        oracle.ca_backward(tasks, q, k, v, o, do, threads=nthreads)
    dt = (time.perf_counter() - t0) / reps
    pairs = sum(l * (l + 1) // 2 for l in lengths)
    flops = 14.0 * 128 * h_q * pairs
    return flops / dt / 1e12, dt, nthreads


def reference_arm(args, rank):
    """--impl reference: the reference's CPU path on the host cores."""
    if rank != 0:
        return
    lengths = cpu_sample_tasks()[:1]
    lengths = [min(lengths[0], 2048)]
    vals, nth = [], 0
    for i in range(args.warmup + args.steps):
        tf, dt, nth = run_cpu_oracle(lengths)
        if i >= args.warmup:
            vals.append((tf, dt))
    tf = statistics.mean(v[0] for v in vals)
    ms = statistics.mean(v[1] for v in vals) * 1e3
    sample = (f"oracle port (oracle/ca_oracle.c, fp32 IO/fp64 accumulate) fwd+bwd of one {lengths[0]}-token "
              f"document, 4 query heads / 1 KV head, d=128, per step")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": tf, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic",
        "config": {"workload": "config 2 sample (CPU-bounded)", "sample": sample},
        "cpu_baseline": {"value": tf, "unit": "TFLOP/s", "cores": nth,
                         "kind": "port", "sample": sample},
        "e2e": {"value": tf, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# --------------------------------------------------------------------------- GPU, N=1
def time_region(fn, steps, stream):
    import torch
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    st.record(stream)
    for _ in range(steps):
        fn()
    en.record(stream)
    torch.cuda.synchronize()
    return st.elapsed_time(en) / steps


def single_gpu(args):
    import torch
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import scheduler as S
    from paper_2510_18121_b200.ca import BWD_DELTA, BWD_DKDV, BWD_DQ, CAPlan, CATaskRows

    shape = CF.LLAMA8B
    lengths = S.sample_batch(CF.length_dist("pretrain", SEED), 131072)
    T = sum(lengths)
    tasks, off = [], 0
    for l in lengths:
        tasks.append(CATaskRows(off, l, off, l))
        off += l
    plan = CAPlan(tasks, shape.h_q, shape.h_kv, T, T)
    flops = CF.ca_flops(shape, plan.causal_pairs)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    q = torch.randn(T, shape.h_q, 128, device=dev, dtype=torch.bfloat16, generator=g)
    k = torch.randn(T, shape.h_kv, 128, device=dev, dtype=torch.bfloat16, generator=g)
    v = torch.randn(T, shape.h_kv, 128, device=dev, dtype=torch.bfloat16, generator=g)
    do = torch.randn(T, shape.h_q, 128, device=dev, dtype=torch.bfloat16, generator=g)
    o = torch.empty_like(q)
    lse = torch.empty(shape.h_q, T, device=dev)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    def step():
        plan.forward(q, k, v, o, lse)
        plan.backward(q, k, v, o, lse, do, dq, dk, dv, ws)

    for _ in range(args.warmup):
        step()
    clocks = ClockSampler(0)
    clocks.start()
    ms = time_region(step, args.steps, stream)
    clk = clocks.stop()

    # per-kernel breakdown (same stream, events; outside the headline region)
    reps = max(2, min(5, args.steps))
    parts = {
        "ca_fwd": (lambda: plan.forward(q, k, v, o, lse), flops["fwd"], flops["fwd"]),
        "ca_delta": (lambda: plan.backward(q, k, v, o, lse, do, dq, dk, dv, ws, parts=BWD_DELTA), 0.0, 0.0),
        "ca_bwd_dkdv": (lambda: plan.backward(q, k, v, o, lse, do, dq, dk, dv, ws, parts=BWD_DKDV),
                        0.8 * flops["bwd"], 0.8 * flops["bwd"]),
        "ca_bwd_dq": (lambda: plan.backward(q, k, v, o, lse, do, dq, dk, dv, ws, parts=BWD_DQ),
                      0.2 * flops["bwd"], 0.6 * flops["bwd"]),
    }
    kernels = {}
    for name, (fn, alg, exe) in parts.items():
        kms = time_region(fn, reps, stream)
        kernels[name] = {"ms": kms, "alg_tflops": alg / kms / 1e9 if alg else None,
                         "executed_tflops": exe / kms / 1e9 if exe else None}

    # end to end through the public API: pinned host inputs in, grads out
    hq, hk, hv, hdo = (t.cpu().pin_memory() for t in (q, k, v, do))
    hdq, hdk, hdv = (torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in (dq, dk, dv))
    h2d = sum(t.numel() * t.element_size() for t in (hq, hk, hv, hdo))
    d2h = sum(t.numel() * t.element_size() for t in (hdq, hdk, hdv))

    # Double-buffered: step j's inputs go host -> device on a copy stream while
    # step j-1 computes, and step j's gradients come back while step j+1
    # computes; every step still moves its own inputs and results.
    sets = [(q, k, v, do, o, lse, dq, dk, dv),
            tuple(torch.empty_like(t) for t in (q, k, v, do, o, lse, dq, dk, dv))]
    copy = torch.cuda.Stream(device=dev)

    def e2e_run(n):
        ev = torch.cuda.Event
        h2d_done, comp_done = [None, None], [None, None]
        st, en = ev(enable_timing=True), ev(enable_timing=True)
        torch.cuda.synchronize()
        st.record(copy)
        for j in range(n + 1):
            if j < n:  # inputs of step j
                b = sets[j % 2]
                if comp_done[j % 2] is not None:
                    copy.wait_event(comp_done[j % 2])  # step j-2 done with this set
                with torch.cuda.stream(copy):
                    for dst, src in zip(b[:4], (hq, hk, hv, hdo)):
                        dst.copy_(src, non_blocking=True)
                h2d_done[j % 2] = ev()
                h2d_done[j % 2].record(copy)
            if j >= 1:  # results of step j-1
                with torch.cuda.stream(copy):
                    copy.wait_event(comp_done[(j - 1) % 2])
                    b = sets[(j - 1) % 2]
                    for dst, src in zip((hdq, hdk, hdv), b[6:]):
                        dst.copy_(src, non_blocking=True)
            if j < n:  # compute step j
                b = sets[j % 2]
                stream.wait_event(h2d_done[j % 2])
                plan.forward(b[0], b[1], b[2], b[4], b[5])
                plan.backward(b[0], b[1], b[2], b[4], b[5], b[3], b[6], b[7], b[8], ws)
                comp_done[j % 2] = ev()
                comp_done[j % 2].record(stream)
        en.record(copy)
        torch.cuda.synchronize()
        return st.elapsed_time(en) / n

    e2e_run(2)
    e2e_ms = e2e_run(max(3, args.steps))  # first upload and last download amortised over the K steps

    peak, peak_sus, peak_kind = load_peaks()
    value = flops["total"] / ms / 1e9
    dom = max(kernels, key=lambda n: kernels[n]["ms"])
    dk_ = kernels[dom]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(dom)
    except Exception:
        pass
    roof = {"kernel": dom, "bound": "tensor", "achieved": dk_["alg_tflops"], "peak": peak, "unit": "TFLOP/s",
            "frac": (dk_["alg_tflops"] or 0) / peak, "traffic": traffic, "peak_kind": peak_kind,
            "executed_tflops": dk_["executed_tflops"],
            # the kernel repeats back to back for ~1 s: the sustained peak is the
            # power-capped ceiling it actually runs under
            "peak_sustained": peak_sus, "frac_sustained": (dk_["alg_tflops"] or 0) / peak_sus}

    cpu = None
    if not args.no_cpu:
        sample = cpu_sample_tasks()
        tf, dt, nth = run_cpu_oracle(sample)
        cpu = {"value": tf, "unit": "TFLOP/s", "cores": nth, "kind": "port",
               "sample": f"oracle fwd+bwd of docs {sample} (first 6144 tokens of the batch), "
                         f"4 query heads of 1 KV head, {dt:.1f} s"}
        # reference scheduler on the same batch (the reference's own CPU code)
        try:
            cpu["scheduler_ms_ref"] = ref_scheduler_ms(lengths, 1, shape)
        except Exception as e:  # reference library absent
            cpu["scheduler_ms_ref"] = f"unavailable: {e}"

    out = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "BASELINE config 2: Llama-3-8B CA (32 Q / 8 KV heads, d=128), 131072 packed "
                               "tokens, pretrain_upsampled docs seed 1, one layer fwd+bwd",
                   "docs": lengths, "causal_pairs": plan.causal_pairs, "flops_per_step": flops["total"],
                   "l2": "inputs larger than L2 (Q alone is 1 GiB)", "parallelism": "single GPU"},
        "per_gpu_tflops": value, "pct_bf16_peak": value / peak, "pct_bf16_peak_sustained": value / peak_sus,
        "tokens_per_s": T / (ms / 1e3),
        "imbalance": {"max_over_mean_pairs": 1.0, "max_over_mean_time": 1.0},
        "roofline": roof, "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": {"value": flops["total"] / e2e_ms / 1e9, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": 4 * args.steps,
        "clocks": clk,
    }
    print(json.dumps(out))


def ref_scheduler_ms(lengths, n_gpus, shape):
    import ctypes as C
    import oracle
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import scheduler as S
    from paper_2510_18121_b200 import _native as N
    T = sum(lengths)
    items = S.place_sequential(lengths, n_gpus, T // n_gpus)
    arr = (N.cad_item * len(items))(*[i.to_c() for i in items])
    reps = 200
    secs = oracle.ref_lib().ref_schedule_seconds(arr, len(items), n_gpus, C.byref(CF.sched_config(shape).to_c()), reps)
    return secs / reps * 1e3


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cad", choices=["cad", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        reference_arm(args, rank)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        import bench_dist
        bench_dist.run(args, METRIC, load_peaks, ClockSampler)
        return
    single_gpu(args)


if __name__ == "__main__":
    main()
