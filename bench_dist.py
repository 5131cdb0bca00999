"""N>1 leg of bench.py (launched by torchrun, one process per GPU).

Workload: BASELINE config 3 shape (Llama-3-8B CA, 32 Q / 8 KV heads), 65536
tokens per GPU (512K at 8 GPUs), pretrain_upsampled documents (seed 1),
placed sequentially; CA-tasks sharded by the bit-exact scheduler; per layer
the Q/KV dispatch, CA fwd, O/LSE return, dO dispatch, CA bwd, dQ and dK/dV
return run with ping/pong halves through the C-ABI executor (cad_layer_ctx,
one cad_layer_step call per step): CUDA-IPC copy-engine pushes with GPU
flags (default) and, in the same run, the NCCL all-to-allv transport. A step
is CAD_LAYERS (default 4) stacked CA layers, forward then backward, with the
identity between layers (benchmark mode: dK/dV summed over the layers), so
the transfers of one layer overlap the neighbouring layer's CA compute.
Scaling is weak (fixed tokens per GPU). Times are CUDA events on the compute
stream, max over ranks.
"""
import json
import os

import torch
import torch.distributed as dist


_WORKLOADS = {"cfg3": "BASELINE config 3", "cfg4": "BASELINE config 4", "cfg5": "BASELINE config 5 (imbalance sweep)"}


def _timed(fn, steps, stream):
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dist.barrier()
    torch.cuda.synchronize()
    st.record(stream)
    for _ in range(steps):
        fn()
    en.record(stream)
    torch.cuda.synchronize()
    dist.barrier()
    ms = st.elapsed_time(en) / steps
    t = torch.tensor([ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item(), ms


def _log(msg):
    if os.environ.get("CAD_BENCH_VERBOSE"):
        print(f"[rank {os.environ.get('RANK', '0')}] {msg}", file=__import__("sys").stderr, flush=True)


def run(args, metric, load_peaks, ClockSampler):
    os.environ.setdefault("NCCL_MAX_NCHANNELS", os.environ.get("CAD_NCCL_CHANNELS", "8"))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import dispatch as D
    from paper_2510_18121_b200 import scheduler as S

    # CAD_WORKLOAD: cfg3 (default; 8B, 64K tokens per GPU, weak scaling),
    # cfg4 (34B, 64 Q / 8 KV heads, 1M tokens over the N GPUs: strong
    # scaling, docs up to 256K) or cfg5-<uniform|lognormal|prolong|fixed>
    workload = os.environ.get("CAD_WORKLOAD", "cfg3")
    seed = int(os.environ.get("CAD_SEED", "1"))
    if workload == "cfg4":
        shape, total, scaling = CF.LLAMA34B, 1 << 20, "strong"
        dist_ = CF.length_dist("pretrain", seed, max_doc_len=262144)
    elif workload == "cfg3" or workload.startswith("cfg5-"):
        shape, total, scaling = CF.LLAMA8B, 65536 * world, "weak"
        dist_ = CF.length_dist("pretrain" if workload == "cfg3" else workload[5:], seed)
    else:
        raise ValueError(f"unknown CAD_WORKLOAD {workload!r}")
    per_gpu = total // world
    lengths = S.sample_batch(dist_, total)
    # halves: 0 = the reference's assign_halves split, 1 = evened out per
    # server, 2 = one half (no ping-pong)
    balance = int(os.environ.get("CAD_BALANCE_HALVES", "0"))
    lp = D.LayerPlan(lengths, world, rank, shape, balance_halves=balance)
    layers = int(os.environ.get("CAD_LAYERS", "1" if workload == "cfg4" else "4"))
    dev = torch.device("cuda", local)
    layer = D.DistCALayer(lp, dev, "ipc", layers=layers, balance_halves=balance, bench_stacked=layers > 1)
    H = lp.home_rows
    g = torch.Generator(device=dev).manual_seed(rank)
    bf = dict(device=dev, dtype=torch.bfloat16)
    q = torch.randn(H, shape.h_q, 128, generator=g, **bf)
    k = torch.randn(H, shape.h_kv, 128, generator=g, **bf)
    v = torch.randn(H, shape.h_kv, 128, generator=g, **bf)
    do = torch.randn(H, shape.h_q, 128, generator=g, **bf)
    o = torch.empty_like(q)
    lse = torch.empty(shape.h_q, H, device=dev)
    dq = torch.empty_like(q)
    dk = torch.empty_like(k)
    dv = torch.empty_like(v)
    layer.connect_dist()

    def fill_homes(L):
        # zero-copy: every stacked layer's inputs written once into the
        # context's home buffers (a real stack's projections would write them
        # there); the timed steps then stage nothing in or out
        for l in range(layers):
            hm = L.home(l)
            for name, t in (("q", q), ("k", k), ("v", v), ("do", do)):
                hm[name].copy_(t)

    fill_homes(layer)
    io = layer.io(None, None, None, None, None, None, None, dk, dv)
    comp = torch.cuda.current_stream(dev)

    def step(L=layer, mode="pingpong", io_=None):
        L.step(io_ or io, mode, comp)

    _log("warmup")
    for _ in range(args.warmup):
        step()
    l0 = layer.launches
    clocks = ClockSampler(local)
    clocks.start()
    ms, my_ms = _timed(step, args.steps, comp)
    clk = clocks.stop()
    launches = layer.launches - l0
    n_side = max(2, args.steps // 2)
    _log("compute-only")
    ms_compute, my_compute = _timed(lambda: step(mode="compute"), n_side, comp)
    _log("comm-only")
    ms_comm, _ = _timed(lambda: step(mode="comm"), n_side, comp)
    _log("signal")
    ms_signal, _ = _timed(lambda: step(mode="signal"), n_side, comp)
    _log("comm-local")
    ms_comm_local, _ = _timed(lambda: step(mode="comm_local"), n_side, comp)
    _log("serial")
    ms_serial, _ = _timed(lambda: step(mode="serial"), n_side, comp)

    _log("trace")
    # CAD_TRACE=1: the phase timeline of one ping-pong step on every rank
    traces = None
    if os.environ.get("CAD_TRACE"):
        layer.set_trace(True)
        dist.barrier()
        step()
        torch.cuda.synchronize()
        tr = layer.trace()
        layer.set_trace(False)
        traces = [None] * world
        dist.all_gather_object(traces, tr)

    _log("nccl")
    # NCCL transport (north_star's all-to-allv on a side stream), same
    # schedule and layers, CA grid leaving CAD_NCCL_RESERVE SMs to NCCL
    nccl = None
    # on by default up to 4 GPUs (the sizes it was validated at); CAD_NCCL_LINE=1/0 forces it
    if os.environ.get("CAD_NCCL_LINE", "1" if world <= 4 else "0") != "0":
        reserve = int(os.environ.get("CAD_NCCL_RESERVE", "8"))
        obj = [D.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = D.Comm(obj[0], rank, world)
        ln = D.DistCALayer(lp, dev, "nccl", layers=layers, reserve_sms=reserve, balance_halves=balance,
                           bench_stacked=layers > 1)
        ln.set_comm(comm)
        fill_homes(ln)
        for _ in range(2):
            step(ln)
        n_ms, _ = _timed(lambda: step(ln), max(3, args.steps // 2), comp)
        n_comp, _ = _timed(lambda: step(ln, "compute"), n_side, comp)
        n_comm, _ = _timed(lambda: step(ln, "comm"), n_side, comp)
        n_serial, _ = _timed(lambda: step(ln, "serial"), n_side, comp)
        ln.close()
        comm.close()
        nccl = {"ms_pingpong": n_ms, "ms_compute_only": n_comp, "ms_comm_only": n_comm, "ms_serial": n_serial,
                "reserve_sms": reserve,
                "hidden_fraction": max(0.0, min(1.0, 1.0 - (n_ms - n_comp) / n_comm)) if n_comm > 0 else None}

    _log("e2e")
    # e2e: home inputs from pinned host memory, O/LSE/dQ/dK/dV back to host,
    # double-buffered: step j's inputs go host -> device on a copy stream
    # while step j-1 runs, step j's outputs come back while step j+1 runs.
    # The step stages the inputs into the context's home buffers and its
    # outputs out of them (into the per-set stage buffers) on the compute
    # stream.
    hq_, hk_, hv_, hdo_ = (t.cpu().pin_memory() for t in (q, k, v, do))
    outs = (o, lse, dq, dk, dv)
    host_out = [torch.empty(t.shape, dtype=t.dtype).pin_memory() for t in outs]
    sets = []
    for j in range(2):
        ins = (q, k, v, do) if j == 0 else tuple(torch.empty_like(t) for t in (q, k, v, do))
        stage = tuple(torch.empty_like(t) for t in outs)
        sets.append((ins, stage, layer.io(*ins, stage[0], stage[1], stage[2], stage[3], stage[4])))
    copy = torch.cuda.Stream(device=dev)

    def e2e_run(n):
        ev = torch.cuda.Event
        h2d_done, comp_done = [None, None], [None, None]
        st, en = ev(enable_timing=True), ev(enable_timing=True)
        dist.barrier()
        torch.cuda.synchronize()
        st.record(copy)
        for j in range(n + 1):
            if j < n:  # inputs of step j
                ins, _, _ = sets[j % 2]
                if comp_done[j % 2] is not None:
                    copy.wait_event(comp_done[j % 2])
                with torch.cuda.stream(copy):
                    for dst, src in zip(ins, (hq_, hk_, hv_, hdo_)):
                        dst.copy_(src, non_blocking=True)
                h2d_done[j % 2] = ev()
                h2d_done[j % 2].record(copy)
            if j >= 1:  # outputs of step j-1
                with torch.cuda.stream(copy):
                    copy.wait_event(comp_done[(j - 1) % 2])
                    for dst, src in zip(host_out, sets[(j - 1) % 2][1]):
                        dst.copy_(src, non_blocking=True)
            if j < n:  # step j
                _, stage, io_j = sets[j % 2]
                comp.wait_event(h2d_done[j % 2])
                step(io_=io_j)
                comp_done[j % 2] = ev()
                comp_done[j % 2].record(comp)
        en.record(copy)
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([st.elapsed_time(en) / n], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    e2e_run(2)
    ms_e2e = e2e_run(max(3, args.steps))

    _log("probe")
    # NVLink probe: one half's forward dispatch (Q + K/V rows this rank pushes
    # into its peers' buffers) alone on a stream, own rows on another stream;
    # achieved GB/s = remote bytes / time of the pushes, per rank
    ps, loc = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    probe = []
    for h in (0, 1):
        nbytes = layer.wire_bytes[h][0] + 2 * layer.wire_bytes[h][1]
        ms_h = []
        for _ in range(3):
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ps)
            layer.dispatch(0, h, D.DISPATCH_QKV, io, ps, loc)
            e1.record(ps)
            torch.cuda.synchronize()
            ms_h.append(e0.elapsed_time(e1))
        probe.append((nbytes, min(ms_h)))
    dist.barrier()
    probes = [None] * world
    dist.all_gather_object(probes, probe)

    h2d = sum(t.numel() * t.element_size() for t in (hq_, hk_, hv_, hdo_)) * world
    d2h = sum(t.numel() * t.element_size() for t in host_out) * world
    pairs = layer.served_pairs
    wire = sum(layer.wire_bytes[h][0] * 2 + layer.wire_bytes[h][1] * 2 + layer.wire_bytes[h][2] * 2
               + layer.wire_bytes[h][3] * 2 for h in (0, 1)) * layers
    stats = torch.tensor([pairs, my_compute, wire, my_ms], dtype=torch.float64, device=dev)
    allst = [torch.zeros_like(stats) for _ in range(world)]
    dist.all_gather(allst, stats)
    allst = torch.stack(allst).cpu().numpy()
    if rank == 0:
        peak, peak_sus, peak_kind = load_peaks()
        total_pairs = allst[:, 0].sum()
        flops = 14.0 * 128 * shape.h_q * total_pairs * layers
        value = flops / ms / 1e9
        # hidden = 1 - (T_pingpong - T_signal) / T_wire (the
        # reference's signal/ping-pong modes, P/tests/acceptance.cpp:272-290):
        # signal = the same step with every transfer to a peer shrunk to its
        # flag; T_wire = the peer transfers alone (comm-only minus comm-only
        # without them). hidden_all also charges the rank's own row copies,
        # the dK/dV reduction and the kernels' slowdown under concurrent
        # copies against all data movement: 1 - (T_pp - T_compute) / T_comm.
        wire_ms = ms_comm - ms_comm_local
        hidden = max(0.0, min(1.0, 1.0 - (ms - ms_signal) / wire_ms)) if wire_ms > 0 else None
        hidden_vs_compute = max(0.0, min(1.0, 1.0 - (ms - ms_compute) / ms_comm)) if ms_comm > 0 else None
        naive_pairs = []
        for r in range(world):
            its = [it for it in lp.home_items if it.home_device == r]
            naive_pairs.append(sum(S.exact_causal_pairs(it.q_end - it.q_begin, it.q_end) for it in its))
        out = {
            "metric": metric, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{_WORKLOADS[workload.split('-')[0]]}: {shape.name} CA ({shape.h_q} Q / {shape.h_kv} KV), "
                                   f"{per_gpu} tokens per GPU ({total} total), "
                                   f"{'pretrain_upsampled' if workload in ('cfg3', 'cfg4') else workload[5:]} lengths seed {seed}, scheduler-sharded, "
                                   "copy-engine (CUDA IPC) pushes through cad_layer_step, "
                                   f"ping-pong halves, {layers} stacked CA layer(s) fwd+bwd per step "
                                   "(identity between layers)",
                       "workload_id": workload, "layers_per_step": layers,
                       "halves": ["reference assign_halves", "balanced per server", "one half (no ping-pong)"][balance],
                       "docs": len(lengths), "tasks": len(lp.plan.tasks), "migrations": lp.plan.migrations,
                       "flops_per_step": flops, "l2": "inputs larger than L2",
                       "parallelism": f"CA servers x{world} (scheduler sharding)", "transport": "ipc"},
            "per_gpu_tflops": value / world, "pct_bf16_peak": value / world / peak,
            "tokens_per_s": per_gpu * world * layers / (ms / 1e3),  # token-layers (fwd+bwd) per second
            "imbalance": {"max_over_mean_pairs": float(allst[:, 0].max() / allst[:, 0].mean()),
                          "max_over_mean_ca_time": float(allst[:, 1].max() / allst[:, 1].mean()),
                          "naive_max_over_mean_pairs": max(naive_pairs) / (sum(naive_pairs) / world)},
            "comm": {"ms_compute_only": ms_compute, "ms_signal": ms_signal, "ms_comm_only": ms_comm,
                     "ms_comm_local_only": ms_comm_local, "ms_wire": wire_ms,
                     "ms_serial": ms_serial, "ms_pingpong": ms, "hidden_fraction": hidden,
                     # the peer transfers' cost as the step sees it: ping-pong minus the same
                     # step with every peer transfer shrunk to its flag
                     "exposed_wire_ms": ms - ms_signal, "exposed_wire_share_of_step": (ms - ms_signal) / ms,
                     "hidden_fraction_all_movement": hidden_vs_compute,
                     "nccl": nccl,
                     "wire_bytes_per_step_max_rank": float(allst[:, 2].max()),
                     "nvlink_gbs_per_gpu": float(allst[:, 2].max()) / (ms_comm / 1e3) / 1e9 if ms_comm else None,
                     # per rank and half: a forward dispatch pushed alone (copy engines, peer
                     # memory over NVLink), remote bytes / time, against 900 GB/s per direction
                     "nvlink_probe_gbs": [[round(b / (t / 1e3) / 1e9, 1) if t > 0 and b > 0 else None
                                           for (b, t) in pr] for pr in probes],
                     "nvlink_probe_bytes": [[b for (b, t) in pr] for pr in probes],
                     "nvlink_link_gbs": 900.0,
                     "ref_total_comm_bytes": lp.plan.total_comm_bytes},
            "roofline": {"kernel": "ca fwd+bwd (4 launches per half)", "bound": "tensor",
                         "achieved": flops / world / ms_compute / 1e9, "peak": peak, "unit": "TFLOP/s",
                         "frac": flops / world / ms_compute / 1e9 / peak, "traffic": None, "peak_kind": peak_kind},
            "cpu_baseline": None,
            "e2e": {"value": flops / ms_e2e / 1e9, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": ms_e2e},
            "gpu_launches": launches,
            "clocks": clk,
        }
        if traces is not None:
            out["trace_ranks"] = {"columns": ["phase", "layer", "half", "t_begin_ms", "t_ready_ms", "t_end_ms"],
                                  "ranks": traces}
        print(json.dumps(out))
    layer.close()
    dist.barrier()
    dist.destroy_process_group()
