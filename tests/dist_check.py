"""torchrun script: the distributed CA layer (C-ABI executor cad_layer_ctx,
IPC copy-engine pushes or NCCL all-to-allv, ping-pong and serial steps)
against the CPU oracle on the whole batch. Prints one JSON line of errors per
rank and exits non-zero on a mismatch.
    torchrun --nproc-per-node 2 tests/dist_check.py [tokens_per_gpu]
Env: CAD_TRANSPORT=ipc|nccl, CAD_LAYERS=L (stacked benchmark layers: every
layer sees the same inputs, so O/LSE/dQ match one layer and dK/dV are L x)."""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)
import numpy as np
import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import oracle
    from ca_cases import GRAD_TOL, LSE_ABS, O_ABS, error_report
    from dist_sim import home_arrays
    from layer_local import bf16_round
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import dispatch as D
    from paper_2510_18121_b200 import scheduler as S
    per = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    shape = CF.Shape("check", 8, 2)
    lengths = S.sample_batch(CF.length_dist("pretrain", 3, max_doc_len=per), per * world)
    transport = os.environ.get("CAD_TRANSPORT", "ipc")
    layers = int(os.environ.get("CAD_LAYERS", "1"))
    plans = [D.LayerPlan(lengths, world, r, shape) for r in range(world)]
    lp = plans[rank]
    dev = torch.device("cuda", local)
    layer = D.DistCALayer(lp, dev, transport, layers=layers, reserve_sms=8 if transport == "nccl" else 0,
                          bench_stacked=layers > 1)
    rng = np.random.default_rng(5)
    per_doc = {n: [bf16_round(rng.standard_normal((l, h, 128), dtype=np.float32)) for l in lengths]
               for n, h in (("q", shape.h_q), ("k", shape.h_kv), ("v", shape.h_kv), ("do", shape.h_q))}
    home = {n: torch.from_numpy(home_arrays(plans, lengths, per_doc[n])[rank]).to(torch.bfloat16).to(dev)
            for n in per_doc}
    H = lp.home_rows
    o = torch.empty_like(home["q"])
    lse = torch.empty(shape.h_q, H, device=dev)
    dq = torch.empty_like(home["q"])
    dk = torch.empty_like(home["k"])
    dv = torch.empty_like(home["v"])
    comm = None
    if transport == "nccl":
        obj = [D.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = D.Comm(obj[0], rank, world)
        layer.set_comm(comm)
    else:
        layer.bind_outputs(o, lse, dq)
        layer.connect_dist()
    io = layer.io(home["q"], home["k"], home["v"], home["do"], o, lse, dq, dk, dv)
    results = {}
    for mode in ("pingpong", "serial", "pingpong"):
        o.fill_(float("nan")); dq.fill_(float("nan")); lse.fill_(float("nan"))
        layer.step(io, mode)
        torch.cuda.synchronize()
        results[mode] = {n: t.float().cpu().numpy() for n, t in (("o", o), ("lse", lse), ("dq", dq), ("dk", dk),
                                                                  ("dv", dv))}
    if layers == 1:
        # a forward-only step, then a backward-only step that re-dispatches Q/K/V
        # and the forward state (O, LSE) with dO: the two passes of a pipeline tick
        o.fill_(float("nan")); dq.fill_(float("nan")); lse.fill_(float("nan"))
        layer.step(io, "pingpong", passes="fwd")
        torch.cuda.synchronize()
        fwd_o, fwd_lse = o.float().cpu().numpy(), lse.cpu().numpy()
        layer.step(io, "pingpong", passes="bwd")
        torch.cuda.synchronize()
        results["split-passes"] = {"o": fwd_o, "lse": fwd_lse, "dq": dq.float().cpu().numpy(),
                                   "dk": dk.float().cpu().numpy(), "dv": dv.float().cpu().numpy()}
    # the CPU oracle on the whole batch (every document one task), in this rank's home rows
    tasks, off = [], 0
    for l in lengths:
        tasks.append((off, l, off, l))
        off += l
    cat = {n: np.concatenate(per_doc[n]) for n in per_doc}
    ro, rlse = oracle.ca_forward(tasks, cat["q"], cat["k"], cat["v"])
    rdq, rdk, rdv = oracle.ca_backward(tasks, cat["q"], cat["k"], cat["v"], bf16_round(ro), cat["do"])
    cuts = np.cumsum(lengths)[:-1]
    ref = {n: home_arrays(plans, lengths, np.split(a, cuts))[rank]
           for n, a in (("o", ro), ("dq", rdq), ("dk", rdk * layers), ("dv", rdv * layers), ("lse", rlse.T))}
    err, ok = {}, True
    for mode, out in results.items():
        for n in ("o", "lse", "dq", "dk", "dv"):
            got = out[n].T if n == "lse" else out[n]
            rep = error_report(n, got, ref[n])
            key = f"{mode}:{n}"
            err[key] = {"abs": rep["abs"], "row_rel": rep["row_rel"]}
            good = np.isfinite(got).all() and (
                rep["abs"] <= O_ABS if n == "o" else rep["abs"] <= LSE_ABS if n == "lse" else
                rep["row_rel"] <= GRAD_TOL)
            ok = ok and bool(good)
    print(json.dumps({"rank": rank, "transport": transport, "layers": layers, "migrations": lp.plan.migrations,
                      "launches": layer.launches, "errors": err, "ok": ok}), flush=True)
    layer.close()
    if comm is not None:
        comm.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
