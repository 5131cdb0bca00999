"""A world-W CA layer on ONE GPU through the C-ABI executor (cad_layer_ctx,
CAD_TRANSPORT_LOCAL): every rank's context lives in this process, its home and
server buffers on cuda:0, and the rows move by the same push/flag code the
IPC transport uses across GPUs (cad_copy_runs, cad_copy_runs_cols,
cuStreamWriteValue32/WaitValue32, cad_scatter_add_bf16, cad_f32_to_bf16).
Returns each rank's home outputs next to the CPU oracle's whole-batch result
laid out in the same home rows (dist_sim.home_arrays)."""
import numpy as np
import torch

import oracle
from dist_sim import home_arrays


def bf16_round(x):
    return torch.from_numpy(x).to(torch.bfloat16).float().numpy()


def run_local(lengths, world, shape, seed=0, items=None, cfg=None, tokens_per_device=None):
    """The per-layer entry points (cad_layer_begin, cad_dispatch,
    cad_layer_compute, cad_return, cad_layer_finish) called rank by rank in
    dependency order on one stream."""
    from paper_2510_18121_b200 import dispatch as D
    dev = torch.device("cuda", 0)
    plans = [D.LayerPlan(lengths, world, r, shape, cfg=cfg, items=items, tokens_per_device=tokens_per_device)
             for r in range(world)]
    hq, hkv, d = shape.h_q, shape.h_kv, shape.head_dim
    rng = np.random.default_rng(seed)
    per = {n: [bf16_round(rng.standard_normal((l, h, d), dtype=np.float32)) for l in lengths]
           for n, h in (("q", hq), ("k", hkv), ("v", hkv), ("do", hq))}
    home = {n: home_arrays(plans, lengths, per[n]) for n in per}
    layers = [D.DistCALayer(plans[r], dev, "local") for r in range(world)]
    bufs, ios = [], []
    for r in range(world):
        H = layers[r].home_rows
        assert H == plans[r].home_rows
        b = {n: torch.from_numpy(home[n][r]).to(torch.bfloat16).to(dev) for n in home}
        b["o"] = torch.full((H, hq, d), float("nan"), dtype=torch.bfloat16, device=dev)
        b["lse"] = torch.full((hq, H), float("nan"), device=dev)
        b["dq"] = torch.full((H, hq, d), float("nan"), dtype=torch.bfloat16, device=dev)
        b["dk"] = torch.empty(H, hkv, d, dtype=torch.bfloat16, device=dev)
        b["dv"] = torch.empty(H, hkv, d, dtype=torch.bfloat16, device=dev)
        layers[r].bind_outputs(b["o"], b["lse"], b["dq"])
        bufs.append(b)
        ios.append(layers[r].io(b["q"], b["k"], b["v"], b["do"], b["o"], b["lse"], b["dq"], b["dk"], b["dv"]))
    blobs = [L.export() for L in layers]
    for L in layers:
        L.connect(blobs)
    s = torch.cuda.current_stream(dev)
    for L in layers:
        L.begin(s)
    for what, bwd, ret in ((D.DISPATCH_QKV, False, D.RETURN_O), (D.DISPATCH_DO, True, D.RETURN_GRAD)):
        for h in (0, 1):
            for r, L in enumerate(layers):
                L.dispatch(0, h, what, ios[r], s)
        for h in (0, 1):
            for L in layers:
                L.compute(0, h, bwd, s)
        for h in (0, 1):
            for r, L in enumerate(layers):
                L.ret(0, h, ret, ios[r], s)
    for r, L in enumerate(layers):
        L.finish(ios[r], s)
    torch.cuda.synchronize()
    out = {n: [bufs[r][n].float().cpu().numpy() for r in range(world)] for n in ("o", "lse", "dq", "dk", "dv")}
    launches = sum(L.launches for L in layers)
    for L in layers:
        L.close()
    # CPU oracle on the whole batch (every document one task)
    tasks, off = [], 0
    for l in lengths:
        tasks.append((off, l, off, l))
        off += l
    cat = {n: np.concatenate(per[n]) for n in per}
    o, lse = oracle.ca_forward(tasks, cat["q"], cat["k"], cat["v"])
    dq, dk, dv = oracle.ca_backward(tasks, cat["q"], cat["k"], cat["v"], bf16_round(o), cat["do"])
    cuts = np.cumsum(lengths)[:-1]
    ref_doc = {"o": np.split(o, cuts), "dq": np.split(dq, cuts), "dk": np.split(dk, cuts),
               "dv": np.split(dv, cuts), "lse": np.split(lse.T, cuts)}
    ref = {n: home_arrays(plans, lengths, ref_doc[n]) for n in ref_doc}
    ref["lse"] = [x.T for x in ref["lse"]]
    return out, ref, plans, launches
