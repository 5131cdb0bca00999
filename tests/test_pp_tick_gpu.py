"""A pipeline-parallel iteration executed tick by tick on ONE GPU (SURVEY.md
8f next #3): the phase-synchronised tick table (cad_pp_tick_table,
P/src/sim.cpp:318-353); per tick, the attention of every active stage pooled
and scheduled with schedule_pp_tick (P/src/scheduler.cpp:359-373), then run as
one pass through the per-layer executor -- forward ticks dispatch Q/K/V, run
the CA forward and return O/LSE; backward ticks dispatch Q/K/V, the forward
state (O, LSE) and dO, run the CA backward and return dQ and the dK/dV
partials -- with every stage's context in this process (CAD_TRANSPORT_LOCAL,
phase by phase). Every (microbatch, stage)'s outputs are compared with the
CPU oracle."""
import random

import numpy as np
import pytest
import torch

import oracle
from ca_cases import assert_within, error_report
from layer_local import bf16_round

pytestmark = pytest.mark.gpu


def _home(items, rank, per_doc, width):
    parts = [per_doc[it.doc][it.q_begin:it.q_end] for it in items if it.home_device == rank]
    return np.concatenate(parts) if parts else np.zeros((0,) + width, np.float32)


@pytest.mark.parametrize("S_,M", [(2, 3), (3, 4)])
def test_pp_phase_sync_iteration_on_one_gpu(S_, M):
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import dispatch as D
    from paper_2510_18121_b200 import scheduler as S
    dev = torch.device("cuda", 0)
    shape = CF.Shape("t", 8, 2)
    hq, hkv, d = shape.h_q, shape.h_kv, 128
    rng = random.Random(S_ * 10 + M)
    nrng = np.random.default_rng(S_ * 10 + M)
    mbs, lengths = [], []
    for m in range(M):
        its = []
        for _ in range(1 + rng.randrange(3)):
            L = 64 + rng.randrange(900)
            its.append(S.Item(len(lengths), 0, L, L, 0, 0, S.CONTIGUOUS))
            lengths.append(L)
        mbs.append(its)
    # CA inputs of stage s for microbatch m (one layer per stage)
    data = {(m, s): {n: {it.doc: bf16_round(nrng.standard_normal((it.q_end, h, d), dtype=np.float32))
                         for it in mbs[m]} for n, h in (("q", hq), ("k", hkv), ("v", hkv), ("do", hq))}
            for m in range(M) for s in range(S_)}
    cfg = CF.sched_config(shape)
    table = S.pp_tick_table(M, S_, S.PP_PHASE_SYNC)
    got = {}
    fwd_state = {}
    for t, row in enumerate(table):
        bwd = next(w[0] for w in row if w is not None)
        per_stage = [mbs[w[1]] if w is not None else [] for w in row]
        items = [S.Item(it.doc, it.q_begin, it.q_end, it.kv_extent, it.ht_mirror, s, it.layout)
                 for s, its in enumerate(per_stage) for it in its]
        plans = [D.LayerPlan(lengths, S_, r, shape, cfg=cfg, items=items) for r in range(S_)]
        assert plans[0].plan.text == S.schedule_pp_tick(per_stage, S_, cfg).text
        layers = [D.DistCALayer(plans[r], dev, "local") for r in range(S_)]
        bufs, ios = [], []
        for r, L in enumerate(layers):
            H = max(1, L.home_rows)
            m = row[r][1] if row[r] is not None else None
            b = {}
            for n, h in (("q", hq), ("k", hkv), ("v", hkv), ("do", hq)):
                a = _home(items, r, data[(m, r)][n], (h, d)) if m is not None else np.zeros((0, h, d), np.float32)
                b[n] = torch.zeros(H, h, d, dtype=torch.bfloat16, device=dev)
                b[n][:len(a)] = torch.from_numpy(a).to(torch.bfloat16)
            if bwd and m is not None:
                b["o"], b["lse"] = fwd_state[(m, r)]
            else:
                b["o"] = torch.full((H, hq, d), float("nan"), dtype=torch.bfloat16, device=dev)
                b["lse"] = torch.full((hq, H), float("nan"), device=dev)
            b["dq"] = torch.full((H, hq, d), float("nan"), dtype=torch.bfloat16, device=dev)
            b["dk"] = torch.empty(H, hkv, d, dtype=torch.bfloat16, device=dev)
            b["dv"] = torch.empty(H, hkv, d, dtype=torch.bfloat16, device=dev)
            L.bind_outputs(b["o"], b["lse"], b["dq"])
            bufs.append(b)
            ios.append(L.io(b["q"], b["k"], b["v"], b["do"], b["o"], b["lse"], b["dq"], b["dk"], b["dv"]))
        blobs = [L.export() for L in layers]
        for L in layers:
            L.connect(blobs)
        st = torch.cuda.current_stream(dev)
        for L in layers:
            L.begin(st, "bwd" if bwd else "fwd")
        kinds = ([D.DISPATCH_QKV, D.DISPATCH_FWD_STATE, D.DISPATCH_DO] if bwd else [D.DISPATCH_QKV])
        for h in (0, 1):
            for kind in kinds:
                for r, L in enumerate(layers):
                    L.dispatch(0, h, kind, ios[r], st)
        for h in (0, 1):
            for L in layers:
                L.compute(0, h, bwd, st)
        for h in (0, 1):
            for r, L in enumerate(layers):
                L.ret(0, h, D.RETURN_GRAD if bwd else D.RETURN_O, ios[r], st)
        for r, L in enumerate(layers):
            L.finish(ios[r], st)
        torch.cuda.synchronize()
        for r, w in enumerate(row):
            if w is None:
                continue
            m, n = w[1], layers[r].home_rows
            if not bwd:
                fwd_state[(m, r)] = (bufs[r]["o"].clone(), bufs[r]["lse"].clone())
                got[(m, r, "o")] = bufs[r]["o"][:n].float().cpu().numpy()
                got[(m, r, "lse")] = bufs[r]["lse"][:, :n].cpu().numpy().T
            else:
                for name in ("dq", "dk", "dv"):
                    got[(m, r, name)] = bufs[r][name][:n].float().cpu().numpy()
        for L in layers:
            L.close()
    # every (microbatch, stage) ran its forward and its backward
    assert len(got) == 5 * M * S_
    worst = {}
    for m in range(M):
        its = mbs[m]
        for s in range(S_):
            tasks, off = [], 0
            for it in its:
                tasks.append((off, it.q_end, off, it.q_end))
                off += it.q_end
            cat = {n: np.concatenate([data[(m, s)][n][it.doc] for it in its]) for n in ("q", "k", "v", "do")}
            o, lse = oracle.ca_forward(tasks, cat["q"], cat["k"], cat["v"])
            dq, dk, dv = oracle.ca_backward(tasks, cat["q"], cat["k"], cat["v"], bf16_round(o), cat["do"])
            for name, ref in (("o", o), ("lse", lse.T), ("dq", dq), ("dk", dk), ("dv", dv)):
                rep = error_report(name, got[(m, s, name)], ref)
                if name not in worst or rep["row_rel"] > worst[name]["row_rel"] or rep["abs"] > worst[name]["abs"]:
                    worst[name] = rep
    print(f"PP S={S_} M={M}: {len(table)} ticks")
    for name in ("o", "lse", "dq", "dk", "dv"):
        assert_within(worst[name])
