"""The N>1 host path over real process boundaries (gloo, world size 2 and 8, CPU):
every rank builds its own cad_layer_plan, the row exchanges run as
torch.distributed all_to_all_single with the plan's per-peer counts, the
oracle plays the server kernels, and each rank checks its home rows against
the whole-batch oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CASES = {2: [900, 50, 70, 180, 200, 136],
         # 8 ranks (the driver's largest scaling run): a long document over 4 ranks
         8: [1400, 40, 100, 500, 60, 300, 200, 128, 72]}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _a2a(x, rows, shape_tail):
    """all_to_all_single of a row-major array with per-peer row counts."""
    send = torch.from_numpy(np.ascontiguousarray(x["send"]))
    out = torch.empty((int(sum(x["recv_counts"])),) + shape_tail, dtype=send.dtype)
    dist.all_to_all_single(out, send, [int(c) for c in x["recv_counts"]], [int(c) for c in x["send_counts"]])
    return out.numpy()


def _worker(rank, port, q, WORLD, LENGTHS):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import oracle
        from paper_2510_18121_b200 import configs as CF
        from paper_2510_18121_b200 import dispatch as D
        from dist_sim import home_arrays
        shape = CF.Shape("test", 2, 1)
        rng = np.random.default_rng(11)
        per = {n: [rng.standard_normal((l, h, 128), dtype=np.float32) for l in LENGTHS]
               for n, h in (("q", 2), ("k", 1), ("v", 1), ("do", 2))}
        lp = D.LayerPlan(LENGTHS, WORLD, rank, shape)
        # home rows of this rank (every rank knows the placement)
        items = [it for it in lp.home_items if it.home_device == rank]
        home = {n: np.concatenate([per[n][it.doc][it.q_begin:it.q_end] for it in items]) for n in per}
        H = lp.home_rows
        o_home = np.zeros((H, 2, 128), np.float32)
        dq_home = np.zeros_like(o_home)
        dk_home = np.zeros((H, 1, 128), np.float32)
        dv_home = np.zeros_like(dk_home)

        def xchg(x, src, dst, add=False):
            send = src[x.send_idx]
            got = _a2a({"send": send, "send_counts": x.send_counts, "recv_counts": x.recv_counts},
                       None, src.shape[1:])
            if add:
                np.add.at(dst, x.recv_idx, got)
            else:
                dst[x.recv_idx] = got

        for h in (0, 1):
            hp = lp.halves[h]
            qs = np.zeros((hp.q_rows, 2, 128), np.float32)
            dos = np.zeros_like(qs)
            ks = np.zeros((hp.kv_rows, 1, 128), np.float32)
            vs = np.zeros_like(ks)
            xchg(hp.xfers[D.XFER_Q], home["q"], qs)
            xchg(hp.xfers[D.XFER_Q], home["do"], dos)
            xchg(hp.xfers[D.XFER_KV], home["k"], ks)
            xchg(hp.xfers[D.XFER_KV], home["v"], vs)
            tasks = [(t.q_off, t.n_q, t.kv_off, t.kv_len) for t in hp.tasks]
            if tasks:
                o, _ = oracle.ca_forward(tasks, qs, ks, vs)
                dq, dk, dv = oracle.ca_backward(tasks, qs, ks, vs, o, dos)
            else:
                o, dq = np.zeros_like(qs), np.zeros_like(qs)
                dk, dv = np.zeros_like(ks), np.zeros_like(ks)
            xchg(hp.xfers[D.XFER_O_RET], o, o_home)
            xchg(hp.xfers[D.XFER_O_RET], dq, dq_home)
            xchg(hp.xfers[D.XFER_KV_RET], dk, dk_home, add=True)
            xchg(hp.xfers[D.XFER_KV_RET], dv, dv_home, add=True)
        tasks, off = [], 0
        for l in LENGTHS:
            tasks.append((off, l, off, l))
            off += l
        cat = {n: np.concatenate(per[n]) for n in per}
        o, _ = oracle.ca_forward(tasks, cat["q"], cat["k"], cat["v"])
        dq, dk, dv = oracle.ca_backward(tasks, cat["q"], cat["k"], cat["v"], o, cat["do"])
        cut = np.cumsum(LENGTHS)[:-1]
        ref = {n: np.concatenate([a[it.q_begin:it.q_end] for it in items for a in [np.split(arr, cut)[it.doc]]])
               for n, arr in (("o", o), ("dq", dq), ("dk", dk), ("dv", dv))}
        errs = {"o": np.abs(o_home - ref["o"]).max(), "dq": np.abs(dq_home - ref["dq"]).max(),
                "dk": np.abs(dk_home - ref["dk"]).max(), "dv": np.abs(dv_home - ref["dv"]).max(),
                "migrations": lp.plan.migrations}
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", sorted(CASES))
def test_gloo_dispatch_roundtrip(world):
    WORLD, LENGTHS = world, CASES[world]
    assert sum(LENGTHS) % WORLD == 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q, WORLD, LENGTHS)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r, e in res.items():
        assert e["migrations"] > 0
        for k in ("o", "dq", "dk", "dv"):
            assert e[k] < 1e-4, (r, k, e[k])
