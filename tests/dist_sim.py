"""Numpy execution of cad_layer_plan's row exchanges (no GPU, no NCCL): the
same gather -> all-to-allv -> scatter(-add) steps as dispatch.DistCALayer,
with the CA oracle standing in for the server kernels. Used by the CPU tests
of the dispatcher (in-process and over gloo)."""
import numpy as np

import oracle
from paper_2510_18121_b200 import dispatch as D
from paper_2510_18121_b200 import scheduler as S


def split(counts, arr):
    out, o = [], 0
    for c in counts:
        out.append(arr[o:o + c])
        o += c
    return out


def exchange(plans, h, which, src, dst_shapes, add=False, dtype=np.float32):
    """src[r]: rank r's source array (rows first). Returns dst[p]."""
    W = len(plans)
    dst = [np.zeros(s, dtype=dtype) for s in dst_shapes]
    for r in range(W):
        x = plans[r].halves[h].xfers[which]
        for p, idx in enumerate(split(x.send_counts, x.send_idx)):
            rows = src[r][idx]
            xp = plans[p].halves[h].xfers[which]
            ridx = split(xp.recv_counts, xp.recv_idx)[r]
            assert len(ridx) == len(rows)
            if add:
                np.add.at(dst[p], ridx, rows)
            else:
                dst[p][ridx] = rows
    return dst


def home_arrays(plans, lengths, per_doc):
    """Lay per-document arrays [L, ...] out in each rank's home rows."""
    W = len(plans)
    homes = []
    for r in range(W):
        items = [it for it in plans[0].home_items if it.home_device == r]
        parts = []
        for it in items:
            parts.append(per_doc[it.doc][it.q_begin:it.q_end])
            if it.layout == S.HEAD_TAIL:  # tail rows follow the head rows
                parts.append(per_doc[it.doc][it.ht_mirror - it.q_end:it.ht_mirror - it.q_begin])
        homes.append(np.concatenate(parts))
    return homes


def run_layer(lengths, world, shape, seed=0, items=None, balance_halves=False):
    """Returns (home outputs of the distributed run, whole-batch reference),
    both in home layout per rank: dicts of o, lse, dq, dk, dv. `items`:
    explicit home items (default: place_sequential of the lengths)."""
    rng = np.random.default_rng(seed)
    plans = [D.LayerPlan(lengths, world, r, shape, items=items, balance_halves=balance_halves) for r in range(world)]
    hq, hkv, d = shape.h_q, shape.h_kv, shape.head_dim
    per = {n: [rng.standard_normal((l, h, d), dtype=np.float32) for l in lengths]
           for n, h in (("q", hq), ("k", hkv), ("v", hkv), ("do", hq))}
    home = {n: home_arrays(plans, lengths, per[n]) for n in per}
    W = world
    hr = [p.home_rows for p in plans]
    out = {"o": [np.zeros((hr[r], hq, d), np.float32) for r in range(W)],
           "lse": [np.zeros((hq, hr[r]), np.float32) for r in range(W)],
           "dq": [np.zeros((hr[r], hq, d), np.float32) for r in range(W)],
           "dk": [np.zeros((hr[r], hkv, d), np.float32) for r in range(W)],
           "dv": [np.zeros((hr[r], hkv, d), np.float32) for r in range(W)]}
    for h in (0, 1):
        hp = [p.halves[h] for p in plans]
        qs = exchange(plans, h, D.XFER_Q, home["q"], [(x.q_rows, hq, d) for x in hp])
        ks = exchange(plans, h, D.XFER_KV, home["k"], [(x.kv_rows, hkv, d) for x in hp])
        vs = exchange(plans, h, D.XFER_KV, home["v"], [(x.kv_rows, hkv, d) for x in hp])
        dos = exchange(plans, h, D.XFER_Q, home["do"], [(x.q_rows, hq, d) for x in hp])
        os_, lses, dqs, dks, dvs = [], [], [], [], []
        for s in range(W):
            tasks = [(t.q_off, t.n_q, t.kv_off, t.kv_len) for t in hp[s].tasks]
            if not tasks:
                os_.append(np.zeros((0, hq, d), np.float32)); lses.append(np.zeros((hq, 0), np.float32))
                dqs.append(np.zeros((0, hq, d), np.float32)); dks.append(np.zeros((0, hkv, d), np.float32))
                dvs.append(np.zeros((0, hkv, d), np.float32))
                continue
            o, lse = oracle.ca_forward(tasks, qs[s], ks[s], vs[s])
            dq, dk, dv = oracle.ca_backward(tasks, qs[s], ks[s], vs[s], o, dos[s])
            os_.append(o); lses.append(lse); dqs.append(dq); dks.append(dk); dvs.append(dv)
        # return paths (server -> home); O_RET rows are server q rows
        o_h = exchange(plans, h, D.XFER_O_RET, os_, [(r, hq, d) for r in hr])
        dq_h = exchange(plans, h, D.XFER_O_RET, dqs, [(r, hq, d) for r in hr])
        lse_rows = exchange(plans, h, D.XFER_O_RET, [l.T.copy() for l in lses], [(r, hq) for r in hr])
        dk_h = exchange(plans, h, D.XFER_KV_RET, dks, [(r, hkv, d) for r in hr], add=True)
        dv_h = exchange(plans, h, D.XFER_KV_RET, dvs, [(r, hkv, d) for r in hr], add=True)
        covered = exchange(plans, h, D.XFER_O_RET, [np.ones((x.q_rows, 1), np.float32) for x in hp],
                           [(r, 1) for r in hr])
        for r in range(W):
            m = covered[r][:, 0] > 0
            out["o"][r][m] = o_h[r][m]
            out["dq"][r][m] = dq_h[r][m]
            out["lse"][r][:, m] = lse_rows[r][m].T
            out["dk"][r] += dk_h[r]
            out["dv"][r] += dv_h[r]
    # whole-batch reference: every document as one task on one "GPU"
    tasks, off = [], 0
    for l in lengths:
        tasks.append((off, l, off, l))
        off += l
    cat = {n: np.concatenate(per[n]) for n in per}
    o, lse = oracle.ca_forward(tasks, cat["q"], cat["k"], cat["v"])
    dq, dk, dv = oracle.ca_backward(tasks, cat["q"], cat["k"], cat["v"], o, cat["do"])
    ref_doc = {"o": np.split(o, np.cumsum(lengths)[:-1]), "dq": np.split(dq, np.cumsum(lengths)[:-1]),
               "dk": np.split(dk, np.cumsum(lengths)[:-1]), "dv": np.split(dv, np.cumsum(lengths)[:-1]),
               "lse": np.split(lse.T, np.cumsum(lengths)[:-1])}
    ref = {n: home_arrays(plans, lengths, ref_doc[n]) for n in ref_doc}
    ref["lse"] = [x.T for x in ref["lse"]]
    return out, ref, plans
