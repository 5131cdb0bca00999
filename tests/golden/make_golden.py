"""Generates tests/golden/ca_small.npz: CA fwd/bwd golden vectors computed
independently of oracle/ca_oracle.c with torch float64 autograd (dense
softmax with an explicit bottom-right causal mask per task, the mask of
P/src/oracle.cpp:50-54). Inputs are bf16-representable float32 values.

    python tests/golden/make_golden.py
"""
import os

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))


def reference(tasks, q, k, v, do, scale):
    """Per-task dense attention in float64 with autograd."""
    q = torch.tensor(q, dtype=torch.float64, requires_grad=True)
    k = torch.tensor(k, dtype=torch.float64, requires_grad=True)
    v = torch.tensor(v, dtype=torch.float64, requires_grad=True)
    h_q, h_kv = q.shape[1], k.shape[1]
    g = h_q // h_kv
    o = torch.zeros_like(q)
    lse = torch.full((h_q, q.shape[0]), float("nan"), dtype=torch.float64)
    outs = []
    for (qo, nq, ko, nk) in tasks:
        qs = q[qo:qo + nq]                                 # [nq, Hq, d]
        ks = k[ko:ko + nk].repeat_interleave(g, dim=1)     # [nk, Hq, d]
        vs = v[ko:ko + nk].repeat_interleave(g, dim=1)
        s = torch.einsum("ihd,jhd->hij", qs, ks) * scale
        qi = torch.arange(nq)[:, None] + (nk - nq)
        kj = torch.arange(nk)[None, :]
        s = s.masked_fill(kj > qi, float("-inf"))
        p = torch.softmax(s, dim=-1)
        outs.append((qo, nq, torch.einsum("hij,jhd->ihd", p, vs), torch.logsumexp(s, dim=-1)))
    rows = []
    for qo, nq, ot, lt in outs:
        o = o.index_put((torch.arange(qo, qo + nq),), ot)
        lse[:, qo:qo + nq] = lt.detach()
        rows.append(torch.arange(qo, qo + nq))
    (o * torch.tensor(do, dtype=torch.float64)).sum().backward()
    return o.detach().numpy(), lse.numpy(), q.grad.numpy(), k.grad.numpy(), v.grad.numpy()


def bf16_round(x):
    return torch.tensor(x).to(torch.bfloat16).to(torch.float32).numpy()


def main():
    rng = np.random.default_rng(2510_18121)
    cases = {
        # name: (tasks, q_rows, kv_rows, h_q, h_kv)
        "whole_docs": ([(0, 37, 0, 37), (37, 60, 37, 60), (97, 1, 97, 1)], 98, 98, 2, 1),
        "split_doc": ([(0, 30, 0, 30), (30, 50, 0, 80), (80, 40, 0, 120)], 120, 120, 2, 2),
        "shared_kv": ([(0, 20, 0, 20), (20, 60, 0, 90)], 80, 90, 4, 1),
    }
    out = {}
    for name, (tasks, qr, kr, hq, hkv) in cases.items():
        q = bf16_round(rng.standard_normal((qr, hq, 128), dtype=np.float32))
        k = bf16_round(rng.standard_normal((kr, hkv, 128), dtype=np.float32))
        v = bf16_round(rng.standard_normal((kr, hkv, 128), dtype=np.float32))
        do = bf16_round(rng.standard_normal((qr, hq, 128), dtype=np.float32))
        o, lse, dq, dk, dv = reference(tasks, q, k, v, do, 1.0 / np.sqrt(128))
        out[f"{name}/tasks"] = np.array(tasks, dtype=np.int64)
        for key, val in (("q", q), ("k", k), ("v", v), ("do", do), ("o", o), ("lse", lse), ("dq", dq),
                         ("dk", dk), ("dv", dv)):
            out[f"{name}/{key}"] = val.astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "ca_small.npz"), **out)
    print("wrote", os.path.join(HERE, "ca_small.npz"))


if __name__ == "__main__":
    main()
