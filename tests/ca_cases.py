"""Shared CA test cases: task sets in packed-row form plus input builders.

A case is (name, h_q, h_kv, q_rows, kv_rows, tasks) with tasks as
(q_off, n_q, kv_off, kv_len). Inputs are i.i.d. N(0,1) rounded to bf16
from a fixed torch seed.
"""
import numpy as np
import torch


def whole_docs(lengths):
    """Every document served whole on one server: Q and KV rows coincide."""
    tasks, off = [], 0
    for l in lengths:
        tasks.append((off, l, off, l))
        off += l
    return tasks, off


def split_doc(length, cuts):
    """One document split into query shards at `cuts`; every shard attends to
    the full causal prefix, KV rows = the whole document (rows 0..length)."""
    bounds = [0] + list(cuts) + [length]
    tasks = []
    for a, b in zip(bounds[:-1], bounds[1:]):
        tasks.append((a, b - a, 0, b))
    return tasks, length


def make_inputs(q_rows, kv_rows, h_q, h_kv, seed=0, device="cuda"):
    g = torch.Generator().manual_seed(seed)
    q = torch.randn(q_rows, h_q, 128, generator=g).to(torch.bfloat16)
    k = torch.randn(kv_rows, h_kv, 128, generator=g).to(torch.bfloat16)
    v = torch.randn(kv_rows, h_kv, 128, generator=g).to(torch.bfloat16)
    return q.to(device), k.to(device), v.to(device)


def f32(t):
    return t.detach().float().cpu().numpy()


def covered_rows(tasks):
    rows = np.zeros(0, dtype=np.int64)
    for t in tasks:
        rows = np.concatenate([rows, np.arange(t[0], t[0] + t[1])])
    return rows


def error_report(name, got, ref, axis_rows=0):
    """Max abs error and the worst per-row relative error
    (max |err| of a row / max(1, max |ref| of that row)) of one output.
    Rows are the first axis (the packed-row axis; LSE is passed transposed)."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if got.size == 0:
        return {"name": name, "abs": 0.0, "row_rel": 0.0, "max_ref": 0.0}
    err = np.abs(got - ref).reshape(got.shape[0], -1).max(axis=1)
    mag = np.abs(ref).reshape(ref.shape[0], -1).max(axis=1)
    return {"name": name, "abs": float(err.max()), "row_rel": float((err / np.maximum(1.0, mag)).max()),
            "max_ref": float(mag.max())}


# north_star tolerances: bf16 inputs, fp32 accumulation vs the fp32 oracle
O_ABS, LSE_ABS, GRAD_TOL = 2e-2, 1e-3, 2e-2


def assert_within(rep):
    """O: max abs <= 2e-2; LSE: max abs <= 1e-3; gradients: the worst row's
    max abs error <= 2e-2 * max(1, that row's max |ref|) (bf16 output
    rounding alone is 2^-9 of the magnitude). Both numbers are printed."""
    print(f"  {rep['name']:>4}: max abs {rep['abs']:.3e}  worst row rel {rep['row_rel']:.3e}  "
          f"(max |ref| {rep['max_ref']:.3g})")
    if rep["name"] == "o":
        assert rep["abs"] <= O_ABS, rep
    elif rep["name"] == "lse":
        assert rep["abs"] <= LSE_ABS, rep
    else:
        assert rep["row_rel"] <= GRAD_TOL, rep
