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
