"""CA forward on the B200 vs the CPU oracle (fp32 IO, fp64 accumulation).

Tolerance (north_star): bf16 inputs with fp32 accumulation against the fp32
CPU oracle, max |O - O_ref| <= 2e-2 and max |LSE - LSE_ref| <= 1e-3.
"""
import numpy as np
import pytest
import torch

import oracle
from ca_cases import covered_rows, f32, make_inputs, split_doc, whole_docs

pytestmark = pytest.mark.gpu

O_TOL, LSE_TOL = 2e-2, 1e-3


def run_case(tasks, q_rows, kv_rows, h_q, h_kv, seed=0):
    from paper_2510_18121_b200.ca import CAPlan, CATaskRows
    q, k, v = make_inputs(q_rows, kv_rows, h_q, h_kv, seed)
    plan = CAPlan([CATaskRows(*t) for t in tasks], h_q, h_kv, q_rows, kv_rows)
    o, lse = plan.forward(q, k, v)
    torch.cuda.synchronize()
    o_ref, lse_ref = oracle.ca_forward(tasks, f32(q), f32(k), f32(v))
    rows = covered_rows(tasks)
    do = np.abs(f32(o)[rows] - o_ref[rows]).max()
    dl = np.abs(f32(lse)[:, rows] - lse_ref[:, rows]).max()
    return do, dl


CASES = {
    "one_tile": (lambda: whole_docs([128]), 2, 2),
    "gqa4_2tiles": (lambda: whole_docs([256]), 8, 2),
    "gqa1": (lambda: whole_docs([300]), 2, 2),
    "unaligned_docs": (lambda: whole_docs([1, 77, 128, 129, 500, 1000]), 4, 1),
    "split_shards": (lambda: split_doc(1000, [130, 384, 640]), 4, 2),
    "gqa8": (lambda: whole_docs([700, 333]), 8, 1),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_fwd_matches_oracle(name):
    build, h_q, h_kv = CASES[name]
    tasks, rows = build()
    do, dl = run_case(tasks, rows, rows, h_q, h_kv)
    assert do <= O_TOL, f"O max abs err {do}"
    assert dl <= LSE_TOL, f"LSE max abs err {dl}"


def test_fwd_split_plan_equals_whole_doc():
    """Composability: running the shards of a split plan
    reproduces the whole-document rows."""
    from paper_2510_18121_b200.ca import CAPlan, CATaskRows
    q, k, v = make_inputs(2048, 2048, 4, 2, seed=3)
    whole = CAPlan([CATaskRows(0, 2048, 0, 2048)], 4, 2, 2048, 2048)
    parts = CAPlan([CATaskRows(*t) for t in split_doc(2048, [512, 1280, 1536])[0]], 4, 2, 2048, 2048)
    o1, l1 = whole.forward(q, k, v)
    o2, l2 = parts.forward(q, k, v)
    torch.cuda.synchronize()
    assert (o1.float() - o2.float()).abs().max().item() <= 1e-2
    assert (l1 - l2).abs().max().item() <= 1e-4
