"""CA kernel edge cases the scheduler produces at scale, through the C-ABI
kernels against the CPU oracle (fp32 IO, fp64 accumulation), with both the
max abs error and the worst per-row relative error printed:

* a 1-row shard with a 100K-token causal prefix (the document-final
  remainder place_sequential leaves on the next device);
* shards cut at a non-tile boundary past 64K (tile-aligned shards before and
  after an unaligned cut at 65601, all sharing the document's KV prefix);
* head_tail per-document-CP shards (P/include/cadsim/types.hpp:107-111): a
  head [b, e) over keys [0, e) and its mirrored tail [M-e, M-b) over keys
  [0, M-b), sharing one KV group, for several (b, e, M);
* GQA group 8 (the config-4 Llama-34B ratio) with split shards."""
import numpy as np
import pytest
import torch

import oracle
from ca_cases import assert_within, error_report, f32, make_inputs

pytestmark = pytest.mark.gpu


def run_case(tasks, q_rows, kv_rows, h_q, h_kv, seed=0):
    from paper_2510_18121_b200.ca import CAPlan, CATaskRows
    q, k, v = make_inputs(q_rows, kv_rows, h_q, h_kv, seed)
    g = torch.Generator().manual_seed(seed + 100)
    do = torch.randn(q_rows, h_q, 128, generator=g).to(torch.bfloat16).cuda()
    plan = CAPlan([CATaskRows(*t) for t in tasks], h_q, h_kv, q_rows, kv_rows)
    o, lse = plan.forward(q, k, v)
    dq, dk, dv = plan.backward(q, k, v, o, lse, do)
    torch.cuda.synchronize()
    ro, rlse = oracle.ca_forward(tasks, f32(q), f32(k), f32(v))
    rdq, rdk, rdv = oracle.ca_backward(tasks, f32(q), f32(k), f32(v), f32(o), f32(do))
    qr = np.concatenate([np.arange(t[0], t[0] + t[1]) for t in tasks])
    kr = np.unique(np.concatenate([np.arange(t[2], t[2] + t[3]) for t in tasks]))
    reps = [error_report("o", f32(o)[qr], ro[qr]), error_report("lse", f32(lse).T[qr], rlse.T[qr]),
            error_report("dq", f32(dq)[qr], rdq[qr]), error_report("dk", f32(dk)[kr], rdk[kr]),
            error_report("dv", f32(dv)[kr], rdv[kr])]
    for r in reps:
        assert_within(r)


def test_one_row_shard_with_100k_prefix():
    # alone, and next to a whole short document and a 2-row shard of the same
    # long prefix (same KV group)
    run_case([(0, 1, 0, 100000)], 1, 100000, 8, 2, seed=1)
    run_case([(0, 1, 0, 100001), (1, 2, 0, 100000), (3, 300, 100001, 300)], 303, 100301, 8, 2, seed=2)


def test_unaligned_cut_past_64k():
    cut = 65601
    tasks = [(0, 128, 0, 65536),            # tile-aligned shard ending at 64K
             (128, cut - 65536, 0, cut),    # [65536, 65601): 65 rows ending at the unaligned cut
             (128 + cut - 65536, 399, 0, cut + 399)]  # [65601, 66000)
    q_rows = 128 + cut - 65536 + 399
    run_case(tasks, q_rows, cut + 399, 4, 1, seed=3)


@pytest.mark.parametrize("b,e,M", [(0, 128, 512), (100, 300, 1000), (1, 2, 4), (384, 512, 2048),
                                   (0, 700, 1400)])
def test_head_tail_shards_share_kv(b, e, M):
    n = e - b
    head = (0, n, 0, e)           # queries [b, e) over keys [0, e)
    tail = (n, n, 0, M - b)       # queries [M-e, M-b) over keys [0, M-b)
    run_case([head, tail], 2 * n, M - b, 8, 2, seed=b + e)


def test_gqa8_split_shards():
    tasks = [(0, 500, 0, 500), (500, 333, 0, 833), (833, 1, 0, 834), (834, 640, 834, 640)]
    run_case(tasks, 1474, 1474, 16, 2, seed=9)
