"""The distributed CA layer executed on
ONE GPU through the C-ABI executor: world-W LayerPlans with every rank's
context in this process (CAD_TRANSPORT_LOCAL, the IPC transport's push/flag
code path), compared row by row with the CPU oracle on the whole batch.

Also BASELINE config 1 (P/tests/test_scheduler.cpp:163-180): the reference's
golden 2-server, 7-task plan (homes place_sequential(docs, 2, 4096)) and the
same documents as 5 whole-document tasks on one server must agree with each
other and with the oracle."""
import os
import subprocess
import sys

import numpy as np
import pytest

from ca_cases import assert_within, error_report

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _check(out, ref, world):
    worst = {}
    for r in range(world):
        for n in ("o", "lse", "dq", "dk", "dv"):
            got, want = out[n][r], ref[n][r]
            if n == "lse":
                got, want = got.T, want.T
            assert np.isfinite(got).all(), (r, n, "unwritten rows")
            rep = error_report(n, got, want)
            if n not in worst or rep["row_rel"] > worst[n]["row_rel"] or rep["abs"] > worst[n]["abs"]:
                worst[n] = rep
    for n in ("o", "lse", "dq", "dk", "dv"):
        assert_within(worst[n])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_layer_world_on_one_gpu(world):
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import scheduler as S
    from layer_local import run_local
    per = 1024
    lengths = S.sample_batch(CF.length_dist("pretrain", 3, max_doc_len=2 * per), per * world)
    shape = CF.Shape("t", 8, 2)
    out, ref, plans, launches = run_local(lengths, world, shape, seed=world)
    moved = sum(1 for t in plans[0].plan.tasks if t.assigned_server != t.source_device)
    print(f"world {world}: {len(lengths)} docs, {len(plans[0].plan.tasks)} tasks ({moved} served remotely), "
          f"{launches} kernel launches")
    _check(out, ref, world)


def test_layer_head_tail_items_on_one_gpu():
    """head_tail (per-document CP) shards: a head and its mirrored tail served
    as two CA-tasks sharing the document's KV group (P/include/cadsim/
    types.hpp:107-111, P/src/sim.cpp:22-30), through the kernels."""
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import scheduler as S
    from layer_local import run_local
    lengths = [1536, 1024, 640]
    world = 2
    items = []
    for doc, L in enumerate(lengths):
        half = L // (2 * world)
        for r in range(world):  # rank r owns head [r*half, (r+1)*half) and its mirror
            items.append(S.Item(doc, r * half, (r + 1) * half, (r + 1) * half, L, r, S.HEAD_TAIL))
    shape = CF.Shape("t", 8, 2)
    out, ref, plans, _ = run_local(lengths, world, shape, seed=7, items=items)
    assert any(t.item.layout == S.HEAD_TAIL for t in plans[0].plan.tasks)
    _check(out, ref, world)


def test_config1_golden_plan_equals_whole_documents():
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import scheduler as S
    from layer_local import run_local
    from test_scheduler_parity import GOLDEN, ref_config
    lengths = CF.cfg1_lengths()
    shape = CF.CFG1  # 8 Q / 8 KV heads
    # (ii) the reference's golden 2-server plan: homes place_sequential(docs, 2, 4096)
    out2, ref2, plans2, _ = run_local(lengths, 2, shape, seed=1, cfg=ref_config(), tokens_per_device=4096)
    assert plans2[0].plan.text == GOLDEN
    _check(out2, ref2, 2)
    # (i) the 5 whole documents on one server
    out1, ref1, plans1, _ = run_local(lengths, 1, shape, seed=1, cfg=ref_config(), tokens_per_device=8192)
    assert len(plans1[0].plan.tasks) == 5
    _check(out1, ref1, 1)
    # the two runs agree row for row (homes: ranks 0+1 of (ii) = rank 0 of (i))
    for n in ("o", "dq", "dk", "dv"):
        a = np.concatenate([out2[n][0], out2[n][1]])
        b = out1[n][0]
        rep = error_report(n, a, b)
        print(f"config 1 golden plan vs whole documents, {n}: max abs {rep['abs']:.3e}")
        assert rep["row_rel"] <= 1e-2, rep
    lse2 = np.concatenate([out2["lse"][0], out2["lse"][1]], axis=1)
    assert np.abs(lse2 - out1["lse"][0]).max() <= 1e-4


def test_local_contexts_refuse_whole_steps():
    """cad_layer_step needs one process per rank: one thread enqueueing rank
    0's whole step before rank 1's would park GPU waits ahead of the work
    that releases them (streams of one context may share a hardware queue)."""
    import torch
    from paper_2510_18121_b200 import _native as N
    from paper_2510_18121_b200 import configs as CF
    from paper_2510_18121_b200 import dispatch as D
    plans = [D.LayerPlan([700, 300], 2, r, CF.Shape("t", 8, 2)) for r in range(2)]
    L = D.DistCALayer(plans[0], torch.device("cuda", 0), "local")
    with pytest.raises(N.ConfigError):
        L.step(N.cad_layer_io(), "pingpong")
    L.close()
