"""Bit-exact parity of the product scheduler (libcad.so) with the reference
cadsim scheduler compiled unmodified from /root/reference (oracle/_ref).

Pins: the golden plan fixture P/tests/test_scheduler.cpp:163-180
and the hand-traced shard :133-161, then differential checks on random and
BASELINE-shaped instances comparing the full plan_to_stream text, the
IEEE-double stats (hex), counters, per-server loads and the per-device
served/sent lists with ping/pong halves.
"""
import random

import pytest

from paper_2510_18121_b200 import scheduler as S
from sched_util import baseline_dist, ours_plan, random_items, ref_place, ref_plan, ref_sample


def ref_config():
    # P/tests/test_scheduler.cpp:29-38
    return S.SchedulerConfig(epsilon=0.0, e_threshold=1e-9, tile_size=128, alpha_ca=1.0,
                             size_q=16384, size_kv=8192)


def scenario_items():
    items = [S.doc_item(0, 4096, 0)]
    items += [S.doc_item(d, 1024, 1) for d in range(1, 5)]
    return items


GOLDEN = (
    "# plan v1\n"
    "# doc q_begin q_end kv_extent ht_mirror layout source server core bytes\n"
    "0 0 2560 2560 0 contiguous 0 0 6553600 0\n"
    "0 3584 4096 4096 0 contiguous 0 0 3932160 0\n"
    "1 0 1024 1024 0 contiguous 1 1 1048576 0\n"
    "2 0 1024 1024 0 contiguous 1 1 1048576 0\n"
    "3 0 1024 1024 0 contiguous 1 1 1048576 0\n"
    "4 0 1024 1024 0 contiguous 1 1 1048576 0\n"
    "0 2560 3584 3584 0 contiguous 0 1 6291456 46137344\n"
)


def test_golden_plan_fixture():
    plan = S.schedule(scenario_items(), 2, ref_config())
    assert S.plan_to_stream(plan) == GOLDEN
    assert ref_plan(scenario_items(), 2, ref_config())["text"] == GOLDEN


def test_golden_shard_and_loads():
    # P/tests/test_scheduler.cpp:133-161
    plan = S.schedule(scenario_items(), 2, ref_config())
    assert plan.target == 10485760.0
    assert plan.migrations == 1 and plan.splits == 1 and plan.tolerance_met
    moved = [t for t in plan.tasks if t.assigned_server != t.source_device]
    assert len(moved) == 1
    t = moved[0]
    assert (t.item.doc, t.item.q_begin, t.item.q_end, t.item.kv_extent) == (0, 2560, 3584, 3584)
    assert t.comm_bytes == 46137344 and t.assigned_server == 1
    assert plan.max_load == plan.target == plan.min_load
    assert sum(S.ca_flops_core(t.item) for t in plan.tasks) == 16777216 + 4 * 1048576


def compare(items, n_servers, cfg, stages=None):
    ours, _ = ours_plan(items, n_servers, cfg, stages)
    ref = ref_plan(items, n_servers, cfg, stages)
    assert ours["text"] == ref["text"]
    assert ours["stats"] == ref["stats"]
    assert ours["servers"] == ref["servers"]
    assert ours["devices"] == ref["devices"]


@pytest.mark.parametrize("seed", range(8))
def test_random_aligned_instances(seed):
    rng = random.Random(1000 + seed)
    for trial in range(150):
        n_servers = 2 + rng.randrange(15)
        items = random_items(rng, n_servers, 1 + rng.randrange(64))
        cfg = ref_config()
        cfg.epsilon = [0.0, 0.05, 0.15][trial % 3]
        compare(items, n_servers, cfg)


@pytest.mark.parametrize("seed", range(8))
def test_random_unaligned_and_knobs(seed):
    """Unaligned items, head_tail items, and every SchedulerConfig knob."""
    rng = random.Random(7000 + seed)
    for trial in range(150):
        n_servers = 1 + rng.randrange(12)
        items = random_items(rng, n_servers, 1 + rng.randrange(40), aligned=False,
                             head_tail=(trial % 4 == 0))
        cfg = S.SchedulerConfig(
            epsilon=rng.choice([0.0, 0.01, 0.1, 0.3]),
            e_threshold=rng.choice([0.0, 1e-9, 0.01, 0.1, 1.0]),
            tile_size=rng.choice([1, 16, 64, 128, 256]),
            alpha_ca=rng.choice([1.0, 0.5, 3.0, 4.0 * 4096 * 32]),
            size_q=rng.choice([2, 8192, 16384]),
            size_kv=rng.choice([1, 4096, 8192]),
            double_query_head_tail=rng.random() < 0.3,
            max_moves=rng.choice([1 << 20, 1, 3, 17]))
        compare(items, n_servers, cfg)


@pytest.mark.parametrize("kind,seeds", [("pretrain", range(1, 31)), ("lognormal", range(1, 6)),
                                        ("uniform", range(1, 4)), ("fixed", range(1, 3)),
                                        ("prolong", range(1, 6))])
def test_baseline_configs(kind, seeds):
    """BASELINE.json configs: 8B shape (size_q=8192, size_kv=4096) at 512K
    tokens on 8 GPUs for every distribution of the imbalance sweep."""
    cfg = S.SchedulerConfig(epsilon=0.0, e_threshold=0.01, tile_size=128, alpha_ca=1.0,
                            size_q=8192, size_kv=4096)
    for seed in seeds:
        dist = baseline_dist(kind, seed)
        lengths = S.sample_batch(dist, 524288)
        assert lengths == ref_sample(dist, 524288)
        items = S.place_sequential(lengths, 8, 65536)
        assert [i.key() for i in items] == [i.key() for i in ref_place(lengths, 8, 65536)]
        compare(items, 8, cfg)


@pytest.mark.parametrize("n_gpus", [1, 2, 4, 8])
def test_34b_config(n_gpus):
    """Llama-34B shape (64Q/8KV: size_q=16384, size_kv=4096), 1M tokens, docs
    up to 256K, at 1/2/4/8 GPUs."""
    cfg = S.SchedulerConfig(epsilon=0.0, e_threshold=0.01, tile_size=128, alpha_ca=1.0,
                            size_q=16384, size_kv=4096)
    for seed in (1, 2):
        dist = baseline_dist("pretrain", seed, max_doc_len=262144)
        lengths = S.sample_batch(dist, 1 << 20)
        items = S.place_sequential(lengths, n_gpus, (1 << 20) // n_gpus)
        compare(items, n_gpus, cfg)


def test_pp_tick_parity():
    rng = random.Random(5)
    for trial in range(60):
        n_servers = 2 + rng.randrange(7)
        stages = [random_items(rng, 1, rng.randrange(6)) for _ in range(1 + rng.randrange(n_servers))]
        compare(None, n_servers, ref_config(), stages=stages)
