"""The reference's own unit tests for the hot path, restated against the
product API (paper_2510_18121_b200.scheduler -> libcad.so):
P/tests/test_scheduler.cpp, test_comm.cpp, test_cost.cpp, test_workload.cpp.
Each test cites the reference case it mirrors."""
import math
import random

import pytest

from paper_2510_18121_b200 import scheduler as S
from paper_2510_18121_b200.scheduler import doc_item


def ref_config():  # test_scheduler.cpp:29-38
    return S.SchedulerConfig(epsilon=0.0, e_threshold=1e-9, tile_size=128, alpha_ca=1.0,
                             size_q=16384, size_kv=8192)


def plan_core(plan):
    return sum(S.ca_flops_core(t.item) for t in plan.tasks)


# ---------------------------------------------------------------- cost (test_cost.cpp)
def test_core_identities():
    # whole documents come out as length^2; causal identity 2*pairs - core = n_q (test_cost.cpp:120-129)
    for L in (1, 7, 128, 1000):
        assert S.ca_flops_core(doc_item(0, L, 0)) == L * L
    rng = random.Random(5)
    for _ in range(200):
        kv = 1 + rng.randrange(5000)
        nq = 1 + rng.randrange(kv)
        it = S.Item(0, kv - nq, kv, kv, 0, 0)
        assert 2 * S.exact_causal_pairs(nq, kv) - S.ca_flops_core(it) == nq


def test_sharding_conserves_core():
    # test_cost.cpp:79-94: random partitions of a document telescope exactly
    rng = random.Random(9)
    for _ in range(300):
        L = 2 + rng.randrange(4000)
        cuts = sorted(rng.sample(range(1, L), min(L - 1, 1 + rng.randrange(6))))
        bounds = [0] + cuts + [L]
        total = sum(S.ca_flops_core(S.Item(0, a, b, b, 0, 0)) for a, b in zip(bounds[:-1], bounds[1:]))
        assert total == L * L


def test_head_tail_core():
    it = S.Item(0, 10, 30, 30, 100, 0, S.HEAD_TAIL)
    assert S.ca_flops_core(it) == 2 * 20 * 100


# ---------------------------------------------------------------- scheduler
def test_target_load_is_exact_mean():  # test_scheduler.cpp:42-48
    items = [doc_item(0, 10, 0), doc_item(1, 10, 1)]
    assert S.target_load(items, 2, 1.0) == 100.0
    assert S.target_load(items, 1, 1.0) == 200.0
    assert S.target_load(items, 2, 3.0) == 300.0


def test_target_load_scenario():  # :50-55
    items = [doc_item(0, 4096, 0)] + [doc_item(d, 1024, 1) for d in range(1, 5)]
    assert S.target_load(items, 2, 1.0) == 10485760.0


def test_classify_servers():  # :57-72
    s, d = S.classify_servers([300, 100], 200)
    assert s == [(0, 100.0)] and d == [(1, 100.0)]
    s, d = S.classify_servers([200, 200], 200)
    assert s == [] and d == []
    _, d = S.classify_servers([400, 150, 50], 200)
    assert [x[0] for x in d] == [2, 1]


def test_propose_delta_is_min_of_bounds():  # :74-99
    cfg = ref_config()
    cfg.tile_size = 1
    src, dst = S.ServerLoad(device=0, assigned_flops=250), S.ServerLoad(device=1, assigned_flops=-80)
    p = S.propose_migration(src, dst, doc_item(0, 10, 0), 0.0, cfg)
    assert p is not None and p.delta_f_max == 80.0 and not p.whole_item
    dst.assigned_flops = -150
    p = S.propose_migration(src, dst, doc_item(0, 10, 0), 0.0, cfg)
    assert p.delta_f_max == 100.0 and p.whole_item and p.remainders == []


def test_propose_priority_halves_with_double_bytes():  # :101-122
    cfg = ref_config()
    cfg.tile_size = 1
    src, dst = S.ServerLoad(assigned_flops=300), S.ServerLoad(device=1, assigned_flops=-200)
    a = S.propose_migration(src, dst, doc_item(0, 10, 0), 0.0, cfg)
    b = S.propose_migration(src, dst, doc_item(1, 10, 2), 0.0, cfg)
    assert a.priority == b.priority
    heavy = ref_config()
    heavy.tile_size, heavy.size_q, heavy.size_kv = 1, 2 * cfg.size_q, 2 * cfg.size_kv
    c = S.propose_migration(src, dst, doc_item(1, 10, 2), 0.0, heavy)
    assert c.priority == pytest.approx(b.priority / 2)


def test_balanced_input_no_migration():  # :124-131
    plan = S.schedule([doc_item(0, 2048, 0), doc_item(1, 2048, 1)], 2, ref_config())
    assert plan.migrations == 0 and plan.total_comm_bytes == 0 and plan.tolerance_met
    assert plan.max_load == plan.min_load


def test_conservation_and_alignment_random():  # :182-213
    rng = random.Random(17)
    for trial in range(50):
        n_servers = 2 + rng.randrange(8)
        items = [doc_item(i, 128 * (1 + rng.randrange(40)), rng.randrange(n_servers))
                 for i in range(1 + rng.randrange(32))]
        cfg = ref_config()
        cfg.epsilon = (trial % 3) * 0.05
        plan = S.schedule(items, n_servers, cfg)
        assert plan_core(plan) == sum(S.ca_flops_core(i) for i in items)
        if plan.tolerance_met:
            slack = S.one_tile_slack(items, cfg)
            assert plan.max_load - plan.target <= cfg.epsilon * plan.target + slack + 1e-6
            assert plan.target - plan.min_load <= cfg.epsilon * plan.target + slack + 1e-6
        for t in plan.tasks:
            assert t.item.q_begin % 128 == 0 and t.item.q_end % 128 == 0


def test_comm_non_increasing_in_epsilon():  # :215-230
    rng = random.Random(23)
    items = [doc_item(i, 128 * (1 + rng.randrange(64)), rng.randrange(4)) for i in range(24)]
    prev = None
    for eps in (0.0, 0.05, 0.10, 0.15, 0.20, 0.25):
        cfg = ref_config()
        cfg.epsilon = eps
        b = S.schedule(items, 4, cfg).total_comm_bytes
        if prev is not None:
            assert b <= prev
        prev = b


def test_deterministic():  # :232-245
    rng = random.Random(29)
    items = [doc_item(i, 128 * (1 + rng.randrange(32)), rng.randrange(3)) for i in range(16)]
    assert S.schedule(items, 3, ref_config()).text == S.schedule(items, 3, ref_config()).text


def test_sub_tile_moves_rejected():  # :247-256
    plan = S.schedule([doc_item(0, 128, 1), doc_item(1, 128, 1)], 3, ref_config())
    assert plan.migrations == 0 and plan.rejected_small > 0 and not plan.tolerance_met
    assert plan_core(plan) == 2 * 128 * 128


def test_doc_final_remainders_unaligned():  # :258-269
    plan = S.schedule([doc_item(0, 1000, 0), doc_item(1, 128, 1)], 2, ref_config())
    assert plan_core(plan) == 1000 * 1000 + 128 * 128
    for t in plan.tasks:
        aligned = t.item.q_begin % 128 == 0 and t.item.q_end % 128 == 0
        assert aligned or t.item.q_end in (1000, 128)


def test_pp_tick_idle_stages_absorb():  # :271-286
    per_stage = [[doc_item(0, 4096, 0)], [doc_item(1, 4096, 0)], [], []]
    plan = S.schedule_pp_tick(per_stage, 4, ref_config())
    assert plan.target == pytest.approx(2 * 4096 * 4096 / 4)
    for sv in plan.per_server:
        assert sv.assigned_flops == pytest.approx(plan.target, rel=0.15)


def test_pp_tick_balanced_noop():  # :288-296
    per_stage = [[doc_item(s, 2048, s)] for s in range(4)]
    plan = S.schedule_pp_tick(per_stage, 4, ref_config())
    assert plan.migrations == 0 and plan.total_comm_bytes == 0


def test_single_doc_hot_spot():  # :298-306
    items = [doc_item(0, 16384, 0)]
    plan = S.schedule(items, 4, ref_config())
    slack = S.one_tile_slack(items, ref_config())
    for sv in plan.per_server:
        assert abs(sv.assigned_flops - plan.target) <= slack
    assert plan_core(plan) == 16384 * 16384


# ---------------------------------------------------------------- v_min_comm (test_comm.cpp)
def test_v_min_comm_whole_item():  # test_comm.cpp:190-203
    q = S.CommQuery(4096.0 * 4096.0, 4096.0 * 4096.0, 4096, 4096, 16384, 8192)
    s = S.v_min_comm(q, 128)
    assert (s.n_q, s.n_kv, s.bytes) == (4096, 4096, 4096 * (16384 + 8192))


def test_v_min_comm_rejects_infeasible():  # :205-215
    with pytest.raises(S.DomainError):
        S.v_min_comm(S.CommQuery(2.0 * 1024 * 1024, 1024.0 * 1024, 1024, 1024, 2, 1), 128)


def _grid_search(q, tile):
    """Exhaustive tile-aligned minimal-byte shard (restates vcomm_grid_search,
    P/src/oracle.cpp:9-48, independently)."""
    G = q.L_q * (2 * q.L_kv - q.L_q)
    frac = min(1.0, q.delta_f_max / q.f_item)
    target = max(1, min(G, math.ceil(frac * G - 1e-9)))
    best = None
    for n in list(range(tile, q.L_q + 1, tile)) + [q.L_q]:
        kv = max((target + n * n + 2 * n - 1) // (2 * n), n + q.L_kv - q.L_q)
        if kv > q.L_kv:
            continue
        kv = max(kv, min(-(-kv // tile) * tile, q.L_kv))
        b = n * q.size_q + kv * q.size_kv if q.layout == S.CONTIGUOUS else \
            n * q.size_q + (q.ht_mirror - (kv - n)) * q.size_kv
        if best is None or b < best:
            best = b
    return best


def test_v_min_comm_vs_exhaustive():  # :215-231 (within 1% of the grid search)
    rng = random.Random(2024)
    for i in range(300):
        L_q = 128 * (1 + rng.randrange(40))
        L_kv = L_q + 128 * rng.randrange(40)
        layout = S.HEAD_TAIL if i % 2 else S.CONTIGUOUS
        f_item = float(L_q * (2 * L_kv - L_q))
        q = S.CommQuery(f_item * (0.05 + 0.9 * rng.random()), f_item, L_q, L_kv, 16384, 8192, layout,
                        2 * L_kv + 128 * rng.randrange(10))
        s = S.v_min_comm(q, 128)
        assert 0 < s.n_q <= L_q and s.n_q + L_kv - L_q <= s.n_kv <= L_kv
        assert s.bytes <= 1.01 * _grid_search(q, 128)


def test_head_tail_closed_form():  # :250-267
    L = 8192
    for frac in (0.1, 0.33, 0.5, 0.75):
        q = S.CommQuery(frac * L * L, float(L * L), L, L, 16384, 8192, S.HEAD_TAIL, 2 * L)
        s = S.v_min_comm(q, 1)
        assert abs(s.n_q - L * (1 - math.sqrt(1 - frac))) <= 1.0


# ---------------------------------------------------------------- workload (test_workload.cpp)
def test_fixed_lengths_and_truncation():  # test_workload.cpp:11-26
    assert S.sample_batch(S.LengthDistribution(kind=S.FIXED, fixed_len=1024), 4096) == [1024] * 4
    assert S.sample_batch(S.LengthDistribution(kind=S.FIXED, fixed_len=1000), 2500) == [1000, 1000, 500]


def test_seed_determinism():  # :28-42
    d = S.LengthDistribution(kind=S.PRETRAIN_UPSAMPLED, max_doc_len=65536, min_len_threshold=2048, seed=99)
    assert S.sample_batch(d, 1 << 18) == S.sample_batch(d, 1 << 18)


def test_zero_threshold_noop():  # :44-56
    a = S.LengthDistribution(kind=S.PRETRAIN_UPSAMPLED, max_doc_len=65536, seed=4)
    b = S.LengthDistribution(kind=S.PRETRAIN_UPSAMPLED, max_doc_len=65536, seed=4, upsample_drop_prob=0.99)
    assert S.sample_batch(a, 1 << 16) == S.sample_batch(b, 1 << 16)


def test_upsampling_raises_mean():  # :58-76
    base = S.LengthDistribution(kind=S.PRETRAIN_UPSAMPLED, max_doc_len=65536, seed=12)
    up = S.LengthDistribution(kind=S.PRETRAIN_UPSAMPLED, max_doc_len=65536, seed=12, min_len_threshold=4096,
                              upsample_drop_prob=0.9)
    mean = lambda x: sum(x) / len(x)
    assert mean(S.sample_batch(up, 1 << 20)) > mean(S.sample_batch(base, 1 << 20))


def test_place_sequential_tiles_documents():  # :272-309
    lengths = S.sample_batch(S.LengthDistribution(kind=S.PROLONG_LIKE, max_doc_len=32768, seed=20), 1 << 16)
    items = S.place_sequential(lengths, 8, (1 << 16) // 8)
    per_dev = [0] * 8
    cover = {}
    for it in items:
        per_dev[it.home_device] += it.query_tokens()
        cover.setdefault(it.doc, []).append((it.q_begin, it.q_end))
    assert per_dev == [(1 << 16) // 8] * 8
    for doc, segs in cover.items():
        segs.sort()
        assert segs[0][0] == 0 and segs[-1][1] == lengths[doc]
        assert all(a[1] == b[0] for a, b in zip(segs[:-1], segs[1:]))


def test_custom_histogram():  # :168-177
    d = S.LengthDistribution(kind=S.CUSTOM_HISTOGRAM, max_doc_len=1 << 16, seed=5,
                             histogram=[(128, 0.5), (4096, 0.5)])
    for l in S.sample_batch(d, 1 << 14):
        assert l in (128, 4096) or l < 4096
