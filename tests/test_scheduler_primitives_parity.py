"""Direct differentials of the scheduler's building blocks against the
unmodified reference (oracle/_ref/libcadsim_ref.so) on random queries,
including ones `schedule` never issues (propose_migration
P/src/scheduler.cpp:109-194, v_min_comm P/src/comm.cpp:98-178, one_tile_slack
:36-49, target_load :13-19), and a >= 10^4-instance differential of whole
plans. Results must agree bit for bit (doubles compared as IEEE hex), and an
error in one must be the same error code in the other."""
import ctypes as C
import random

import pytest

import oracle
from paper_2510_18121_b200 import _native as N
from paper_2510_18121_b200 import scheduler as S
from sched_util import items_c, ours_plan, random_items, ref_plan


def _item_t(c):
    return (c.doc, c.q_begin, c.q_end, c.kv_extent, c.ht_mirror, c.home_device, c.layout)


def _rand_cfg(rng):
    return S.SchedulerConfig(
        epsilon=rng.choice([0.0, 0.01, 0.1]),
        e_threshold=rng.choice([0.0, 1e-9, 0.01, 0.1, 1.0, 10.0]),
        tile_size=rng.choice([1, 7, 16, 64, 128, 256]),
        alpha_ca=rng.choice([1.0, 0.5, 3.0, 2.0 * 128 * 32]),
        size_q=rng.choice([2, 8192, 16384]),
        size_kv=rng.choice([1, 4096, 8192]),
        double_query_head_tail=rng.random() < 0.3,
        max_moves=1 << 20)


def _rand_item(rng, home):
    r = rng.random()
    length = rng.choice([1 + rng.randrange(300), 128 * (1 + rng.randrange(64)), 1 + rng.randrange(200000)])
    if r < 0.2:  # head_tail
        b = rng.randrange(length)
        e = b + 1 + rng.randrange(max(1, length // 2))
        m = 2 * e + rng.randrange(length + 1)
        return S.Item(rng.randrange(50), b, e, e, m, home, S.HEAD_TAIL)
    if r < 0.5:
        b = rng.randrange(length)
        return S.Item(rng.randrange(50), b, length, length, 0, home, S.CONTIGUOUS)
    return S.doc_item(rng.randrange(50), length, home)


def test_propose_migration_differential():
    rng = random.Random(20261019)
    L, R = N.lib(), oracle.ref_lib()
    n_some = 0
    for trial in range(6000):
        cfg = _rand_cfg(rng).to_c()
        item = _rand_item(rng, 0).to_c()
        core = N.i64()
        assert L.cad_ca_flops_core(C.byref(item), C.byref(core)) == 0
        f_item = cfg.alpha_ca * core.value
        target = f_item * rng.choice([0.1, 0.5, 1.0, 2.0, 5.0]) + rng.random()
        src = N.cad_server_load(0, 0, target + f_item * rng.random() * 2, 0)
        dst = N.cad_server_load(rng.choice([0, 1]), 0, target - f_item * rng.random() * 2, 0)
        src.assigned_core = int(src.assigned_flops / max(cfg.alpha_ca, 1e-300))
        dst.assigned_core = max(0, int(dst.assigned_flops / max(cfg.alpha_ca, 1e-300)))
        a, b = N.cad_proposal(), N.cad_proposal()
        ha, hb = N.i32(), N.i32()
        ra = L.cad_propose_migration(C.byref(src), C.byref(dst), C.byref(item), target, C.byref(cfg), C.byref(a),
                                     C.byref(ha))
        rb = R.ref_propose_migration(C.byref(src), C.byref(dst), C.byref(item), target, C.byref(cfg), C.byref(b),
                                     C.byref(hb))
        assert ra == rb, (trial, ra, rb)
        if ra != 0:
            continue
        assert ha.value == hb.value, trial
        if not ha.value:
            continue
        n_some += 1
        assert a.delta_f_max.hex() == b.delta_f_max.hex(), trial
        assert _item_t(a.shard) == _item_t(b.shard), trial
        assert a.n_remainders == b.n_remainders, trial
        for i in range(a.n_remainders):
            assert _item_t(a.remainders[i]) == _item_t(b.remainders[i]), trial
        assert (a.whole_item, a.v_comm) == (b.whole_item, b.v_comm), trial
        assert a.priority.hex() == b.priority.hex(), trial
    assert n_some > 1000


def test_v_min_comm_differential():
    rng = random.Random(7)
    L, R = N.lib(), oracle.ref_lib()
    n_ok = 0
    for trial in range(10000):
        lq = 1 + rng.randrange(rng.choice([200, 5000, 200000]))
        lkv = lq + rng.choice([0, rng.randrange(1 + lq), rng.randrange(200000)])
        ht = rng.random() < 0.3
        g = lq * (2 * lkv - lq)
        f_item = float(g) * rng.choice([1.0, 0.5, 2.0 * 128 * 32])
        dfm = f_item * rng.choice([rng.random(), 1.0, 1e-6, 0.999999, 1.0 + 1e-13, 1.5])
        if rng.random() < 0.02:
            dfm = -1.0
        q = N.cad_comm_query(dfm, f_item, lq, lkv, rng.choice([2, 8192, 16384, 0]) if rng.random() < 0.05 else
                             rng.choice([2, 8192, 16384]), rng.choice([1, 4096, 8192]),
                             S.HEAD_TAIL if ht else S.CONTIGUOUS)
        q.ht_mirror = (2 * lkv + rng.randrange(lkv + 1)) if ht else 0
        if ht and rng.random() < 0.05:
            q.ht_mirror = 2 * lkv - 1  # invalid mirror
        tile = rng.choice([0, 1, 16, 64, 128, 256])
        a, b = N.cad_shard_choice(), N.cad_shard_choice()
        ra = L.cad_v_min_comm(C.byref(q), tile, C.byref(a))
        rb = R.ref_v_min_comm(C.byref(q), tile, C.byref(b))
        assert ra == rb, (trial, ra, rb)
        if ra == 0:
            n_ok += 1
            assert (a.n_q, a.n_kv, a.bytes, a.core) == (b.n_q, b.n_kv, b.bytes, b.core), trial
    assert n_ok > 7000


def test_one_tile_slack_and_target_load_differential():
    rng = random.Random(11)
    L, R = N.lib(), oracle.ref_lib()
    for trial in range(3000):
        n_servers = 1 + rng.randrange(16)
        items = [_rand_item(rng, rng.randrange(n_servers)) for _ in range(1 + rng.randrange(30))]
        arr = items_c(items)
        cfg = _rand_cfg(rng).to_c()
        a, b = N.f64(), N.f64()
        ra = L.cad_one_tile_slack(arr, len(items), C.byref(cfg), C.byref(a))
        rb = R.ref_one_tile_slack(arr, len(items), C.byref(cfg), C.byref(b))
        assert ra == rb and (ra != 0 or a.value.hex() == b.value.hex()), trial
        alpha = rng.choice([1.0, 0.5, 3.0, 8192.0])
        ra = L.cad_target_load(arr, len(items), n_servers, alpha, C.byref(a))
        rb = R.ref_target_load(arr, len(items), n_servers, alpha, C.byref(b))
        assert ra == rb and (ra != 0 or a.value.hex() == b.value.hex()), trial


@pytest.mark.parametrize("block", range(8))
def test_random_plans_differential_1e4(block):
    """8 x 1500 random instances here + 2400 in test_scheduler_parity.py:
    >= 10^4 whole-plan differentials (text, stats as IEEE hex, loads,
    served/sent lists with halves)."""
    rng = random.Random(424242 + block)
    for trial in range(1500):
        n_servers = 1 + rng.randrange(12)
        aligned = rng.random() < 0.5
        items = random_items(rng, n_servers, 1 + rng.randrange(48), aligned=aligned,
                             head_tail=rng.random() < 0.25, max_tiles=rng.choice([4, 64, 512]))
        cfg = _rand_cfg(rng)
        cfg.max_moves = rng.choice([1 << 20, 1 << 20, 1, 5])
        ours, _ = ours_plan(items, n_servers, cfg)
        ref = ref_plan(items, n_servers, cfg)
        assert ours == ref, (block, trial)
