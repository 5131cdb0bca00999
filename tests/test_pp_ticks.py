"""Pipeline ticks: the tick table of
simulate_pp_iteration (P/src/sim.cpp:297-353, cad_pp_tick_table) against the
unmodified reference run here (oracle/_ref), and the pooled per-tick plans
(schedule_pp_tick, P/src/scheduler.cpp:359-373) it drives:

* vanilla 1F1B: every stage's forward/backward sequence equals the order of
  the reference's recorded events; tick counts equal;
* phase-synchronised: tick counts equal, every tick is one pass across the
  stages, and the total wire bytes of the per-tick pooled plans scheduled from
  our table equal the reference's (which schedules from its own table), with
  microbatches of distinct shapes so a different table would change them."""
import ctypes as C
import random

import pytest

import oracle
from paper_2510_18121_b200 import _native as N
from paper_2510_18121_b200 import scheduler as S


def _microbatches(rng, M):
    mbs, doc = [], 0
    for m in range(M):
        items = []
        for _ in range(1 + rng.randrange(4)):
            L = 128 * (1 + rng.randrange(24)) + rng.randrange(2) * rng.randrange(128)
            items.append(S.Item(doc, 0, L, L, 0, 0, S.CONTIGUOUS))
            doc += 1
        mbs.append(items)
    return mbs


def _ref(mbs, S_, kind, cfg):
    R = oracle.ref_lib()
    flat, mb_of, tokens = [], [], []
    for m, its in enumerate(mbs):
        flat += its
        mb_of += [m] * len(its)
        tokens.append(sum(i.q_end - i.q_begin for i in its))
    arr = (N.cad_item * max(1, len(flat)))(*[i.to_c() for i in flat])
    mb = (N.i64 * max(1, len(flat)))(*mb_of)
    tk = (N.i64 * len(mbs))(*tokens)
    cap = 4 * (len(mbs) + S_)
    ev = (C.c_int32 * (S_ * cap))()
    cnt = (N.i64 * S_)()
    ticks, wire = N.i64(), N.i64()
    rc = R.ref_pp_iteration(arr, mb, len(flat), tk, len(mbs), S_, kind, C.byref(cfg.to_c()), C.byref(ticks),
                            C.byref(wire), ev, cap, cnt)
    assert rc == 0, R.ref_last_error()
    kinds = [[ev[s * cap + e] for e in range(cnt[s])] for s in range(S_)]
    return ticks.value, wire.value, kinds


def _cfg():
    # the shim's model: hidden 4096, kv_hidden 1024, bf16 (size_q 8192, size_kv 4096)
    return S.SchedulerConfig(epsilon=0.0, e_threshold=1e-9, tile_size=128, alpha_ca=4.0 * 4096 * 4,
                             size_q=8192, size_kv=4096)


@pytest.mark.parametrize("S_,M", [(2, 2), (2, 5), (3, 3), (4, 4), (4, 9), (8, 8), (8, 13)])
def test_1f1b_table_matches_reference_events(S_, M):
    rng = random.Random(S_ * 100 + M)
    mbs = _microbatches(rng, M)
    ticks, _, kinds = _ref(mbs, S_, S.PP_1F1B, _cfg())
    table = S.pp_tick_table(M, S_, S.PP_1F1B)
    assert len(table) == ticks == 2 * (M + S_ - 1)
    for s in range(S_):
        ours = [int(row[s][0]) for row in table if row[s] is not None]
        assert ours == kinds[s], s
        fw = [row[s][1] for row in table if row[s] is not None and not row[s][0]]
        bw = [row[s][1] for row in table if row[s] is not None and row[s][0]]
        assert fw == list(range(M)) and bw == list(range(M))


@pytest.mark.parametrize("S_,M", [(2, 2), (2, 5), (3, 4), (4, 4), (4, 7), (8, 8), (8, 11)])
def test_phase_sync_table_matches_reference_wire(S_, M):
    rng = random.Random(7 * S_ + M)
    mbs = _microbatches(rng, M)
    cfg = _cfg()
    ticks, wire, _ = _ref(mbs, S_, S.PP_PHASE_SYNC, cfg)
    table = S.pp_tick_table(M, S_, S.PP_PHASE_SYNC)
    assert len(table) == ticks == 2 * (M + S_ - 1)
    ours = 0
    for row in table:
        passes = {w[0] for w in row if w is not None}
        assert len(passes) == 1  # one pass per tick: the pooling is legal
        per_stage = [mbs[w[1]] if w is not None else [] for w in row]
        plan = S.schedule_pp_tick(per_stage, S_, cfg)
        ours += sum(sv.received_bytes for sv in plan.per_server)
    assert ours == wire
    # every (stage, microbatch) runs one forward and, later, one backward
    for s in range(S_):
        seen = {}
        for t, row in enumerate(table):
            if row[s] is not None:
                seen.setdefault(row[s][1], []).append((t, row[s][0]))
        assert sorted(seen) == list(range(M))
        for m, ev in seen.items():
            assert [b for _, b in ev] == [False, True]


def test_tick_table_errors_match_reference():
    for M, S_ in ((1, 2), (3, 0)):
        with pytest.raises(N.ConfigError):
            S.pp_tick_table(M, S_)
