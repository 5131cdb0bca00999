"""Helpers shared by the scheduler parity tests: run the product scheduler
(libcad.so through paper_2510_18121_b200.scheduler) and the unmodified
reference (oracle/_ref/libcadsim_ref.so) on the same inputs and flatten both
plans into directly comparable records."""
import ctypes as C
import math
import random

import oracle
from paper_2510_18121_b200 import _native as N
from paper_2510_18121_b200 import scheduler as S


def items_c(items):
    arr = (N.cad_item * max(1, len(items)))()
    for i, it in enumerate(items):
        arr[i] = it.to_c()
    return arr


def ref_plan(items, n_servers, cfg, stages=None):
    L = oracle.ref_lib()
    st_arr, n_st = None, 0
    if stages is not None:
        flat, st = [], []
        for s, its in enumerate(stages):
            flat += its
            st += [s] * len(its)
        items = flat
        st_arr = (N.i32 * max(1, len(st)))(*st)
        n_st = len(stages)
    h = L.ref_schedule(items_c(items), len(items), n_servers, C.byref(cfg.to_c()), st_arr, n_st)
    if not h:
        raise RuntimeError(L.ref_last_error().decode())
    try:
        stats = N.cad_plan_stats()
        L.ref_plan_stats(h, C.byref(stats))
        ns = stats.n_servers
        fl, co, se, re = (N.f64 * ns)(), (N.i64 * ns)(), (N.i64 * ns)(), (N.i64 * ns)()
        L.ref_plan_servers(h, fl, co, se, re)
        return {
            "text": L.ref_plan_text(h).decode(),
            "devices": L.ref_plan_devices(h).decode(),
            "stats": stats_tuple(stats),
            "servers": [(fl[i].hex(), co[i], se[i], re[i]) for i in range(ns)],
        }
    finally:
        L.ref_plan_free(h)


def stats_tuple(st):
    return (st.target.hex(), st.max_load.hex(), st.min_load.hex(), st.epsilon_used.hex(),
            st.total_comm_bytes, st.total_output_bytes, st.migrations, st.splits,
            st.rejected_small, st.n_tasks, st.n_servers, st.tolerance_met)


def ours_plan(items, n_servers, cfg, stages=None):
    if stages is not None:
        p = S.schedule_pp_tick(stages, n_servers, cfg)
    else:
        p = S.schedule(items, n_servers, cfg)
    lines = []
    for dp in p.devices:
        for kind, lst in (("served", dp.served), ("sent", dp.sent)):
            for s in lst:
                lines.append(f"{dp.device} {kind} {s.item.doc} {s.item.q_begin} {s.item.q_end} "
                             f"{s.half} {s.in_bytes} {s.out_bytes}")
    # the reference emits served then sent per device
    by_dev = {}
    for ln in lines:
        by_dev.setdefault(int(ln.split()[0]), []).append(ln)
    devices = "".join(l + "\n" for d in sorted(by_dev) for l in by_dev[d])
    stats = (p.target.hex(), p.max_load.hex(), p.min_load.hex(), p.epsilon_used.hex(),
             p.total_comm_bytes, p.total_output_bytes, p.migrations, p.splits, p.rejected_small,
             len(p.tasks), len(p.per_server), int(p.tolerance_met))
    return {
        "text": p.text,
        "devices": devices,
        "stats": stats,
        "servers": [(s.assigned_flops.hex(), s.assigned_core, s.sent_bytes, s.received_bytes)
                    for s in p.per_server],
    }, p


def ref_sample(dist, total):
    L = oracle.ref_lib()
    c, keep = dist.to_c()
    n = N.i64()
    assert L.ref_sample_batch(C.byref(c), total, None, 0, C.byref(n)) == 0
    out = (N.i64 * max(1, n.value))()
    assert L.ref_sample_batch(C.byref(c), total, out, n.value, C.byref(n)) == 0
    del keep
    return list(out[: n.value])


def ref_place(lengths, devices, per_device):
    L = oracle.ref_lib()
    la = (N.i64 * max(1, len(lengths)))(*lengths)
    n = N.i64()
    rc = L.ref_place_sequential(la, len(lengths), devices, per_device, None, 0, C.byref(n))
    if rc != 0:
        raise RuntimeError(L.ref_last_error().decode())
    out = (N.cad_item * max(1, n.value))()
    L.ref_place_sequential(la, len(lengths), devices, per_device, out, n.value, C.byref(n))
    return [S.Item.from_c(out[i]) for i in range(n.value)]


def baseline_dist(kind, seed, max_doc_len=131072):
    """BASELINE.json configs 2-5."""
    d = S.LengthDistribution(seed=seed, max_doc_len=max_doc_len)
    if kind == "pretrain":
        d.kind, d.min_len_threshold, d.upsample_drop_prob = S.PRETRAIN_UPSAMPLED, 32768, 0.9
    elif kind == "lognormal":
        d.kind, d.min_len_threshold = S.PRETRAIN_UPSAMPLED, 0
    elif kind == "uniform":
        d.kind, d.max_doc_len = S.UNIFORM, 4096
    elif kind == "fixed":
        d.kind, d.fixed_len, d.max_doc_len = S.FIXED, 4096, 4096
    elif kind == "prolong":
        d.kind, d.long_mix_weight, d.long_log_mu, d.long_log_sigma = S.PROLONG_LIKE, 0.3, math.log(65536.0), 0.7
        d.max_doc_len = 262144
    else:
        raise ValueError(kind)
    return d


def random_items(rng: random.Random, n_servers, n_items, aligned=True, head_tail=False, max_tiles=64):
    items = []
    for i in range(n_items):
        if aligned:
            length = 128 * (1 + rng.randrange(max_tiles))
        else:
            length = 1 + rng.randrange(128 * max_tiles)
        home = rng.randrange(n_servers)
        if head_tail and rng.random() < 0.5:
            # a head-tail pair: head [b, e) and tail mirrored at M
            b = rng.randrange(0, length)
            e = b + 1 + rng.randrange(max(1, length // 2))
            m = 2 * e + rng.randrange(length + 1)
            items.append(S.Item(i, b, e, e, m, home, S.HEAD_TAIL))
        elif not aligned and rng.random() < 0.3:
            b = rng.randrange(length)
            items.append(S.Item(i, b, length, length, 0, home, S.CONTIGUOUS))
        else:
            items.append(S.doc_item(i, length, home))
    return items
