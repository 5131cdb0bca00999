"""Host-side CA-task API, mirroring the reference's cadsim C++ surface.

Names, argument meaning and error behaviour follow the reference so its
tests read the same here:
  Item / CATask                 P/include/cadsim/types.hpp:112-137
  SchedulerConfig / SchedulePlan P/include/cadsim/scheduler.hpp:12-45
  schedule, propose_migration, target_load, classify_servers,
  one_tile_slack, schedule_pp_tick, plan_to_stream
                                P/include/cadsim/scheduler.hpp:48-100
  v_min_comm / CommQuery        P/include/cadsim/comm.hpp:41-68
  sample_batch, place_sequential P/include/cadsim/workload.hpp:48-60
  device_plans_from_schedule    P/include/cadsim/sim.hpp:79
All work happens in libcad.so (C++); this module only marshals.
DomainError / ConfigError are raised where the reference throws them; an
unmet tolerance is flagged on the plan, never raised.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

from . import _native as N
from ._native import ConfigError, DomainError, check, lib  # noqa: F401 (re-export)

CONTIGUOUS, HEAD_TAIL = 0, 1
PRETRAIN_UPSAMPLED, PROLONG_LIKE, UNIFORM, FIXED, CUSTOM_HISTOGRAM = range(5)


@dataclass
class Item:
    doc: int = 0
    q_begin: int = 0
    q_end: int = 0
    kv_extent: int = 0
    ht_mirror: int = 0
    home_device: int = 0
    layout: int = CONTIGUOUS

    def query_tokens(self) -> int:
        return self.q_end - self.q_begin

    def to_c(self) -> N.cad_item:
        return N.cad_item(self.doc, self.q_begin, self.q_end, self.kv_extent, self.ht_mirror,
                          self.home_device, self.layout)

    @staticmethod
    def from_c(c: N.cad_item) -> "Item":
        return Item(c.doc, c.q_begin, c.q_end, c.kv_extent, c.ht_mirror, c.home_device, c.layout)

    def key(self):
        return (self.doc, self.q_begin, self.q_end, self.kv_extent, self.ht_mirror,
                self.home_device, self.layout)


def doc_item(doc: int, length: int, home: int) -> Item:
    return Item(doc, 0, length, length, 0, home, CONTIGUOUS)


@dataclass
class CATask:
    item: Item
    source_device: int
    assigned_server: int
    comm_bytes: int
    output_bytes: int


@dataclass
class SchedulerConfig:
    epsilon: float = 0.0
    e_threshold: float = 0.01
    tile_size: int = 128
    alpha_ca: float = 1.0
    size_q: int = 2
    size_kv: int = 2
    double_query_head_tail: bool = False
    max_moves: int = 1 << 20

    def to_c(self) -> N.cad_sched_cfg:
        c = N.cad_sched_cfg()
        c.epsilon, c.e_threshold, c.tile_size, c.alpha_ca = (self.epsilon, self.e_threshold,
                                                            self.tile_size, self.alpha_ca)
        c.size_q, c.size_kv = self.size_q, self.size_kv
        c.double_query_head_tail = 1 if self.double_query_head_tail else 0
        c.max_moves = self.max_moves
        return c


@dataclass
class ServerLoad:
    device: int = 0
    assigned_flops: float = 0.0
    assigned_core: int = 0
    items: List[Item] = field(default_factory=list)
    sent_bytes: int = 0
    received_bytes: int = 0

    def to_c(self) -> N.cad_server_load:
        return N.cad_server_load(self.device, 0, self.assigned_flops, self.assigned_core,
                                 len(self.items), self.sent_bytes, self.received_bytes)


@dataclass
class ServedTask:
    task_index: int
    item: Item
    in_bytes: int
    out_bytes: int
    half: int


@dataclass
class DevicePlan:
    device: int
    served: List[ServedTask]
    sent: List[ServedTask]


@dataclass
class SchedulePlan:
    tasks: List[CATask]
    per_server: List[ServerLoad]
    target: float
    max_load: float
    min_load: float
    total_comm_bytes: int
    total_output_bytes: int
    epsilon_used: float
    tolerance_met: bool
    migrations: int
    splits: int
    rejected_small: int
    text: str = ""
    devices: List[DevicePlan] = field(default_factory=list)


def _items_array(items: Sequence[Item]):
    arr = (N.cad_item * max(1, len(items)))()
    for i, it in enumerate(items):
        arr[i] = it.to_c()
    return arr


def ca_flops_core(item: Item) -> int:
    out = N.i64()
    check(lib().cad_ca_flops_core(C.byref(item.to_c()), C.byref(out)))
    return out.value


def exact_causal_pairs(n_q: int, n_kv: int) -> int:
    return lib().cad_causal_pairs(n_q, n_kv)


def target_load(items: Sequence[Item], n_servers: int, alpha_ca: float) -> float:
    out = N.f64()
    check(lib().cad_target_load(_items_array(items), len(items), n_servers, alpha_ca, C.byref(out)))
    return out.value


def classify_servers(loads: Sequence[float], target: float):
    n = len(loads)
    la = (N.f64 * max(1, n))(*loads)
    sd, sg, dd, dg = (N.i32 * max(1, n))(), (N.f64 * max(1, n))(), (N.i32 * max(1, n))(), (N.f64 * max(1, n))()
    ns, nd = N.i64(), N.i64()
    check(lib().cad_classify_servers(la, n, target, sd, sg, C.byref(ns), dd, dg, C.byref(nd)))
    return ([(sd[i], sg[i]) for i in range(ns.value)], [(dd[i], dg[i]) for i in range(nd.value)])


def one_tile_slack(items: Sequence[Item], cfg: SchedulerConfig) -> float:
    out = N.f64()
    check(lib().cad_one_tile_slack(_items_array(items), len(items), C.byref(cfg.to_c()), C.byref(out)))
    return out.value


@dataclass
class CommQuery:
    delta_f_max: float = 0.0
    f_item: float = 0.0
    L_q: int = 0
    L_kv: int = 0
    size_q: int = 0
    size_kv: int = 0
    layout: int = CONTIGUOUS
    ht_mirror: int = 0

    def to_c(self) -> N.cad_comm_query:
        c = N.cad_comm_query()
        c.delta_f_max, c.f_item, c.L_q, c.L_kv = self.delta_f_max, self.f_item, self.L_q, self.L_kv
        c.size_q, c.size_kv, c.layout, c.ht_mirror = self.size_q, self.size_kv, self.layout, self.ht_mirror
        return c


@dataclass
class ShardChoice:
    n_q: int
    n_kv: int
    bytes: int
    core: int


def v_min_comm(q: CommQuery, tile_size: int) -> ShardChoice:
    out = N.cad_shard_choice()
    check(lib().cad_v_min_comm(C.byref(q.to_c()), tile_size, C.byref(out)))
    return ShardChoice(out.n_q, out.n_kv, out.bytes, out.core)


@dataclass
class MigrationProposal:
    delta_f_max: float
    shard: Item
    remainders: List[Item]
    v_comm: int
    priority: float
    whole_item: bool


def propose_migration(source: ServerLoad, dest: ServerLoad, item: Item, target: float,
                      cfg: SchedulerConfig) -> Optional[MigrationProposal]:
    out, has = N.cad_proposal(), N.i32()
    check(lib().cad_propose_migration(C.byref(source.to_c()), C.byref(dest.to_c()),
                                      C.byref(item.to_c()), target, C.byref(cfg.to_c()),
                                      C.byref(out), C.byref(has)))
    if not has.value:
        return None
    return MigrationProposal(out.delta_f_max, Item.from_c(out.shard),
                             [Item.from_c(out.remainders[i]) for i in range(out.n_remainders)],
                             out.v_comm, out.priority, bool(out.whole_item))


def _unwrap_plan(h: C.c_void_p, free: bool = True) -> SchedulePlan:
    L = lib()
    try:
        st = N.cad_plan_stats()
        check(L.cad_plan_get_stats(h, C.byref(st)))
        tp, nt = C.POINTER(N.cad_task)(), N.i64()
        check(L.cad_plan_tasks(h, C.byref(tp), C.byref(nt)))
        tasks = [CATask(Item.from_c(tp[i].item), tp[i].source_device, tp[i].assigned_server,
                        tp[i].comm_bytes, tp[i].output_bytes) for i in range(nt.value)]
        servers = []
        for s in range(st.n_servers):
            ld, ip = N.cad_server_load(), C.POINTER(N.cad_item)()
            check(L.cad_plan_server(h, s, C.byref(ld), C.byref(ip)))
            servers.append(ServerLoad(ld.device, ld.assigned_flops, ld.assigned_core,
                                      [Item.from_c(ip[i]) for i in range(ld.n_items)],
                                      ld.sent_bytes, ld.received_bytes))
        need = C.c_size_t()
        check(L.cad_plan_to_text(h, None, 0, C.byref(need)))
        buf = C.create_string_buffer(need.value)
        check(L.cad_plan_to_text(h, buf, need.value, C.byref(need)))
        devices = []
        for d in range(st.n_servers):
            ns, nn = N.i64(), N.i64()
            check(L.cad_device_plan(h, d, None, 0, C.byref(ns), None, 0, C.byref(nn)))
            sa = (N.cad_served_task * max(1, ns.value))()
            sb = (N.cad_served_task * max(1, nn.value))()
            check(L.cad_device_plan(h, d, sa, ns.value, C.byref(ns), sb, nn.value, C.byref(nn)))
            conv = lambda x: ServedTask(x.task_index, tasks[x.task_index].item, x.in_bytes, x.out_bytes, x.half)
            devices.append(DevicePlan(d, [conv(sa[i]) for i in range(ns.value)],
                                      [conv(sb[i]) for i in range(nn.value)]))
        return SchedulePlan(tasks, servers, st.target, st.max_load, st.min_load,
                            st.total_comm_bytes, st.total_output_bytes, st.epsilon_used,
                            bool(st.tolerance_met), st.migrations, st.splits, st.rejected_small,
                            buf.value.decode(), devices)
    finally:
        if free:
            L.cad_plan_free(h)


def schedule(items: Sequence[Item], n_servers: int, cfg: SchedulerConfig) -> SchedulePlan:
    h = C.c_void_p()
    check(lib().cad_schedule(_items_array(items), len(items), n_servers, C.byref(cfg.to_c()), C.byref(h)))
    return _unwrap_plan(h)


class PlanHandle:
    """A live cad_plan (for consumers of the C-ABI such as cad_layer_plan);
    .plan is its Python mirror."""

    def __init__(self, items: Sequence[Item], n_servers: int, cfg: SchedulerConfig):
        self.h = C.c_void_p()
        check(lib().cad_schedule(_items_array(items), len(items), n_servers, C.byref(cfg.to_c()),
                                 C.byref(self.h)))
        self.plan = _unwrap_plan(self.h, free=False)

    def close(self):
        if self.h:
            lib().cad_plan_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def schedule_pp_tick(per_stage_items: Sequence[Sequence[Item]], n_servers: int,
                     cfg: SchedulerConfig) -> SchedulePlan:
    flat, stage = [], []
    for s, its in enumerate(per_stage_items):
        for it in its:
            flat.append(it)
            stage.append(s)
    st = (N.i32 * max(1, len(stage)))(*stage)
    h = C.c_void_p()
    check(lib().cad_schedule_pp_tick(_items_array(flat), st, len(flat), len(per_stage_items),
                                     n_servers, C.byref(cfg.to_c()), C.byref(h)))
    return _unwrap_plan(h)


def plan_to_stream(plan: SchedulePlan) -> str:
    return plan.text


def device_plans_from_schedule(plan: SchedulePlan) -> List[DevicePlan]:
    return plan.devices


@dataclass
class LengthDistribution:
    kind: int = FIXED
    max_doc_len: int = 1 << 20
    min_len_threshold: int = 0
    seed: int = 0
    log_mu: float = math.log(2048.0)
    log_sigma: float = 1.4
    upsample_drop_prob: float = 0.8
    long_mix_weight: float = 0.3
    long_log_mu: float = math.log(65536.0)
    long_log_sigma: float = 0.7
    fixed_len: int = 1024
    uniform_min: int = 1
    histogram: List[tuple] = field(default_factory=list)

    def to_c(self):
        c = N.cad_length_dist()
        lib().cad_length_dist_default(C.byref(c))
        for name in ("kind", "max_doc_len", "min_len_threshold", "seed", "log_mu", "log_sigma",
                     "upsample_drop_prob", "long_mix_weight", "long_log_mu", "long_log_sigma",
                     "fixed_len", "uniform_min"):
            setattr(c, name, getattr(self, name))
        keep = None
        if self.histogram:
            lens = (N.i64 * len(self.histogram))(*[h[0] for h in self.histogram])
            ps = (N.f64 * len(self.histogram))(*[h[1] for h in self.histogram])
            c.hist_len, c.hist_p, c.hist_n = lens, ps, len(self.histogram)
            keep = (lens, ps)
        return c, keep


def sample_batch(dist: LengthDistribution, total_tokens: int) -> List[int]:
    """Document lengths (ids are 0..n-1 in order)."""
    c, keep = dist.to_c()
    n = N.i64()
    check(lib().cad_sample_batch(C.byref(c), total_tokens, None, 0, C.byref(n)))
    out = (N.i64 * max(1, n.value))()
    check(lib().cad_sample_batch(C.byref(c), total_tokens, out, n.value, C.byref(n)))
    del keep
    return list(out[: n.value])


def place_sequential(lengths: Sequence[int], num_devices: int, tokens_per_device: int) -> List[Item]:
    """place_sequential + chunk_items: contiguous items per device chunk."""
    la = (N.i64 * max(1, len(lengths)))(*lengths)
    n = N.i64()
    check(lib().cad_place_sequential(la, len(lengths), num_devices, tokens_per_device, None, 0, C.byref(n)))
    out = (N.cad_item * max(1, n.value))()
    check(lib().cad_place_sequential(la, len(lengths), num_devices, tokens_per_device, out, n.value, C.byref(n)))
    return [Item.from_c(out[i]) for i in range(n.value)]


PP_1F1B, PP_PHASE_SYNC = 0, 1


def pp_tick_table(n_microbatches: int, n_stages: int, kind: int = PP_PHASE_SYNC):
    """The pipeline tick table of simulate_pp_iteration (P/src/sim.cpp:297-353):
    table[tick][stage] = None (idle) or (backward: bool, microbatch)."""
    n = N.i64()
    rc = lib().cad_pp_tick_table(n_microbatches, n_stages, kind, None, 0, C.byref(n))
    if rc not in (N.CAD_OK, N.CAD_ERR_CAPACITY):
        check(rc)
    arr = (N.cad_tick_work * max(1, n.value * n_stages))()
    check(lib().cad_pp_tick_table(n_microbatches, n_stages, kind, arr, n.value * n_stages, C.byref(n)))
    return [[(bool(arr[t * n_stages + s].backward), arr[t * n_stages + s].microbatch)
             if arr[t * n_stages + s].active else None for s in range(n_stages)] for t in range(n.value)]
