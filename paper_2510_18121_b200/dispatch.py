"""Per-layer CA dispatch / compute / return on one rank (one GPU).

The reference only models this step: device_plans_from_schedule splits each
device's served tasks into ping/pong halves and layer_windows hides
dispatch(pong) under CA(ping) and return(ping) under CA(pong)
(P/src/sim.cpp:34-46,69-125). Here it runs for real:

  forward   Q/K/V rows home -> server (all-to-allv)  ->  CA fwd on the server
            ->  O/LSE rows server -> home
  backward  dO rows home -> server  ->  CA bwd (Q/K/V/O/LSE stay resident on
            the server from the forward)  ->  dQ rows -> home, dK/dV partial
            rows -> owners, summed there (fp32)

Row lists come from cad_layer_plan (C++, deterministic on every rank);
packing is cad_gather_rows / cad_scatter_rows, the exchange is
cad_alltoallv (grouped ncclSend/ncclRecv over NVLink) on a side stream, and
the CA kernels run on the compute stream with CUDA events between them, so
the exchange of one half overlaps the CA kernel of the other. torch only
provides device memory, streams and events.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _native as N
from . import configs as CF
from . import scheduler as S
from ._native import check, lib
from .ca import CAPlan, CATaskRows

XFER_Q, XFER_KV, XFER_O_RET, XFER_KV_RET = 0, 1, 2, 3


@dataclass
class Xfer:
    """One exchange as seen by this rank (row counts/indices per peer)."""
    send_counts: np.ndarray
    send_idx: np.ndarray
    recv_counts: np.ndarray
    recv_idx: np.ndarray

    @property
    def n_send(self) -> int:
        return int(self.send_counts.sum())

    @property
    def n_recv(self) -> int:
        return int(self.recv_counts.sum())


@dataclass
class HalfPlan:
    home_rows: int
    q_rows: int
    kv_rows: int
    tasks: List[CATaskRows]
    task_index: List[int]
    remote_send_bytes: List[int]
    xfers: List[Xfer]


def _arr(ptr, n) -> np.ndarray:
    return np.ctypeslib.as_array(ptr, shape=(n,)).copy() if n > 0 else np.zeros(0, dtype=np.int64)


class LayerPlan:
    """Schedule + per-rank row movement of one layer (host side, no GPU)."""

    def __init__(self, lengths: Sequence[int], world: int, rank: int, shape: CF.Shape,
                 cfg: Optional[S.SchedulerConfig] = None, tokens_per_device: Optional[int] = None,
                 items: Optional[Sequence[S.Item]] = None, balance_halves: bool = False):
        """Home items from place_sequential(lengths) (DistCA's chunks), or the
        given `items` (e.g. head_tail per-document CP shards; a head_tail
        item's home rows are its head rows, then its tail rows).
        balance_halves: even out each server's ping/pong halves in causal
        pairs (cad_layer_plan_create_ex) instead of the reference's
        assign_halves split."""
        total = sum(lengths)
        self.world, self.rank, self.shape = world, rank, shape
        self.tokens_per_device = tokens_per_device or total // world
        self.home_items = list(items) if items is not None else S.place_sequential(lengths, world,
                                                                                   self.tokens_per_device)
        self.cfg = cfg or CF.sched_config(shape)
        ph = S.PlanHandle(self.home_items, world, self.cfg)
        self.plan = ph.plan
        arr = (N.cad_item * max(1, len(self.home_items)))(*[i.to_c() for i in self.home_items])
        lp = C.c_void_p()
        q_row = shape.h_q * shape.head_dim * 2
        kv_row = 2 * shape.h_kv * shape.head_dim * 2
        check(lib().cad_layer_plan_create_ex(ph.h, arr, len(self.home_items), rank, q_row, kv_row,
                                             int(balance_halves), C.byref(lp)))
        try:
            self.halves: List[HalfPlan] = []
            for h in (0, 1):
                info = N.cad_layer_half_info()
                check(lib().cad_layer_plan_info(lp, h, C.byref(info)))
                tasks = [CATaskRows(info.tasks[i].q_off, info.tasks[i].n_q, info.tasks[i].kv_off,
                                    info.tasks[i].kv_len) for i in range(info.n_tasks)]
                xs = []
                for w in range(4):
                    x = N.cad_xfer()
                    check(lib().cad_layer_plan_xfer(lp, h, w, C.byref(x)))
                    xs.append(Xfer(_arr(x.send_counts, x.n_peers), _arr(x.send_idx, x.n_send),
                                   _arr(x.recv_counts, x.n_peers), _arr(x.recv_idx, x.n_recv)))
                self.halves.append(HalfPlan(info.home_rows, info.q_rows, info.kv_rows, tasks,
                                            [info.task_index[i] for i in range(info.n_tasks)],
                                            list(info.remote_send_bytes), xs))
        finally:
            lib().cad_layer_plan_destroy(lp)
            ph.close()
        self.home_rows = self.halves[0].home_rows

    def server_pairs(self) -> int:
        """Exact causal pairs this rank serves (both halves)."""
        return sum(lib().cad_causal_pairs(t.n_q, t.kv_len) for hp in self.halves for t in hp.tasks)


class Comm:
    """A cad_comm (NCCL) communicator for this rank."""

    def __init__(self, unique_id: bytes, rank: int, world: int):
        buf = (N.u8 * 128).from_buffer_copy(unique_id)
        self.h = C.c_void_p()
        check(lib().cad_comm_init(buf, rank, world, C.byref(self.h)))
        self.rank, self.world = rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = (N.u8 * 128)()
        check(lib().cad_comm_unique_id(buf))
        return bytes(buf)

    def close(self):
        if self.h:
            lib().cad_comm_destroy(self.h)
            self.h = None


class _DevXfer:
    def __init__(self, x: Xfer, device):
        self.x = x
        self.send_idx = torch.from_numpy(x.send_idx).to(device)
        self.recv_idx = torch.from_numpy(x.recv_idx).to(device)

    def counts(self, row_bytes: int):
        sb = (self.x.send_counts * row_bytes).astype(np.int64)
        rb = (self.x.recv_counts * row_bytes).astype(np.int64)
        sd = np.concatenate([[0], np.cumsum(sb)[:-1]]).astype(np.int64)
        rd = np.concatenate([[0], np.cumsum(rb)[:-1]]).astype(np.int64)
        to = lambda a: (N.i64 * len(a))(*a.tolist())
        return to(sb), to(sd), to(rb), to(rd)


def _p(t: torch.Tensor) -> int:
    return t.data_ptr()


class DistCALayer:
    """Executes one CA layer (fwd + bwd) for this rank: dispatch, CA kernels,
    return, with ping/pong halves on a compute and a comm stream."""

    def __init__(self, lp: LayerPlan, comm: Optional[Comm], device: torch.device, reserve_sms: int = 0):
        self.lp, self.comm, self.dev = lp, comm, device
        sh = lp.shape
        self.hq, self.hkv, self.d = sh.h_q, sh.h_kv, sh.head_dim
        self.q_row = self.hq * self.d * 2
        self.kv_row = self.hkv * self.d * 2
        self.comm_stream = torch.cuda.Stream(device=device)
        self.halves = []
        bf = dict(dtype=torch.bfloat16, device=device)
        self._bf = bf
        max_bytes = 1
        for hp in lp.halves:
            plan = CAPlan(hp.tasks, self.hq, self.hkv, max(1, hp.q_rows), max(1, hp.kv_rows)) if hp.tasks else None
            if plan is not None and reserve_sms > 0:
                check(lib().cad_ca_plan_set_max_ctas(plan._h, max(1, torch.cuda.get_device_properties(device)
                                                                    .multi_processor_count - reserve_sms)))
            qr, kr = max(1, hp.q_rows), max(1, hp.kv_rows)
            half = {
                "plan": plan, "hp": hp,
                "x": [_DevXfer(x, device) for x in hp.xfers],
                "q": torch.empty(qr, self.hq, self.d, **bf), "k": torch.empty(kr, self.hkv, self.d, **bf),
                "v": torch.empty(kr, self.hkv, self.d, **bf), "o": torch.empty(qr, self.hq, self.d, **bf),
                "lse": torch.empty(self.hq, qr, dtype=torch.float32, device=device),
                "do": torch.empty(qr, self.hq, self.d, **bf), "dq": torch.empty(qr, self.hq, self.d, **bf),
                "dk": torch.empty(kr, self.hkv, self.d, **bf), "dv": torch.empty(kr, self.hkv, self.d, **bf),
                "ws": torch.empty(max(1, plan.workspace_bytes if plan else 1), dtype=torch.uint8, device=device),
                "ev": {},
            }
            for x in hp.xfers:
                max_bytes = max(max_bytes, x.n_send * self.q_row, x.n_recv * self.q_row)
            self.halves.append(half)
        self.send_buf = torch.empty(max_bytes, dtype=torch.uint8, device=device)
        self._max_bytes = max_bytes
        self.recv_buf = torch.empty(max_bytes, dtype=torch.uint8, device=device)
        self.launches = 0
        self.ce = None

    def alloc_halves(self):
        """Another set of per-half server buffers (a further layer's
        activations), sharing this layer's plans and row lists."""
        out = []
        bf = self._bf
        for H in self.halves:
            qr, kr = H["q"].shape[0], H["k"].shape[0]
            out.append({"q": torch.empty(qr, self.hq, self.d, **bf), "k": torch.empty(kr, self.hkv, self.d, **bf),
                        "v": torch.empty(kr, self.hkv, self.d, **bf), "o": torch.empty(qr, self.hq, self.d, **bf),
                        "lse": torch.empty(self.hq, qr, dtype=torch.float32, device=self.dev),
                        "do": torch.empty(qr, self.hq, self.d, **bf), "dq": torch.empty(qr, self.hq, self.d, **bf),
                        "dk": torch.empty(kr, self.hkv, self.d, **bf), "dv": torch.empty(kr, self.hkv, self.d, **bf)})
        return out

    # ---------------------------------------------------------------- exchange
    def _exchange(self, dx: _DevXfer, src: torch.Tensor, dst: torch.Tensor, row_bytes: int, stream,
                  reverse: bool = False, mode: str = "copy"):
        """Gather src rows (send_idx), all-to-allv, scatter into dst rows
        (recv_idx). mode 'add' sums bf16 rows into an fp32 dst."""
        s = stream.cuda_stream
        L = lib()
        check(L.cad_gather_rows(_p(src), _p(dx.send_idx), dx.x.n_send, row_bytes, _p(self.send_buf), s))
        sb, sd, rb, rd = dx.counts(row_bytes)
        check(L.cad_alltoallv(self.comm.h, _p(self.send_buf), sb, sd, _p(self.recv_buf), rb, rd, s))
        if mode == "copy":
            check(L.cad_scatter_rows(_p(self.recv_buf), _p(dx.recv_idx), dx.x.n_recv, row_bytes, _p(dst), s))
        else:
            check(L.cad_scatter_add_bf16(_p(self.recv_buf), _p(dx.recv_idx), dx.x.n_recv, row_bytes // 2,
                                         _p(dst), s))
        self.launches += 2

    def _exchange_cols(self, dx: _DevXfer, src, src_rows, dst, dst_rows, stream):
        """LSE [heads][rows] transport: column gather, all-to-allv, column scatter."""
        s = stream.cuda_stream
        L = lib()
        row_bytes = self.hq * 4
        check(L.cad_gather_cols_f32(_p(src), src_rows, self.hq, _p(dx.send_idx), dx.x.n_send,
                                    _p(self.send_buf), s))
        sb, sd, rb, rd = dx.counts(row_bytes)
        check(L.cad_alltoallv(self.comm.h, _p(self.send_buf), sb, sd, _p(self.recv_buf), rb, rd, s))
        check(L.cad_scatter_cols_f32(_p(self.recv_buf), _p(dx.recv_idx), dx.x.n_recv, self.hq, _p(dst),
                                     dst_rows, s))
        self.launches += 2

    # ---------------------------------------------------------------- phases
    def dispatch_fwd(self, h, q, k, v, stream):
        H = self.halves[h]
        self._exchange(H["x"][XFER_Q], q, H["q"], self.q_row, stream)
        self._exchange(H["x"][XFER_KV], k, H["k"], self.kv_row, stream)
        self._exchange(H["x"][XFER_KV], v, H["v"], self.kv_row, stream)

    def return_fwd(self, h, o, lse, stream):
        H = self.halves[h]
        self._exchange(H["x"][XFER_O_RET], H["o"], o, self.q_row, stream)
        self._exchange_cols(H["x"][XFER_O_RET], H["lse"], H["lse"].shape[1], lse, lse.shape[1], stream)

    def dispatch_bwd(self, h, do, stream):
        H = self.halves[h]
        self._exchange(H["x"][XFER_Q], do, H["do"], self.q_row, stream)

    def return_bwd(self, h, dq, dk_acc, dv_acc, stream):
        H = self.halves[h]
        self._exchange(H["x"][XFER_O_RET], H["dq"], dq, self.q_row, stream)
        self._exchange(H["x"][XFER_KV_RET], H["dk"], dk_acc, self.kv_row, stream, mode="add")
        self._exchange(H["x"][XFER_KV_RET], H["dv"], dv_acc, self.kv_row, stream, mode="add")

    def _bufs(self, h, layer):
        if layer == 0:
            return self.halves[h]
        return self.ce.lbufs[layer][h]

    def ca_fwd(self, h, stream, layer: int = 0):
        plan = self.halves[h]["plan"]
        H = self._bufs(h, layer)
        if plan is not None:
            plan.forward(H["q"], H["k"], H["v"], H["o"], H["lse"], stream=stream)
            self.launches += 1

    def ca_bwd(self, h, stream, layer: int = 0):
        plan = self.halves[h]["plan"]
        H = self._bufs(h, layer)
        if plan is not None:
            H["dk"].zero_()
            H["dv"].zero_()
            plan.backward(H["q"], H["k"], H["v"], H["o"], H["lse"], H["do"], H["dq"], H["dk"], H["dv"],
                          self.halves[h]["ws"], stream=stream)
            self.launches += 3

    # ---------------------------------------------------------------- step
    def use_copy_engines(self, all_plans: List[LayerPlan], o, lse, dq, layers: int = 1, copy_mode: str = "ce",
                         copy_ctas: int = 4):
        """Switch the exchanges to the copy-engine transport (CUDA IPC pushes);
        o/lse/dq become the registered home output buffers of every step.
        layers > 1: every step runs that many stacked CA layers (see
        CETransport.step)."""
        self.ce = CETransport(self, all_plans, o, lse, dq, layers, copy_mode, copy_ctas)

    def step(self, q, k, v, do, o, lse, dq, dk_acc, dv_acc, mode: str = "pingpong"):
        """One layer fwd+bwd. mode: 'pingpong' (comm of one half under CA of
        the other), 'serial' (single stream, no overlap), 'compute' (CA
        kernels only; server buffers assumed resident: the reference's
        'signal' bound), 'comm' (exchanges only)."""
        comp = torch.cuda.current_stream(self.dev)
        if mode in ("pingpong", "comm", "signal") and getattr(self, "ce", None) is not None:
            if not (o.data_ptr() == self.ce.o.data_ptr() and dq.data_ptr() == self.ce.dq.data_ptr()
                    and lse.data_ptr() == self.ce.lse.data_ptr()):
                raise ValueError("copy-engine transport: outputs must be the registered home buffers")
            self.ce.step(q, k, v, do, dk_acc, dv_acc, compute=(mode != "comm"), move=(mode != "signal"))
            return
        comm = self.comm_stream if mode == "pingpong" else comp
        ev = lambda: torch.cuda.Event()
        dk_acc.zero_()
        dv_acc.zero_()
        if mode == "compute":
            n_layers = self.ce.layers if getattr(self, "ce", None) is not None else 1
            for l in range(n_layers):
                for h in (0, 1):
                    self.ca_fwd(h, comp, l)
            for l in range(n_layers - 1, -1, -1):
                for h in (0, 1):
                    self.ca_bwd(h, comp, l)
            return
        if mode == "comm":
            for h in (0, 1):
                self.dispatch_fwd(h, q, k, v, comp)
            for h in (0, 1):
                self.return_fwd(h, o, lse, comp)
            for h in (0, 1):
                self.dispatch_bwd(h, do, comp)
            for h in (0, 1):
                self.return_bwd(h, dq, dk_acc, dv_acc, comp)
            return
        start = ev()
        start.record(comp)
        comm.wait_event(start)
        # comm stream: D(0) D(1) dO(0) dO(1) | R(0) R(1) | BR(0) BR(1)
        # compute:            F(0) F(1)        B(0) B(1)
        # so R(h) hides under F(1-h)/B(0), dO dispatch under F, BR(0) under B(1);
        # only D(0) and BR(1) are exposed (the reference's ping-pong windows,
        # P/src/sim.cpp:69-72, for a CA-only layer).
        ready_f, ready_b = [], []
        for h in (0, 1):
            self.dispatch_fwd(h, q, k, v, comm)
            e = ev()
            e.record(comm)
            ready_f.append(e)
        for h in (0, 1):
            self.dispatch_bwd(h, do, comm)
            e = ev()
            e.record(comm)
            ready_b.append(e)
        done_f = []
        for h in (0, 1):
            comp.wait_event(ready_f[h])
            self.ca_fwd(h, comp)
            e = ev()
            e.record(comp)
            done_f.append(e)
        for h in (0, 1):
            comm.wait_event(done_f[h])
            self.return_fwd(h, o, lse, comm)
        done_b = []
        for h in (0, 1):
            comp.wait_event(ready_b[h])
            self.ca_bwd(h, comp)
            e = ev()
            e.record(comp)
            done_b.append(e)
        for h in (0, 1):
            comm.wait_event(done_b[h])
            self.return_bwd(h, dq, dk_acc, dv_acc, comm)
        fin = ev()
        fin.record(comm)
        comp.wait_event(fin)


# --------------------------------------------------------------------------
# Copy-engine transport: every rank pushes its rows straight into the peers'
# buffers (CUDA IPC mappings) with cudaMemcpyAsync, so no SM is taken from
# the persistent CA kernels; GPU-side 32-bit flags (cuStreamWriteValue32 on
# the peer's flag word after the copies, cuStreamWaitValue32 on the local
# word before use) order producer and consumer streams across processes
# without host synchronisation.

F_QKV, F_DO, F_O, F_G, F_DONE = 0, 1, 2, 3, 4  # flag kinds (x2 halves, F_DONE uses half 0)
_DEBUG_COPY = bool(os.environ.get("CAD_DEBUG_COPY"))  # per-copy timing prints (rank 0)


def _runs(src: np.ndarray, dst: np.ndarray) -> np.ndarray:
    """Maximal runs where both src and dst rows advance by one."""
    if len(src) == 0:
        return np.zeros((0, 3), dtype=np.int64)
    brk = np.nonzero((np.diff(src) != 1) | (np.diff(dst) != 1))[0] + 1
    starts = np.concatenate([[0], brk])
    ends = np.concatenate([brk, [len(src)]])
    return np.stack([src[starts], dst[starts], ends - starts], axis=1).astype(np.int64)


def _split(counts, arr):
    out, o = [], 0
    for c in counts:
        out.append(arr[o:o + int(c)])
        o += int(c)
    return out


class _RunList:
    def __init__(self, runs: np.ndarray):
        self.n = len(runs)
        self.arr_np = np.asarray(runs, dtype=np.int64).reshape(-1, 3)
        self.arr = (N.cad_run * max(1, self.n))()
        for i, (a, b, c) in enumerate(runs.tolist()):
            self.arr[i] = N.cad_run(a, b, c)


class CETransport:
    """Row pushes over CUDA IPC for one DistCALayer. Needs every rank's
    LayerPlan (all ranks build them deterministically)."""

    def __init__(self, layer: "DistCALayer", all_plans: List[LayerPlan], o, lse, dq, layers: int = 1,
                 copy_mode: str = "ce", copy_ctas: int = 4):
        import torch.distributed as dist
        self.layer, self.plans = layer, all_plans
        lp = layer.lp
        W, me = lp.world, lp.rank
        self.W, self.me = W, me
        dev = layer.dev
        self.o, self.lse, self.dq = o, lse, dq
        self.layers = max(1, layers)
        # Server-side buffers per layer (layer 0 = the DistCALayer's halves):
        # a multi-layer step keeps every layer's forward activations on the
        # server for its backward, as a real stack would.
        self.lbufs = [layer.halves] + [layer.alloc_halves() for _ in range(1, self.layers)]
        # dK/dV partial staging per layer and half (rows in this rank's
        # KV_RET recv order)
        self.stage = []
        for _ in range(self.layers):
            st = []
            for h, hp in enumerate(lp.halves):
                n = max(1, hp.xfers[XFER_KV_RET].n_recv)
                st.append({"dk": torch.empty(n, layer.hkv, layer.d, dtype=torch.bfloat16, device=dev),
                           "dv": torch.empty(n, layer.hkv, layer.d, dtype=torch.bfloat16, device=dev),
                           "idx": layer.halves[h]["x"][XFER_KV_RET].recv_idx})
            self.stage.append(st)
        self.flags = torch.zeros(16 * W, dtype=torch.int32, device=dev)
        # buffers peers write into, exported once
        local = {"flags": self.flags, "o": o, "lse": lse, "dq": dq}
        for l in range(self.layers):
            for h, H in enumerate(self.lbufs[l]):
                for n_ in ("q", "k", "v", "do"):
                    local[f"{n_}{h}_{l}"] = H[n_]
                local[f"sdk{h}_{l}"] = self.stage[l][h]["dk"]
                local[f"sdv{h}_{l}"] = self.stage[l][h]["dv"]
        mine = {}
        for name, t in local.items():
            hb = (N.u8 * 64)()
            off = N.i64()
            check(lib().cad_ipc_handle(t.data_ptr(), hb, C.byref(off)))
            mine[name] = (bytes(hb), off.value)
        allh = [None] * W
        dist.all_gather_object(allh, mine)
        self.bases = []  # opened peer bases (to close)
        self.peer = []   # peer -> name -> device pointer
        for p in range(W):
            if p == me:
                self.peer.append({k: t.data_ptr() for k, t in local.items()})
                continue
            opened, ptrs = {}, {}
            for name, (hb, off) in allh[p].items():
                if hb not in opened:
                    base = C.c_void_p()
                    check(lib().cad_ipc_open((N.u8 * 64).from_buffer_copy(hb), C.byref(base)))
                    opened[hb] = base.value
                    self.bases.append(base.value)
                ptrs[name] = opened[hb] + off
            self.peer.append(ptrs)
        # row runs per (half, exchange, peer): what this rank pushes
        self.runs = {}
        for h in (0, 1):
            for x in range(4):
                mine_x = lp.halves[h].xfers[x]
                sends = _split(mine_x.send_counts, mine_x.send_idx)
                for p in range(W):
                    px = all_plans[p].halves[h].xfers[x]
                    dst = _split(px.recv_counts, px.recv_idx)[me]
                    if x == XFER_KV_RET:  # partials land in the owner's staging, in recv order
                        disp = int(px.recv_counts[:me].sum())
                        dst = np.arange(disp, disp + len(dst), dtype=np.int64)
                    self.runs[(h, x, p)] = _RunList(_runs(sends[p], dst))
        self.gen = 0
        self.launches = 0
        self.move = True
        self.trace = None  # list of (kind, layer, half, ev_before_wait, ev_after_wait, ev_done) when tracing
        self.local_stream = None  # set per step: the compute stream (own rows are copied there)
        self.local_on_comp = os.environ.get("CAD_LOCAL_ON_COMP", "1") != "0"
        # 'ce': copy-engine memcpys; 'sm': one copy kernel per transfer on
        # copy_ctas SMs left free by the CA kernels (the CA kernels' L2
        # traffic starves the copy engines)
        self.copy_mode = copy_mode
        self.copy_ctas = copy_ctas
        self._spans = {}

    def close(self):
        for b in self.bases:
            lib().cad_ipc_close(b)
        self.bases = []

    # flag word of (kind, half, src) on rank p
    def _flag(self, p, kind, h, src):
        return self.peer[p]["flags"] + 4 * ((kind * 2 + h) * self.W + src)

    def _signal(self, kind, h, stream):
        self._signal_v(kind, h, stream, self.gen)

    def _signal_v(self, kind, h, stream, value):
        for p in range(self.W):
            check(lib().cad_stream_write_u32(self._flag(p, kind, h, self.me), value, stream.cuda_stream))

    def _await(self, kind, h, stream, value=None):
        v = self.gen if value is None else value
        for src in range(self.W):
            check(lib().cad_stream_wait_u32(self._flag(self.me, kind, h, src), v, stream.cuda_stream))

    def _copy(self, h, x, src_ptr, dst_name, row_bytes, stream):
        """Push rows of exchange x (half h) from src_ptr into every peer's
        buffer dst_name: copy-engine memcpys, or one SM copy kernel on the
        reserved SMs (copy_mode 'sm')."""
        if self.copy_mode == "sm":
            key = (h, x, src_ptr, dst_name, row_bytes)
            spans = self._spans.get(key)
            if spans is None:
                rows = []
                for p in range(self.W):
                    if p == self.me and self.local_stream is not None:
                        continue  # local rows: copy engine on the compute stream (below)
                    rl = self.runs[(h, x, p)]
                    dst = self.peer[p][dst_name]
                    for r in rl.arr_np:
                        rows.append((src_ptr + int(r[0]) * row_bytes, dst + int(r[1]) * row_bytes,
                                     int(r[2]) * row_bytes))
                spans = torch.tensor(rows if rows else [(0, 0, 0)], dtype=torch.int64).to(self.layer.dev)
                spans = (spans, len(rows))
                self._spans[key] = spans
            if spans[1]:
                if _DEBUG_COPY and self.me == 0:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                check(lib().cad_copy_spans(spans[0].data_ptr(), spans[1], self.copy_ctas, stream.cuda_stream))
                if _DEBUG_COPY and self.me == 0:
                    e1.record(stream)
                    e1.synchronize()
                    sp = spans[0].cpu()
                    print(f"copy {key[:2]} {key[-2:]} spans={spans[1]} bytes={int(sp[:, 2].sum())} "
                          f"max_span={int(sp[:, 2].max())} ms={e0.elapsed_time(e1):.3f}", flush=True)
                self.launches += 1
            if self.local_stream is not None:
                rl = self.runs[(h, x, self.me)]
                if rl.n:
                    check(lib().cad_copy_runs(rl.arr, rl.n, src_ptr, self.peer[self.me][dst_name], row_bytes,
                                              self.local_stream.cuda_stream))
            return
        for p in range(self.W):
            rl = self.runs[(h, x, p)]
            if rl.n:
                # this rank's own rows move between its home and server buffers on
                # the compute stream, between kernels: a local copy overlapping a
                # CA kernel runs 10-30x slower (the kernels' L2 traffic starves the
                # copy engines) and would delay the remote pushes queued behind it
                st = self.local_stream if (p == self.me and self.local_stream is not None) else stream
                check(lib().cad_copy_runs(rl.arr, rl.n, src_ptr, self.peer[p][dst_name], row_bytes,
                                          st.cuda_stream))

    def _push(self, h, x, src, dst_name, row_bytes, stream):
        if not self.move:
            return
        self._copy(h, x, src.data_ptr(), dst_name, row_bytes, stream)

    def _push_lse(self, h, src_lse, stream):
        if not self.move:
            return
        L = self.layer
        if self.copy_mode == "sm":
            key = ("lse", h, src_lse.data_ptr())
            spans = self._spans.get(key)
            if spans is None:
                rows = []
                sr = src_lse.shape[1]
                for p in range(self.W):
                    if p == self.me and self.local_stream is not None:
                        continue
                    rl = self.runs[(h, XFER_O_RET, p)]
                    dr = self.plans[p].home_rows
                    for r in rl.arr_np:
                        for hd in range(L.hq):
                            rows.append((src_lse.data_ptr() + 4 * (hd * sr + int(r[0])),
                                         self.peer[p]["lse"] + 4 * (hd * dr + int(r[1])), 4 * int(r[2])))
                spans = (torch.tensor(rows if rows else [(0, 0, 0)], dtype=torch.int64).to(L.dev), len(rows))
                self._spans[key] = spans
            if spans[1]:
                if _DEBUG_COPY and self.me == 0:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                check(lib().cad_copy_spans(spans[0].data_ptr(), spans[1], self.copy_ctas, stream.cuda_stream))
                if _DEBUG_COPY and self.me == 0:
                    e1.record(stream)
                    e1.synchronize()
                    sp = spans[0].cpu()
                    print(f"copy {key[:2]} {key[-2:]} spans={spans[1]} bytes={int(sp[:, 2].sum())} "
                          f"max_span={int(sp[:, 2].max())} ms={e0.elapsed_time(e1):.3f}", flush=True)
                self.launches += 1
            peers = [self.me] if self.local_stream is not None else []
        else:
            peers = range(self.W)
        for p in peers:
            rl = self.runs[(h, XFER_O_RET, p)]
            if rl.n:
                dst_rows = self.plans[p].home_rows
                st = self.local_stream if (p == self.me and self.local_stream is not None) else stream
                check(lib().cad_copy_runs_cols(rl.arr, rl.n, src_lse.data_ptr(), src_lse.shape[1],
                                               self.peer[p]["lse"], dst_rows, L.hq, st.cuda_stream))

    def step(self, q, k, v, do, dk_acc, dv_acc, compute: bool = True, move: bool = True):
        """One step = self.layers CA layers, forward then backward.
        compute=False moves the same rows without running the CA kernels
        (comm-only time); move=False keeps every flag/ordering but skips the
        row copies (the reference's 'signal' mode, sim.hpp:14-18, where each
        transfer shrinks to a message).

        Between layers the context-independent part of the model is the
        identity: layer l+1's Q/K/V of half h leave home once every server
        has returned O(h, l), and layer l's dO of half h once every dQ/dK/dV
        partial of layer l+1 is back. So with L > 1 the ping-pong also runs
        across layers: the return of half h of layer l and the dispatch of
        half h of layer l+1 hide under CA(1-h) (the reference hides them under
        the CI layers, P/src/sim.cpp:69-125)."""
        if self.layers > 1:
            return self._step_layers(q, k, v, do, dk_acc, dv_acc, compute, move)
        L = self.layer
        self.move = move
        comp = torch.cuda.current_stream(L.dev)
        comm = L.comm_stream
        self.local_stream = comp if self.local_on_comp else None
        self.gen += 1
        g = self.gen
        start = torch.cuda.Event()
        start.record(comp)
        comm.wait_event(start)
        # every peer finished step g-1 (its buffers are free to overwrite)
        self._await(F_DONE, 0, comm, g - 1)
        # host enqueue order interleaves the two streams so the first CA
        # kernel is queued as soon as its inputs are, not after every push
        fwd_done, bwd_done = [], []

        def dispatch_qkv(h):
            self._push(h, XFER_Q, q, f"q{h}_0", L.q_row, comm)
            self._push(h, XFER_KV, k, f"k{h}_0", L.kv_row, comm)
            self._push(h, XFER_KV, v, f"v{h}_0", L.kv_row, comm)
            self._signal(F_QKV, h, comm)

        def ca(h, fwd):
            self._await(F_QKV if fwd else F_DO, h, comp)
            if compute:
                (L.ca_fwd if fwd else L.ca_bwd)(h, comp)
            e = torch.cuda.Event()
            e.record(comp)
            (fwd_done if fwd else bwd_done).append(e)

        dispatch_qkv(0)
        ca(0, True)
        dispatch_qkv(1)
        for h in (0, 1):
            self._push(h, XFER_Q, do, f"do{h}_0", L.q_row, comm)
            self._signal(F_DO, h, comm)
        ca(1, True)
        for h in (0, 1):
            comm.wait_event(fwd_done[h])
            H = L.halves[h]
            self._push(h, XFER_O_RET, H["o"], "o", L.q_row, comm)
            self._push_lse(h, H["lse"], comm)
            self._signal(F_O, h, comm)
            ca(h, False)
        for h in (0, 1):
            comm.wait_event(bwd_done[h])
            H = L.halves[h]
            self._push(h, XFER_O_RET, H["dq"], "dq", L.q_row, comm)
            self._push(h, XFER_KV_RET, H["dk"], f"sdk{h}_0", L.kv_row, comm)
            self._push(h, XFER_KV_RET, H["dv"], f"sdv{h}_0", L.kv_row, comm)
            self._signal(F_G, h, comm)
        dk_acc.zero_()
        dv_acc.zero_()
        for h in (0, 1):
            self._await(F_O, h, comp)
            self._await(F_G, h, comp)
            st = self.stage[0][h]
            n = L.lp.halves[h].xfers[XFER_KV_RET].n_recv
            check(lib().cad_scatter_add_bf16(st["dk"].data_ptr(), st["idx"].data_ptr(), n, L.hkv * L.d,
                                             dk_acc.data_ptr(), comp.cuda_stream))
            check(lib().cad_scatter_add_bf16(st["dv"].data_ptr(), st["idx"].data_ptr(), n, L.hkv * L.d,
                                             dv_acc.data_ptr(), comp.cuda_stream))
            self.launches += 2
        self._signal(F_DONE, 0, comp)

    # ------------------------------------------------------------ L layers
    def _push_l(self, h, x, src, name, l, row_bytes, stream):
        if not self.move:
            return
        self._copy(h, x, src.data_ptr(), f"{name}{h}_{l}", row_bytes, stream)

    def _step_layers(self, q, k, v, do, dk_acc, dv_acc, compute, move):
        L = self.layer
        NL = self.layers
        self.move = move
        comp = torch.cuda.current_stream(L.dev)
        comm = L.comm_stream
        self.local_stream = comp if self.local_on_comp else None
        # flag values of this step, increasing in issue order (waits are >=):
        # forward layer l -> g0 + 1 + l, backward layer l -> g0 + 2 NL - l,
        # F_DONE -> g0 + 2 NL
        g0 = self.gen
        self.gen += 2 * NL
        start = torch.cuda.Event()
        start.record(comp)
        comm.wait_event(start)
        self._await(F_DONE, 0, comm, g0)  # every peer finished the previous step

        def gl(l):
            return g0 + 1 + l

        def gb(l):
            return g0 + 2 * NL - l

        def tr_comm(tag, l, h, fn):
            if self.trace is None:
                return fn()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(comm)
            fn()
            b.record(comm)
            self.trace.append((tag, l, h, a, a, b))

        def dispatch_qkv(h, l):
            def f():
                self._push_l(h, XFER_Q, q, "q", l, L.q_row, comm)
                self._push_l(h, XFER_KV, k, "k", l, L.kv_row, comm)
                self._push_l(h, XFER_KV, v, "v", l, L.kv_row, comm)
            tr_comm("D", l, h, f)
            self._signal_v(F_QKV, h, comm, gl(l))

        def dispatch_do(h, l):
            tr_comm("dO", l, h, lambda: self._push_l(h, XFER_Q, do, "do", l, L.q_row, comm))
            self._signal_v(F_DO, h, comm, gb(l))

        def ca(h, l, fwd):
            if self.trace is not None:
                e_pre = torch.cuda.Event(enable_timing=True)
                e_pre.record(comp)
            self._await(F_QKV if fwd else F_DO, h, comp, gl(l) if fwd else gb(l))
            if self.trace is not None:
                e_go = torch.cuda.Event(enable_timing=True)
                e_go.record(comp)
            H = self.lbufs[l][h]
            if compute and L.halves[h]["plan"] is not None:
                plan = L.halves[h]["plan"]
                if fwd:
                    plan.forward(H["q"], H["k"], H["v"], H["o"], H["lse"], stream=comp)
                    L.launches += 1
                else:
                    H["dk"].zero_()
                    H["dv"].zero_()
                    plan.backward(H["q"], H["k"], H["v"], H["o"], H["lse"], H["do"], H["dq"], H["dk"], H["dv"],
                                  L.halves[h]["ws"], stream=comp)
                    L.launches += 3
            e = torch.cuda.Event(enable_timing=self.trace is not None)
            e.record(comp)
            if self.trace is not None:
                self.trace.append(("F" if fwd else "B", l, h, e_pre, e_go, e))
            return e

        def ret_o(h, l, ev):
            comm.wait_event(ev)
            H = self.lbufs[l][h]
            if self.trace is not None:
                ta = torch.cuda.Event(enable_timing=True)
                ta.record(comm)
            if self.move:
                self._copy(h, XFER_O_RET, H["o"].data_ptr(), "o", L.q_row, comm)
                self._push_lse(h, H["lse"], comm)
            if self.trace is not None:
                tb = torch.cuda.Event(enable_timing=True)
                tb.record(comm)
                self.trace.append(("R", l, h, ta, ta, tb))
            self._signal_v(F_O, h, comm, gl(l))

        def ret_g(h, l, ev):
            comm.wait_event(ev)
            H = self.lbufs[l][h]
            if self.trace is not None:
                ta = torch.cuda.Event(enable_timing=True)
                ta.record(comm)
            if self.move:
                self._copy(h, XFER_O_RET, H["dq"].data_ptr(), "dq", L.q_row, comm)
            self._push_l(h, XFER_KV_RET, H["dk"], "sdk", l, L.kv_row, comm)
            self._push_l(h, XFER_KV_RET, H["dv"], "sdv", l, L.kv_row, comm)
            if self.trace is not None:
                tb = torch.cuda.Event(enable_timing=True)
                tb.record(comm)
                self.trace.append(("G", l, h, ta, ta, tb))
            self._signal_v(F_G, h, comm, gb(l))

        # forward: comm D(0,0) D(1,0) | R(0,l) D(0,l+1) | R(1,l) D(1,l+1) | ...
        #          comp      F(0,0) F(1,0) F(0,1) F(1,1) ...
        dispatch_qkv(0, 0)
        ev0 = ca(0, 0, True)
        dispatch_qkv(1, 0)
        dispatch_do(0, NL - 1)  # the loss gradient of the top layer
        dispatch_do(1, NL - 1)
        pend = [ev0, None]
        pend[1] = ca(1, 0, True)
        for l in range(NL):
            for h in (0, 1):
                ret_o(h, l, pend[h])
                if l + 1 < NL:
                    self._await(F_O, h, comm, gl(l))  # identity CI: O(h, l) home -> Q/K/V(h, l+1)
                    dispatch_qkv(h, l + 1)
                    pend[h] = ca(h, l + 1, True)
        # backward, top layer first: comm G(0,l) dO(0,l-1) | G(1,l) dO(1,l-1) ...
        pend = [ca(0, NL - 1, False), ca(1, NL - 1, False)]
        dk_acc.zero_()
        dv_acc.zero_()
        for l in range(NL - 1, -1, -1):
            for h in (0, 1):
                ret_g(h, l, pend[h])
                if l > 0:
                    self._await(F_G, h, comm, gb(l))  # identity CI: dQ(h, l) home -> dO(h, l-1)
                    dispatch_do(h, l - 1)
                    pend[h] = ca(h, l - 1, False)
        for h in (0, 1):
            self._await(F_O, h, comp, gl(NL - 1))
            self._await(F_G, h, comp, gb(0))
        for l in range(NL - 1, -1, -1):
            for h in (0, 1):
                st = self.stage[l][h]
                n = L.lp.halves[h].xfers[XFER_KV_RET].n_recv
                check(lib().cad_scatter_add_bf16(st["dk"].data_ptr(), st["idx"].data_ptr(), n, L.hkv * L.d,
                                                 dk_acc.data_ptr(), comp.cuda_stream))
                check(lib().cad_scatter_add_bf16(st["dv"].data_ptr(), st["idx"].data_ptr(), n, L.hkv * L.d,
                                                 dv_acc.data_ptr(), comp.cuda_stream))
                self.launches += 2
        self._signal_v(F_DONE, 0, comp, g0 + 2 * NL)
