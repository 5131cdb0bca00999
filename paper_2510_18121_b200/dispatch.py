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
                 cfg: Optional[S.SchedulerConfig] = None, tokens_per_device: Optional[int] = None):
        total = sum(lengths)
        self.world, self.rank, self.shape = world, rank, shape
        self.tokens_per_device = tokens_per_device or total // world
        self.home_items = S.place_sequential(lengths, world, self.tokens_per_device)
        self.cfg = cfg or CF.sched_config(shape)
        ph = S.PlanHandle(self.home_items, world, self.cfg)
        self.plan = ph.plan
        arr = (N.cad_item * max(1, len(self.home_items)))(*[i.to_c() for i in self.home_items])
        lp = C.c_void_p()
        q_row = shape.h_q * shape.head_dim * 2
        kv_row = 2 * shape.h_kv * shape.head_dim * 2
        check(lib().cad_layer_plan_create(ph.h, arr, len(self.home_items), rank, q_row, kv_row, C.byref(lp)))
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
        self.recv_buf = torch.empty(max_bytes, dtype=torch.uint8, device=device)
        self.launches = 0

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

    def ca_fwd(self, h, stream):
        H = self.halves[h]
        if H["plan"] is not None:
            H["plan"].forward(H["q"], H["k"], H["v"], H["o"], H["lse"], stream=stream)
            self.launches += 1

    def ca_bwd(self, h, stream):
        H = self.halves[h]
        if H["plan"] is not None:
            H["dk"].zero_()
            H["dv"].zero_()
            H["plan"].backward(H["q"], H["k"], H["v"], H["o"], H["lse"], H["do"], H["dq"], H["dk"], H["dv"],
                               H["ws"], stream=stream)
            self.launches += 3

    # ---------------------------------------------------------------- step
    def step(self, q, k, v, do, o, lse, dq, dk_acc, dv_acc, mode: str = "pingpong"):
        """One layer fwd+bwd. mode: 'pingpong' (comm of one half under CA of
        the other), 'serial' (single stream, no overlap), 'compute' (CA
        kernels only; server buffers assumed resident: the reference's
        'signal' bound), 'comm' (exchanges only)."""
        comp = torch.cuda.current_stream(self.dev)
        comm = self.comm_stream if mode == "pingpong" else comp
        ev = lambda: torch.cuda.Event()
        dk_acc.zero_()
        dv_acc.zero_()
        if mode == "compute":
            for h in (0, 1):
                self.ca_fwd(h, comp)
            for h in (0, 1):
                self.ca_bwd(h, comp)
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
