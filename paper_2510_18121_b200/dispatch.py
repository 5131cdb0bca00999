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
        self.ce = None

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
    def use_copy_engines(self, all_plans: List[LayerPlan], o, lse, dq):
        """Switch the exchanges to the copy-engine transport (CUDA IPC pushes);
        o/lse/dq become the registered home output buffers of every step."""
        self.ce = CETransport(self, all_plans, o, lse, dq)

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


# --------------------------------------------------------------------------
# Copy-engine transport: every rank pushes its rows straight into the peers'
# buffers (CUDA IPC mappings) with cudaMemcpyAsync, so no SM is taken from
# the persistent CA kernels; GPU-side 32-bit flags (cuStreamWriteValue32 on
# the peer's flag word after the copies, cuStreamWaitValue32 on the local
# word before use) order producer and consumer streams across processes
# without host synchronisation.

F_QKV, F_DO, F_O, F_G, F_DONE = 0, 1, 2, 3, 4  # flag kinds (x2 halves, F_DONE uses half 0)


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
        self.arr = (N.cad_run * max(1, self.n))()
        for i, (a, b, c) in enumerate(runs.tolist()):
            self.arr[i] = N.cad_run(a, b, c)


class CETransport:
    """Row pushes over CUDA IPC for one DistCALayer. Needs every rank's
    LayerPlan (all ranks build them deterministically)."""

    def __init__(self, layer: "DistCALayer", all_plans: List[LayerPlan], o, lse, dq):
        import torch.distributed as dist
        self.layer, self.plans = layer, all_plans
        lp = layer.lp
        W, me = lp.world, lp.rank
        self.W, self.me = W, me
        dev = layer.dev
        self.o, self.lse, self.dq = o, lse, dq
        # dK/dV partial staging per half (rows in this rank's KV_RET recv order)
        self.stage = []
        for hp in lp.halves:
            n = max(1, hp.xfers[XFER_KV_RET].n_recv)
            self.stage.append({"dk": torch.empty(n, layer.hkv, layer.d, dtype=torch.bfloat16, device=dev),
                               "dv": torch.empty(n, layer.hkv, layer.d, dtype=torch.bfloat16, device=dev),
                               "idx": layer.halves[lp.halves.index(hp)]["x"][XFER_KV_RET].recv_idx})
        self.flags = torch.zeros(16 * W, dtype=torch.int32, device=dev)
        # buffers peers write into, exported once
        local = {"flags": self.flags, "o": o, "lse": lse, "dq": dq}
        for h, H in enumerate(layer.halves):
            for n_ in ("q", "k", "v", "do"):
                local[f"{n_}{h}"] = H[n_]
            local[f"sdk{h}"] = self.stage[h]["dk"]
            local[f"sdv{h}"] = self.stage[h]["dv"]
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

    def close(self):
        for b in self.bases:
            lib().cad_ipc_close(b)
        self.bases = []

    # flag word of (kind, half, src) on rank p
    def _flag(self, p, kind, h, src):
        return self.peer[p]["flags"] + 4 * ((kind * 2 + h) * self.W + src)

    def _signal(self, kind, h, stream):
        for p in range(self.W):
            check(lib().cad_stream_write_u32(self._flag(p, kind, h, self.me), self.gen, stream.cuda_stream))

    def _await(self, kind, h, stream, value=None):
        v = self.gen if value is None else value
        for src in range(self.W):
            check(lib().cad_stream_wait_u32(self._flag(self.me, kind, h, src), v, stream.cuda_stream))

    def _push(self, h, x, src, dst_name, row_bytes, stream):
        if not self.move:
            return
        for p in range(self.W):
            rl = self.runs[(h, x, p)]
            if rl.n:
                check(lib().cad_copy_runs(rl.arr, rl.n, src.data_ptr(), self.peer[p][dst_name], row_bytes,
                                          stream.cuda_stream))

    def _push_lse(self, h, src_lse, stream):
        if not self.move:
            return
        L = self.layer
        for p in range(self.W):
            rl = self.runs[(h, XFER_O_RET, p)]
            if rl.n:
                dst_rows = self.plans[p].home_rows
                check(lib().cad_copy_runs_cols(rl.arr, rl.n, src_lse.data_ptr(), src_lse.shape[1],
                                               self.peer[p]["lse"], dst_rows, L.hq, stream.cuda_stream))

    def step(self, q, k, v, do, dk_acc, dv_acc, compute: bool = True, move: bool = True):
        """One layer. compute=False moves the same rows without running the
        CA kernels (comm-only time); move=False keeps every flag/ordering but
        skips the row copies (the reference's 'signal' mode, sim.hpp:14-18,
        where each transfer shrinks to a message)."""
        L = self.layer
        self.move = move
        comp = torch.cuda.current_stream(L.dev)
        comm = L.comm_stream
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
            self._push(h, XFER_Q, q, f"q{h}", L.q_row, comm)
            self._push(h, XFER_KV, k, f"k{h}", L.kv_row, comm)
            self._push(h, XFER_KV, v, f"v{h}", L.kv_row, comm)
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
            self._push(h, XFER_Q, do, f"do{h}", L.q_row, comm)
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
            self._push(h, XFER_KV_RET, H["dk"], f"sdk{h}", L.kv_row, comm)
            self._push(h, XFER_KV_RET, H["dv"], f"sdv{h}", L.kv_row, comm)
            self._signal(F_G, h, comm)
        dk_acc.zero_()
        dv_acc.zero_()
        for h in (0, 1):
            self._await(F_O, h, comp)
            self._await(F_G, h, comp)
            st = self.stage[h]
            n = L.lp.halves[h].xfers[XFER_KV_RET].n_recv
            check(lib().cad_scatter_add_bf16(st["dk"].data_ptr(), st["idx"].data_ptr(), n, L.hkv * L.d,
                                             dk_acc.data_ptr(), comp.cuda_stream))
            check(lib().cad_scatter_add_bf16(st["dv"].data_ptr(), st["idx"].data_ptr(), n, L.hkv * L.d,
                                             dv_acc.data_ptr(), comp.cuda_stream))
            self.launches += 2
        self._signal(F_DONE, 0, comp)
