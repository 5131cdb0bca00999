"""Per-layer CA dispatch / compute / return on one rank (one GPU).

The reference only models this step: device_plans_from_schedule splits each
device's served tasks into ping/pong halves and layer_windows hides
dispatch(pong) under CA(ping) and return(ping) under CA(pong)
(P/src/sim.cpp:34-46,69-125). Here it runs for real, in C++ behind the
C-ABI (cad_layer_ctx, csrc/cuda/layer_exec.cu):

  forward   Q/K/V rows home -> server  ->  CA fwd on the server  ->  O/LSE
            rows server -> home
  backward  dO rows home -> server  ->  CA bwd (Q/K/V/O/LSE stay resident on
            the server from the forward)  ->  dQ rows -> home, dK/dV partial
            rows -> owners, summed there (fp32)

This module is the ctypes binding plus the host-side row plan used by the CPU
tests (LayerPlan). torch only provides device memory, streams and the
torch.distributed exchange of the contexts' export blobs.
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
                                             int(balance_halves), C.byref(lp)))  # 0/False, 1/True, or 2 (one half)
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


TRANSPORTS = {"local": 0, "ipc": 1, "ce": 1, "nccl": 2}
MODES = {"pingpong": 0, "serial": 1, "compute": 2, "comm": 3, "signal": 4, "comm_local": 5}
DISPATCH_QKV, DISPATCH_DO, DISPATCH_FWD_STATE = 0, 1, 2
PASSES = {"fwd": 1, "bwd": 2, "both": 3}
RETURN_O, RETURN_GRAD = 0, 1


def _p(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class _CudaMem:
    """__cuda_array_interface__ over context-owned device memory (no copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


def _wrap(ptr: int, shape, dtype, device) -> torch.Tensor:
    """A torch tensor viewing `ptr` (the context keeps the memory alive)."""
    if dtype == torch.bfloat16:  # no bf16 typestr: view the bits as int16
        t = torch.as_tensor(_CudaMem(ptr, shape, "<i2"), device=device)
        return t.view(torch.bfloat16)
    return torch.as_tensor(_CudaMem(ptr, shape, "<f4"), device=device)


class DistCALayer:
    """One rank's CA layer executor (cad_layer_ctx).

    transport: 'ipc' (alias 'ce'; CUDA-IPC copy-engine pushes + GPU flags,
    one process per GPU), 'nccl' (all-to-allv), or 'local' (every rank's
    context in this process, e.g. a world-W layer on one GPU).
    layers > 1 is a benchmark mode: that many stacked CA layers per step with
    the identity between them; dK/dV come back SUMMED over the layers."""

    def __init__(self, lp: LayerPlan, device: torch.device, transport: str = "ipc", layers: int = 1,
                 reserve_sms: int = 0, balance_halves: bool = False, softmax_scale: float = 0.0,
                 bench_stacked: bool = False):
        if layers > 1 and not bench_stacked:
            # a stacked step sums dK/dV over identical layers: only meaningful as a benchmark
            raise ValueError("layers > 1 is a benchmark mode (dK/dV summed over identical layers); "
                             "pass bench_stacked=True")
        self.lp, self.dev, self.transport, self.layers = lp, device, transport, layers
        sh = lp.shape
        self.hq, self.hkv, self.d = sh.h_q, sh.h_kv, sh.head_dim
        cfg = N.cad_layer_cfg(lp.rank, lp.world, sh.h_q, sh.h_kv, sh.head_dim, softmax_scale,
                              TRANSPORTS[transport], layers, int(balance_halves), reserve_sms)
        ph = S.PlanHandle(lp.home_items, lp.world, lp.cfg)
        arr = (N.cad_item * max(1, len(lp.home_items)))(*[i.to_c() for i in lp.home_items])
        self._h = C.c_void_p()
        with torch.cuda.device(device):
            try:
                check(lib().cad_layer_ctx_create(ph.h, arr, len(lp.home_items), C.byref(cfg), C.byref(self._h)))
            finally:
                ph.close()
        info = self.info()
        self.home_rows = info.home_rows
        self.served_pairs = info.served_pairs
        self.blob_bytes = info.blob_bytes
        self.wire_bytes = [[info.wire_bytes[h][x] for x in range(4)] for h in (0, 1)]
        self.comm: Optional[Comm] = None
        self._io = None

    # ---------------------------------------------------------------- setup
    def info(self) -> N.cad_layer_ctx_info:
        info = N.cad_layer_ctx_info()
        check(lib().cad_layer_ctx_info_get(self._h, C.byref(info)))
        return info

    @property
    def launches(self) -> int:
        return int(self.info().launches)

    def bind_outputs(self, o: torch.Tensor, lse: torch.Tensor, dq: torch.Tensor) -> None:
        """No-op kept for the earlier contract (outputs now live in home())."""
        check(lib().cad_layer_ctx_bind_outputs(self._h, o.data_ptr(), lse.data_ptr(), dq.data_ptr()))

    def home(self, layer: int = 0) -> dict:
        """The layer's home buffers inside the context (zero-copy own rows), as
        tensors viewing that memory: q, k, v, do, o, dq [home_rows][heads][d]
        bf16 and lse [h_q][home_rows] fp32. Writing inputs there (and passing
        None in io) and reading outputs there skips the staging copies."""
        io = N.cad_layer_io()
        check(lib().cad_layer_ctx_home(self._h, layer, C.byref(io)))
        H, d = self.home_rows, self.d
        out = {}
        for name, ptr, heads, dt in (("q", io.q, self.hq, torch.bfloat16), ("k", io.k, self.hkv, torch.bfloat16),
                                     ("v", io.v, self.hkv, torch.bfloat16), ("do", io.dout, self.hq, torch.bfloat16),
                                     ("o", io.o, self.hq, torch.bfloat16), ("dq", io.dq, self.hq, torch.bfloat16)):
            out[name] = _wrap(ptr, (H, heads, d), dt, self.dev)
        out["lse"] = _wrap(io.lse, (self.hq, H), torch.float32, self.dev)
        return out

    def export(self) -> bytes:
        buf = C.create_string_buffer(self.blob_bytes)
        need = C.c_size_t()
        check(lib().cad_layer_ctx_export(self._h, buf, self.blob_bytes, C.byref(need)))
        return buf.raw[:need.value]

    def connect(self, blobs: Sequence[bytes]) -> None:
        joined = b"".join(blobs)
        check(lib().cad_layer_ctx_connect(self._h, joined, self.blob_bytes))

    def connect_dist(self) -> None:
        """Exchange the export blobs over torch.distributed and connect."""
        import torch.distributed as dist
        allb = [None] * self.lp.world
        dist.all_gather_object(allb, self.export())
        self.connect(allb)

    def set_comm(self, comm: "Comm") -> None:
        self.comm = comm
        check(lib().cad_layer_ctx_set_comm(self._h, comm.h))

    # ---------------------------------------------------------------- steps
    def io(self, q, k, v, do, o, lse, dq, dk=None, dv=None, dk_acc=None, dv_acc=None) -> N.cad_layer_io:
        """The home buffers of a step (kept alive by the caller)."""
        return N.cad_layer_io(_p(q), _p(k), _p(v), _p(do), _p(o), _p(lse), _p(dq), _p(dk), _p(dv),
                              _p(dk_acc), _p(dv_acc))

    def step(self, io: N.cad_layer_io, mode: str = "pingpong", stream: Optional[torch.cuda.Stream] = None,
             passes: str = "both"):
        """One step; passes 'fwd' / 'bwd' run one pass (a pipeline tick)."""
        s = (stream or torch.cuda.current_stream(self.dev)).cuda_stream
        check(lib().cad_layer_step_ex(self._h, C.byref(io), MODES[mode], PASSES[passes], s))

    def begin(self, stream, passes: str = "both"):
        check(lib().cad_layer_begin_ex(self._h, PASSES[passes], stream.cuda_stream))

    def dispatch(self, layer, half, what, io, stream, local_stream=None):
        if local_stream is None:
            check(lib().cad_dispatch(self._h, layer, half, what, C.byref(io), stream.cuda_stream))
        else:
            check(lib().cad_dispatch_ex(self._h, layer, half, what, C.byref(io), stream.cuda_stream,
                                        local_stream.cuda_stream))

    def compute(self, layer, half, backward, stream):
        check(lib().cad_layer_compute(self._h, layer, half, int(backward), stream.cuda_stream))

    def ret(self, layer, half, what, io, stream):
        check(lib().cad_return(self._h, layer, half, what, C.byref(io), stream.cuda_stream))

    def finish(self, io, stream):
        check(lib().cad_layer_finish(self._h, C.byref(io), stream.cuda_stream))

    def set_trace(self, on: bool) -> None:
        check(lib().cad_layer_ctx_set_trace(self._h, int(on)))

    TRACE_KINDS = ("D", "dO", "F", "B", "R", "G", "finish")

    def trace(self):
        """Phases of the last traced step: (kind, layer, half, t_begin,
        t_ready, t_end) in ms from the step's start."""
        n = N.i64()
        rc = lib().cad_layer_ctx_trace(self._h, None, 0, C.byref(n))
        if rc not in (0, N.CAD_ERR_CAPACITY):
            check(rc)
        recs = (N.cad_trace_rec * max(1, n.value))()
        check(lib().cad_layer_ctx_trace(self._h, recs, n.value, C.byref(n)))
        return [(self.TRACE_KINDS[r.kind], r.layer, r.half, round(r.t_begin, 3), round(r.t_ready, 3),
                 round(r.t_end, 3)) for r in recs[:n.value]]

    def close(self):
        if getattr(self, "_h", None):
            with torch.cuda.device(self.dev):
                lib().cad_layer_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
