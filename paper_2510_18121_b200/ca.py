"""Device entry points of the CA hot path (cad_ca_* in include/cad.h).

The CA kernel is what the reference only models (task_layer_seconds ->
profile_lookup, P/src/sim.cpp:22-30): one fused call per server and
nano-batch half over all of that server's CA-tasks.
torch is used only for device memory and streams; the compute is the
sm_100a kernels in lib/libcad.so. There is no fallback path: a missing
library or a non-CUDA tensor raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import torch

from . import _native as N
from ._native import check, lib

HEAD_DIM = 128
BWD_DELTA, BWD_DKDV, BWD_DQ, BWD_ALL = 1, 2, 4, 7


@dataclass(frozen=True)
class CATaskRows:
    """One CA-task as the server kernel sees it (rows of the packed buffers):
    q rows [q_off, q_off+n_q) attend kv rows [kv_off, kv_off+kv_len) with a
    bottom-right causal mask (query i sees keys 0..kv_len-n_q+i)."""
    q_off: int
    n_q: int
    kv_off: int
    kv_len: int


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _need(t: torch.Tensor, name: str, dtype=torch.bfloat16) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU path exists)")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t.data_ptr()


class CAPlan:
    """Device work list for one task set (built once, reused per layer)."""

    def __init__(self, tasks: Sequence[CATaskRows], h_q: int, h_kv: int, q_rows: int,
                 kv_rows: int, softmax_scale: float = 0.0, head_dim: int = HEAD_DIM):
        arr = (N.cad_ca_task * max(1, len(tasks)))()
        for i, t in enumerate(tasks):
            arr[i] = N.cad_ca_task(t.q_off, t.n_q, t.kv_off, t.kv_len)
        shape = N.cad_ca_shape(h_q, h_kv, head_dim, softmax_scale, q_rows, kv_rows)
        h = C.c_void_p()
        check(lib().cad_ca_plan_create(arr, len(tasks), C.byref(shape), C.byref(h)))
        self._h = h
        self.tasks = list(tasks)
        self.h_q, self.h_kv, self.q_rows, self.kv_rows = h_q, h_kv, q_rows, kv_rows
        info = N.cad_ca_plan_info()
        check(lib().cad_ca_plan_info_get(self._h, C.byref(info)))
        self.n_fwd_units, self.n_bwd_units = info.n_fwd_units, info.n_bwd_units
        self.causal_pairs = info.causal_pairs
        self.fwd_flops, self.bwd_flops = info.fwd_flops, info.bwd_flops
        self.workspace_bytes = info.workspace_bytes

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().cad_ca_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                o: Optional[torch.Tensor] = None, lse: Optional[torch.Tensor] = None,
                stream: Optional[torch.cuda.Stream] = None) -> Tuple[torch.Tensor, torch.Tensor]:
        if o is None:
            o = torch.empty_like(q)
        if lse is None:
            lse = torch.empty(self.h_q, self.q_rows, dtype=torch.float32, device=q.device)
        check(lib().cad_ca_fwd(self._h, _need(q, "q"), _need(k, "k"), _need(v, "v"), _need(o, "o"),
                               _need(lse, "lse", torch.float32), _stream_ptr(stream)))
        return o, lse

    def backward(self, q, k, v, o, lse, do, dq=None, dk=None, dv=None, workspace=None,
                 stream: Optional[torch.cuda.Stream] = None, parts: int = BWD_ALL):
        if dq is None:
            dq = torch.empty_like(q)
        if dk is None:
            dk = torch.zeros_like(k)
        if dv is None:
            dv = torch.zeros_like(v)
        if workspace is None:
            workspace = torch.empty(max(1, self.workspace_bytes), dtype=torch.uint8, device=q.device)
        check(lib().cad_ca_bwd_parts(self._h, _need(q, "q"), _need(k, "k"), _need(v, "v"), _need(o, "o"),
                                     _need(lse, "lse", torch.float32), _need(do, "do"), _need(dq, "dq"),
                                     _need(dk, "dk"), _need(dv, "dv"),
                                     _need(workspace, "workspace", torch.uint8), workspace.numel(),
                                     parts, _stream_ptr(stream)))
        return dq, dk, dv
