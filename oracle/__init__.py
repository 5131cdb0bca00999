"""TEST INFRASTRUCTURE ONLY: Python access to the checkers under oracle/_ref.

  libcadsim_ref.so  the unmodified reference scheduler (cadsim) + C shim
  libca_oracle.so   the CPU restatement of the CA numerics (ca_oracle.c;
                    parity unpinned upstream, see its header)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
legs may import this package. The product (paper_2510_18121_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")


def build() -> None:
    """make -C oracle (the reference part only where /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(name: str) -> C.CDLL:
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_ref = None
_num = None


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        from paper_2510_18121_b200 import _native as N
        P, vp = C.POINTER, C.c_void_p
        h = _load("libcadsim_ref.so")
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_sample_batch": (C.c_int, [P(N.cad_length_dist), N.i64, P(N.i64), N.i64, P(N.i64)]),
            "ref_place_sequential": (C.c_int, [P(N.i64), N.i64, N.i64, N.i64, P(N.cad_item), N.i64, P(N.i64)]),
            "ref_ca_flops_core": (C.c_int, [P(N.cad_item), P(N.i64)]),
            "ref_one_tile_slack": (C.c_int, [P(N.cad_item), N.i64, P(N.cad_sched_cfg), P(N.f64)]),
            "ref_target_load": (C.c_int, [P(N.cad_item), N.i64, N.i64, N.f64, P(N.f64)]),
            "ref_v_min_comm": (C.c_int, [P(N.cad_comm_query), N.i64, P(N.cad_shard_choice)]),
            "ref_propose_migration": (C.c_int, [P(N.cad_server_load), P(N.cad_server_load), P(N.cad_item),
                                                N.f64, P(N.cad_sched_cfg), P(N.cad_proposal), P(N.i32)]),
            "ref_schedule": (vp, [P(N.cad_item), N.i64, N.i64, P(N.cad_sched_cfg), P(N.i32), N.i64]),
            "ref_plan_text": (C.c_char_p, [vp]),
            "ref_plan_devices": (C.c_char_p, [vp]),
            "ref_plan_stats": (None, [vp, P(N.cad_plan_stats)]),
            "ref_plan_tasks": (P(N.cad_task), [vp, P(N.i64)]),
            "ref_plan_servers": (None, [vp, P(N.f64), P(N.i64), P(N.i64), P(N.i64)]),
            "ref_plan_free": (None, [vp]),
            "ref_schedule_seconds": (N.f64, [P(N.cad_item), N.i64, N.i64, P(N.cad_sched_cfg), N.i64]),
            "ref_grid_lookup": (N.f64, [C.c_char_p, N.f64, N.f64, N.i64, N.i64, N.i64]),
            "ref_pp_iteration": (C.c_int, [P(N.cad_item), P(N.i64), N.i64, P(N.i64), N.i64, N.i64, C.c_int32,
                                           P(N.cad_sched_cfg), P(N.i64), P(N.i64), P(C.c_int32), N.i64,
                                           P(N.i64)]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(h, name)
            fn.restype, fn.argtypes = res, args
        _ref = h
    return _ref


def num_lib() -> C.CDLL:
    global _num
    if _num is None:
        h = _load("libca_oracle.so")
        vp, i64, dbl, ci = C.c_void_p, C.c_int64, C.c_double, C.c_int
        h.oracle_ca_fwd.restype = None
        h.oracle_ca_fwd.argtypes = [vp, i64, ci, ci, ci, dbl, vp, vp, vp, vp, vp, i64, ci]
        h.oracle_ca_bwd.restype = None
        h.oracle_ca_bwd.argtypes = [vp, i64, ci, ci, ci, dbl, vp, vp, vp, vp, vp, vp, vp, vp, i64, i64, ci]
        h.oracle_max_threads.restype = ci
        _num = h
    return _num


def _tasks_array(tasks):
    a = np.zeros((max(1, len(tasks)), 4), dtype=np.int64)
    for i, t in enumerate(tasks):
        a[i] = (t[0], t[1], t[2], t[3]) if not hasattr(t, "q_off") else (t.q_off, t.n_q, t.kv_off, t.kv_len)
    return a


def _f32(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    return x, x.ctypes.data


def ca_forward(tasks, q, k, v, scale=None, threads=0):
    """q [Tq,Hq,D], k/v [Tkv,Hkv,D] float32 -> (o [Tq,Hq,D], lse [Hq,Tq])."""
    q, qp = _f32(q)
    k, kp = _f32(k)
    v, vpp = _f32(v)
    tq, hq, d = q.shape
    hkv = k.shape[1]
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    o = np.zeros_like(q)
    lse = np.full((hq, tq), np.nan, dtype=np.float32)
    ta = _tasks_array(tasks)
    num_lib().oracle_ca_fwd(ta.ctypes.data, len(tasks), hq, hkv, d, scale, qp, kp, vpp,
                            o.ctypes.data, lse.ctypes.data, tq, threads)
    return o, lse


def ca_backward(tasks, q, k, v, o, do, scale=None, threads=0):
    """-> (dq, dk, dv) float32; dk/dv summed over tasks sharing kv rows."""
    q, qp = _f32(q)
    k, kp = _f32(k)
    v, vpp = _f32(v)
    o, op = _f32(o)
    do, dop = _f32(do)
    tq, hq, d = q.shape
    tkv, hkv = k.shape[0], k.shape[1]
    scale = 1.0 / np.sqrt(d) if scale is None else scale
    dq = np.zeros_like(q)
    dk = np.zeros_like(k)
    dv = np.zeros_like(v)
    ta = _tasks_array(tasks)
    num_lib().oracle_ca_bwd(ta.ctypes.data, len(tasks), hq, hkv, d, scale, qp, kp, vpp, op, dop,
                            dq.ctypes.data, dk.ctypes.data, dv.ctypes.data, tq, tkv, threads)
    return dq, dk, dv
