"""Measured B200 latency grid of the CA kernel, in the reference's profiler
schema.

The reference charges every CA-task `profile_lookup(grid, n_q, n_kv)` from a
`ProfilerGrid` that is either synthesised (`synth_grid`,
P/src/cost.cpp:164-202) or loaded from a CSV "q,kv,latency_s"
(`grid_from_csv`, P/src/cost.cpp:204-262). This module measures that grid on
the real sm_100a kernels (one CA call of a single task per point, CUDA
events) so cadsim's simulator runs on B200 data: feed the CSV to
`grid_from_csv(in, peak_throughput, alpha_flops = 4 * hidden, tile_size)`.
"""
from __future__ import annotations

import io
from typing import List, Sequence, Tuple

import torch

from .ca import CAPlan, CATaskRows
from .configs import Shape


def grid_points(tile: int, max_len: int) -> List[int]:
    """The reference's grid abscissae (make_points, P/src/cost.cpp:172-185)."""
    max_len = max(max_len, tile)
    pts, p = [], max(1, tile // 4)
    while p < tile:
        pts.append(p)
        p *= 2
    p = tile
    while p < max_len:
        pts.append(p)
        nxt = -(-(int(p * 1.2) + 1) // tile) * tile
        p = max(nxt, p + tile)
    pts.append(max_len)
    return pts


def measure_grid(shape: Shape, max_len: int, tile: int = 128, part: str = "fwd", reps: int = 3,
                 q_points: Sequence[int] = None, kv_points: Sequence[int] = None
                 ) -> Tuple[List[int], List[int], List[float]]:
    """Latency (s) of one CA call per (q, kv) point. part: 'fwd' or 'fwd+bwd'.
    Points below the causal diagonal (kv < q) carry the (q, q) latency, and
    sub-tile extents the padded tile's, as in synth_grid."""
    qp = list(q_points) if q_points is not None else grid_points(tile, max_len)
    kp = list(kv_points) if kv_points is not None else grid_points(tile, max_len)
    dev = torch.device("cuda")
    cache = {}
    lat = []
    big = max(max(qp), max(kp), tile)
    q = torch.randn(big, shape.h_q, shape.head_dim, device=dev, dtype=torch.bfloat16)
    k = torch.randn(big, shape.h_kv, shape.head_dim, device=dev, dtype=torch.bfloat16)
    v = torch.randn_like(k)
    do = torch.randn_like(q)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for qv in qp:
        for kvv in kp:
            nq = max(qv, 1)
            nk = max(kvv, nq)
            key = (nq, nk)
            if key not in cache:
                plan = CAPlan([CATaskRows(0, nq, 0, nk)], shape.h_q, shape.h_kv, big, big)
                o, lse = plan.forward(q, k, v)
                ws = torch.empty(plan.workspace_bytes, dtype=torch.uint8, device=dev)
                dq, dk, dv = torch.empty_like(q), torch.zeros_like(k), torch.zeros_like(v)

                def run():
                    plan.forward(q, k, v, o, lse)
                    if part != "fwd":
                        plan.backward(q, k, v, o, lse, do, dq, dk, dv, ws)

                run()
                torch.cuda.synchronize()
                st.record()
                for _ in range(reps):
                    run()
                en.record()
                torch.cuda.synchronize()
                cache[key] = st.elapsed_time(en) / reps / 1e3
                plan.close()
            lat.append(cache[key])
    # validate_grid (P/src/cost.cpp:68-91) requires latency non-decreasing in
    # q and in kv; timing noise between neighbouring points can break that,
    # so take the running max along both axes (a noise-level adjustment).
    nk = len(kp)
    for i in range(len(qp)):
        for j in range(nk):
            m = lat[i * nk + j]
            if i > 0:
                m = max(m, lat[(i - 1) * nk + j])
            if j > 0:
                m = max(m, lat[i * nk + j - 1])
            lat[i * nk + j] = m
    return qp, kp, lat


def grid_to_csv(q_points, kv_points, latency_s) -> str:
    """grid_to_csv (P/src/cost.cpp:204-213): header, row-major q then kv, %.17g."""
    out = io.StringIO()
    out.write("q,kv,latency_s\n")
    i = 0
    for qv in q_points:
        for kvv in kv_points:
            out.write(f"{qv},{kvv},{latency_s[i]:.17g}\n")
            i += 1
    return out.getvalue()
