"""ctypes binding of include/cad.h (lib/libcad.so).

The struct layouts below mirror include/cad.h field for field. The library is
built in-tree (``make -C paper_2510_18121_b200``); there is no fallback: if it
cannot be loaded every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CAD_LIB_PATH") or os.path.join(_HERE, "lib", "libcad.so")

i64, i32, u8, u64, f64, f32 = C.c_int64, C.c_int32, C.c_uint8, C.c_uint64, C.c_double, C.c_float

CAD_OK, CAD_ERR_CONFIG, CAD_ERR_DOMAIN, CAD_ERR_CUDA, CAD_ERR_NCCL, CAD_ERR_CAPACITY = 0, -1, -2, -3, -4, -5


class cad_item(C.Structure):
    _fields_ = [("doc", i64), ("q_begin", i64), ("q_end", i64), ("kv_extent", i64),
                ("ht_mirror", i64), ("home_device", i32), ("layout", u8), ("pad_", u8 * 3)]


class cad_task(C.Structure):
    _fields_ = [("item", cad_item), ("source_device", i32), ("assigned_server", i32),
                ("comm_bytes", i64), ("output_bytes", i64)]


class cad_sched_cfg(C.Structure):
    _fields_ = [("epsilon", f64), ("e_threshold", f64), ("tile_size", i64), ("alpha_ca", f64),
                ("size_q", i64), ("size_kv", i64), ("double_query_head_tail", u8),
                ("pad_", u8 * 7), ("max_moves", i64)]


class cad_server_load(C.Structure):
    _fields_ = [("device", i32), ("pad_", i32), ("assigned_flops", f64), ("assigned_core", i64),
                ("n_items", i64), ("sent_bytes", i64), ("received_bytes", i64)]


class cad_plan_stats(C.Structure):
    _fields_ = [("target", f64), ("max_load", f64), ("min_load", f64), ("epsilon_used", f64),
                ("total_comm_bytes", i64), ("total_output_bytes", i64), ("migrations", i64),
                ("splits", i64), ("rejected_small", i64), ("n_tasks", i64), ("n_servers", i64),
                ("tolerance_met", i32), ("pad_", i32)]


class cad_proposal(C.Structure):
    _fields_ = [("delta_f_max", f64), ("shard", cad_item), ("remainders", cad_item * 2),
                ("n_remainders", i32), ("whole_item", i32), ("v_comm", i64), ("priority", f64)]


class cad_comm_query(C.Structure):
    _fields_ = [("delta_f_max", f64), ("f_item", f64), ("L_q", i64), ("L_kv", i64),
                ("size_q", i64), ("size_kv", i64), ("layout", u8), ("pad_", u8 * 7),
                ("ht_mirror", i64)]


class cad_shard_choice(C.Structure):
    _fields_ = [("n_q", i64), ("n_kv", i64), ("bytes", i64), ("core", i64)]


class cad_length_dist(C.Structure):
    _fields_ = [("kind", i32), ("pad_", i32), ("max_doc_len", i64), ("min_len_threshold", i64),
                ("seed", u64), ("log_mu", f64), ("log_sigma", f64), ("upsample_drop_prob", f64),
                ("long_mix_weight", f64), ("long_log_mu", f64), ("long_log_sigma", f64),
                ("fixed_len", i64), ("uniform_min", i64), ("hist_len", C.POINTER(i64)),
                ("hist_p", C.POINTER(f64)), ("hist_n", i64)]


class cad_served_task(C.Structure):
    _fields_ = [("task_index", i64), ("in_bytes", i64), ("out_bytes", i64), ("half", i32),
                ("pad_", i32)]


class cad_ca_task(C.Structure):
    _fields_ = [("q_off", i64), ("n_q", i64), ("kv_off", i64), ("kv_len", i64)]


class cad_ca_shape(C.Structure):
    _fields_ = [("h_q", i32), ("h_kv", i32), ("head_dim", i32), ("softmax_scale", f32),
                ("q_rows", i64), ("kv_rows", i64)]


class cad_ca_plan_info(C.Structure):
    _fields_ = [("n_fwd_units", i64), ("n_bwd_units", i64), ("causal_pairs", i64),
                ("fwd_flops", f64), ("bwd_flops", f64), ("workspace_bytes", C.c_size_t)]


class cad_layer_half_info(C.Structure):
    _fields_ = [("home_rows", i64), ("q_rows", i64), ("kv_rows", i64), ("n_tasks", i64),
                ("tasks", C.POINTER(cad_ca_task)), ("task_index", C.POINTER(i64)),
                ("remote_send_bytes", i64 * 4)]


class cad_xfer(C.Structure):
    _fields_ = [("n_peers", i64), ("send_counts", C.POINTER(i64)), ("send_idx", C.POINTER(i64)),
                ("recv_counts", C.POINTER(i64)), ("recv_idx", C.POINTER(i64)), ("n_send", i64),
                ("n_recv", i64)]


class cad_run(C.Structure):
    _fields_ = [("src_row", i64), ("dst_row", i64), ("n_rows", i64)]


class cad_tick_work(C.Structure):
    _fields_ = [("active", i32), ("backward", i32), ("microbatch", i64)]


class cad_layer_cfg(C.Structure):
    _fields_ = [("rank", i32), ("world", i32), ("h_q", i32), ("h_kv", i32), ("head_dim", i32),
                ("softmax_scale", f32), ("transport", i32), ("layers", i32), ("balance_halves", i32),
                ("reserve_sms", i32), ("pad_", i32 * 2)]


class cad_layer_ctx_info(C.Structure):
    _fields_ = [("home_rows", i64), ("q_rows", i64 * 2), ("kv_rows", i64 * 2), ("n_tasks", i64 * 2),
                ("served_pairs", i64), ("wire_bytes", (i64 * 4) * 2), ("blob_bytes", i64),
                ("launches", i64)]


class cad_trace_rec(C.Structure):
    _fields_ = [("kind", i32), ("layer", i32), ("half", i32), ("pad_", i32), ("t_begin", f32),
                ("t_ready", f32), ("t_end", f32), ("pad2_", f32)]


class cad_layer_io(C.Structure):
    _fields_ = [("q", C.c_void_p), ("k", C.c_void_p), ("v", C.c_void_p), ("dout", C.c_void_p),
                ("o", C.c_void_p), ("lse", C.c_void_p), ("dq", C.c_void_p), ("dk", C.c_void_p),
                ("dv", C.c_void_p), ("dk_acc", C.c_void_p), ("dv_acc", C.c_void_p)]


P = C.POINTER
vp = C.c_void_p

# name -> (restype, argtypes); every declaration of include/cad.h.
SIGNATURES = {
    "cad_last_error": (C.c_char_p, []),
    "cad_version": (C.c_char_p, []),
    "cad_sched_cfg_default": (None, [P(cad_sched_cfg)]),
    "cad_length_dist_default": (None, [P(cad_length_dist)]),
    "cad_validate_item": (C.c_int, [P(cad_item)]),
    "cad_ca_flops_core": (C.c_int, [P(cad_item), P(i64)]),
    "cad_causal_pairs": (i64, [i64, i64]),
    "cad_item_bytes": (C.c_int, [P(cad_item), P(cad_sched_cfg), P(i64)]),
    "cad_sample_batch": (C.c_int, [P(cad_length_dist), i64, P(i64), i64, P(i64)]),
    "cad_place_sequential": (C.c_int, [P(i64), i64, i64, i64, P(cad_item), i64, P(i64)]),
    "cad_target_load": (C.c_int, [P(cad_item), i64, i64, f64, P(f64)]),
    "cad_classify_servers": (C.c_int, [P(f64), i64, f64, P(i32), P(f64), P(i64), P(i32), P(f64), P(i64)]),
    "cad_one_tile_slack": (C.c_int, [P(cad_item), i64, P(cad_sched_cfg), P(f64)]),
    "cad_v_min_comm": (C.c_int, [P(cad_comm_query), i64, P(cad_shard_choice)]),
    "cad_propose_migration": (C.c_int, [P(cad_server_load), P(cad_server_load), P(cad_item), f64,
                                        P(cad_sched_cfg), P(cad_proposal), P(i32)]),
    "cad_schedule": (C.c_int, [P(cad_item), i64, i64, P(cad_sched_cfg), P(vp)]),
    "cad_schedule_pp_tick": (C.c_int, [P(cad_item), P(i32), i64, i64, i64, P(cad_sched_cfg), P(vp)]),
    "cad_plan_get_stats": (C.c_int, [vp, P(cad_plan_stats)]),
    "cad_plan_tasks": (C.c_int, [vp, P(P(cad_task)), P(i64)]),
    "cad_plan_server": (C.c_int, [vp, i64, P(cad_server_load), P(P(cad_item))]),
    "cad_plan_to_text": (C.c_int, [vp, C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    "cad_plan_free": (None, [vp]),
    "cad_device_plan": (C.c_int, [vp, i32, P(cad_served_task), i64, P(i64), P(cad_served_task), i64, P(i64)]),
    "cad_ca_plan_create": (C.c_int, [P(cad_ca_task), i64, P(cad_ca_shape), P(vp)]),
    "cad_ca_plan_info_get": (C.c_int, [vp, P(cad_ca_plan_info)]),
    "cad_ca_plan_destroy": (C.c_int, [vp]),
    "cad_ca_fwd": (C.c_int, [vp, vp, vp, vp, vp, vp, vp]),  # plan q k v o lse stream
    "cad_ca_bwd": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp]),
    "cad_ca_bwd_parts": (C.c_int, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, C.c_int, vp]),
    "cad_ca_plan_set_max_ctas": (C.c_int, [vp, C.c_int]),
    "cad_layer_plan_create": (C.c_int, [vp, P(cad_item), i64, i32, i64, i64, P(vp)]),
    "cad_layer_plan_create_ex": (C.c_int, [vp, P(cad_item), i64, i32, i64, i64, i32, P(vp)]),
    "cad_layer_plan_info": (C.c_int, [vp, i32, P(cad_layer_half_info)]),
    "cad_layer_plan_xfer": (C.c_int, [vp, i32, i32, P(cad_xfer)]),
    "cad_layer_plan_destroy": (None, [vp]),
    "cad_scatter_add_bf16": (C.c_int, [vp, vp, i64, i64, vp, vp]),
    "cad_gather_cols_f32": (C.c_int, [vp, i64, i32, vp, i64, vp, vp]),
    "cad_scatter_cols_f32": (C.c_int, [vp, vp, i64, i32, vp, i64, vp]),
    "cad_f32_to_bf16": (C.c_int, [vp, i64, vp, vp]),
    "cad_ipc_handle": (C.c_int, [vp, P(u8), P(i64)]),
    "cad_ipc_open": (C.c_int, [P(u8), P(vp)]),
    "cad_ipc_close": (C.c_int, [vp]),
    "cad_copy_runs": (C.c_int, [vp, i64, vp, vp, i64, vp]),
    "cad_copy_spans": (C.c_int, [vp, i64, i32, vp]),
    "cad_copy_runs_cols": (C.c_int, [vp, i64, vp, i64, vp, i64, i32, vp]),
    "cad_stream_write_u32": (C.c_int, [vp, C.c_uint32, vp]),
    "cad_stream_wait_u32": (C.c_int, [vp, C.c_uint32, vp]),
    "cad_comm_unique_id": (C.c_int, [P(u8)]),
    "cad_comm_init": (C.c_int, [P(u8), i32, i32, P(vp)]),
    "cad_comm_destroy": (C.c_int, [vp]),
    "cad_gather_rows": (C.c_int, [vp, vp, i64, i64, vp, vp]),
    "cad_scatter_rows": (C.c_int, [vp, vp, i64, i64, vp, vp]),
    "cad_alltoallv": (C.c_int, [vp, vp, P(i64), P(i64), vp, P(i64), P(i64), vp]),
    "cad_layer_ctx_create": (C.c_int, [vp, P(cad_item), i64, P(cad_layer_cfg), P(vp)]),
    "cad_layer_ctx_info_get": (C.c_int, [vp, P(cad_layer_ctx_info)]),
    "cad_layer_ctx_bind_outputs": (C.c_int, [vp, vp, vp, vp]),
    "cad_layer_ctx_home": (C.c_int, [vp, i32, P(cad_layer_io)]),
    "cad_layer_ctx_export": (C.c_int, [vp, vp, C.c_size_t, P(C.c_size_t)]),
    "cad_layer_ctx_connect": (C.c_int, [vp, vp, C.c_size_t]),
    "cad_layer_ctx_set_comm": (C.c_int, [vp, vp]),
    "cad_layer_ctx_destroy": (C.c_int, [vp]),
    "cad_layer_begin": (C.c_int, [vp, vp]),
    "cad_layer_begin_ex": (C.c_int, [vp, i32, vp]),
    "cad_layer_step_ex": (C.c_int, [vp, P(cad_layer_io), i32, i32, vp]),
    "cad_pp_tick_table": (C.c_int, [i64, i64, i32, P(cad_tick_work), i64, P(i64)]),
    "cad_dispatch": (C.c_int, [vp, i32, i32, i32, P(cad_layer_io), vp]),
    "cad_dispatch_ex": (C.c_int, [vp, i32, i32, i32, P(cad_layer_io), vp, vp]),
    "cad_layer_compute": (C.c_int, [vp, i32, i32, i32, vp]),
    "cad_return": (C.c_int, [vp, i32, i32, i32, P(cad_layer_io), vp]),
    "cad_layer_finish": (C.c_int, [vp, P(cad_layer_io), vp]),
    "cad_layer_step": (C.c_int, [vp, P(cad_layer_io), i32, vp]),
    "cad_layer_ctx_set_trace": (C.c_int, [vp, i32]),
    "cad_layer_ctx_trace": (C.c_int, [vp, P(cad_trace_rec), i64, P(i64)]),
}

_lib = None
_lock = threading.Lock()


class CadError(RuntimeError):
    """A non-zero status from libcad; .code is the CAD_ERR_* value."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ConfigError(CadError):
    pass


class DomainError(CadError):
    pass


def lib() -> C.CDLL:
    """Load libcad.so once. Raises if the native library is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {_HERE}` "
                                  "(there is no non-native fallback)")
            h = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(h, name, None)
                if fn is None:
                    continue
                fn.restype = res
                fn.argtypes = args
            _lib = h
    return _lib


def check(rc: int) -> None:
    if rc == CAD_OK:
        return
    msg = lib().cad_last_error().decode()
    if rc == CAD_ERR_CONFIG:
        raise ConfigError(rc, msg)
    if rc == CAD_ERR_DOMAIN:
        raise DomainError(rc, msg)
    raise CadError(rc, msg)
