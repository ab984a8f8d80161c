"""ctypes structs and signatures of the session entry points
(include/pipesim_b200.h, "pipeline session")."""
from __future__ import annotations

import ctypes as C


class pb_train_config(C.Structure):
    _fields_ = [("workers", C.c_int), ("micro_batches", C.c_int),
                ("mini_batch_size", C.c_int), ("mini_batches", C.c_int),
                ("learning_rate", C.c_double), ("mode", C.c_int), ("device", C.c_int),
                ("use_graph", C.c_int), ("snapshots", C.c_int),
                ("fwd_merge", C.c_int), ("timed_kernel", C.c_int),
                ("transport", C.c_int), ("precision", C.c_int),
                ("digests", C.c_int)]


class pb_epoch_out(C.Structure):
    _fields_ = [("mini_loss", C.POINTER(C.c_double)), ("pinned", C.POINTER(C.c_int)),
                ("consumed", C.POINTER(C.c_int)), ("dev_fwd", C.POINTER(C.c_int)),
                ("dev_bwd", C.POINTER(C.c_int)), ("dev_current", C.POINTER(C.c_int)),
                ("device_ms", C.c_float)]


class pb_epoch_profile(C.Structure):
    _fields_ = [("makespan_ms", C.c_float), ("stage_busy_ms", C.POINTER(C.c_float)),
                ("max_nodes", C.c_int), ("n_nodes", C.c_int),
                ("node_stage", C.POINTER(C.c_int)), ("node_fwd", C.POINTER(C.c_int)),
                ("node_mini", C.POINTER(C.c_int)), ("node_micro_lo", C.POINTER(C.c_int)),
                ("node_micro_hi", C.POINTER(C.c_int)), ("node_start_ms", C.POINTER(C.c_float)),
                ("node_end_ms", C.POINTER(C.c_float))]


class pb_session_info(C.Structure):
    _fields_ = [("horizon", C.c_int), ("units", C.c_int), ("kernels_per_epoch", C.c_int),
                ("device_bytes", C.c_int64), ("param_count", C.c_int64),
                ("pool_sizes", C.POINTER(C.c_int)), ("act_slots", C.POINTER(C.c_int)),
                ("stage_first_layer", C.POINTER(C.c_int)),
                ("stage_layers", C.POINTER(C.c_int))]


class pb_layer_spec(C.Structure):
    _fields_ = [("kind", C.c_int), ("in_", C.c_int), ("out", C.c_int), ("height", C.c_int),
                ("width", C.c_int), ("pool", C.c_int), ("act", C.c_int)]


class pb_layer_net(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("layers", C.POINTER(pb_layer_spec)),
                ("loss", C.c_int), ("stage_layers", C.POINTER(C.c_int))]


def signatures():
    from ._native import pb_net_spec
    i, p, i64, u64 = C.c_int, C.c_void_p, C.c_int64, C.c_uint64
    P = C.POINTER
    return {
        "pb_session_create": (i, [P(pb_net_spec), P(pb_train_config), P(p)]),
        "pb_session_destroy": (i, [p]),
        "pb_session_create_layers": (i, [P(pb_layer_net), P(pb_train_config), i, i, C.c_char_p,
                                         C.c_size_t, P(p)]),
        "pb_partition_layers": (i, [P(pb_layer_net), i, P(i), P(i)]),
        "pb_session_info_get": (i, [p, P(pb_session_info)]),
        "pb_session_load_params": (i, [p, P(C.c_double), i64]),
        "pb_session_load_stage_params": (i, [p, i, P(C.c_double), i64]),
        "pb_session_read_params": (i, [p, P(C.c_double), i64]),
        "pb_session_upload": (i, [p, p, i, p, i]),
        "pb_session_run_epoch": (i, [p, P(pb_epoch_out)]),
        "pb_session_train_epoch": (i, [p, p, i, p, i, P(pb_epoch_out)]),
        "pb_session_profile_epoch": (i, [p, P(pb_epoch_out), P(pb_epoch_profile)]),
        "pb_session_kernel_times": (i, [p, P(C.c_float), P(C.c_double), i, P(i)]),
        "pb_session_trace_document": (i, [p, C.c_char_p, i64, P(i64)]),
        "pb_session_snapshot": (i, [p, i, i, P(C.c_double), i64]),
        "pb_session_read_version": (i, [p, i, i, P(C.c_double), i64]),
        "pb_nccl_unique_id": (i, [C.c_char_p]),
        "pb_session_ipc_export": (i, [p, C.c_char_p, i64, P(i64)]),
        "pb_session_ipc_connect": (i, [p, C.c_char_p, P(i64), i]),
        "pb_session_create_dist": (i, [P(pb_net_spec), P(pb_train_config), i, i, C.c_char_p,
                                       C.c_size_t, P(p)]),
        "pb_plan_transfers": (i, [P(pb_net_spec), P(pb_train_config), i, i, P(i), P(i), P(i),
                                  P(i), P(i64), i]),
        "pb_device_digest_f32": (i, [P(C.c_float), i64, C.c_char_p, P(C.c_float)]),
        "pb_device_format_f32": (i, [P(C.c_float), i64, C.c_char_p]),
        "pb_session_digests": (i, [p, C.c_char_p, i64]),
        "pb_session_params_digest": (i, [p, i, C.c_char_p]),
        "pb_plan_memory": (i, [P(pb_net_spec), P(pb_train_config), i, i, P(i64), P(i64), P(i),
                               P(i)]),
        "pb_make_classification_task": (i, [i, i, i, u64, P(C.c_double), P(C.c_float),
                                            P(C.c_int)]),
    }
