"""ctypes binding of the C ABI in ``include/pipesim_b200.h``.

The shared library is built in-tree (``paper_2410_14312_b200/lib``) by
``make`` / ``__graft_entry__.build()``.  There is no fallback: if the library
is missing, importing the package's compute entry points raises.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

_HERE = pathlib.Path(__file__).resolve().parent
# PIPESIM_LIB: an alternative build of the same library (A/B experiments,
# tools/gpu/build_variants.sh); the default is the in-tree build
LIB_PATH = pathlib.Path(os.environ["PIPESIM_LIB"]) if os.environ.get("PIPESIM_LIB") else \
    _HERE / "lib" / "libpipesim_b200.so"


class PipesimError(RuntimeError):
    """Base class; mirrors std::runtime_error of the reference."""


class DomainError(PipesimError):
    """pipesim::domain_error (proj/include/pipesim/errors.hpp:25-35)."""

    def __init__(self, message: str, field: str = ""):
        super().__init__(message)
        self.field = field


class StructuralError(PipesimError):
    """pipesim::structural_error (errors.hpp:37-42)."""


class InsufficientHorizonError(PipesimError):
    """pipesim::insufficient_horizon_error (errors.hpp:44-48)."""


class IntegrityError(PipesimError):
    """pipesim::integrity_error (errors.hpp:50-59)."""

    def __init__(self, message: str, stage_id: int = 0, epoch: int = 0):
        super().__init__(message)
        self.stage_id = stage_id
        self.epoch = epoch


class IoError(PipesimError):
    """pipesim::io_error (errors.hpp:61-65)."""


class CudaError(PipesimError):
    pass


class CapacityError(PipesimError):
    pass


PB_OK = 0


class pb_sim_config(C.Structure):
    _fields_ = [("workers", C.c_int), ("micro_batches", C.c_int),
                ("mini_batches", C.c_int), ("backward_cost_factor", C.c_double),
                ("samples_per_mini_batch", C.c_int), ("seed", C.c_uint64)]


class pb_task(C.Structure):
    _fields_ = [("kind", C.c_int), ("mini", C.c_int), ("micro", C.c_int)]


class pb_commit(C.Structure):
    _fields_ = [("version", C.c_int), ("mini", C.c_int), ("stage", C.c_int),
                ("slot", C.c_int)]


class pb_pin(C.Structure):
    _fields_ = [("mini", C.c_int), ("micro", C.c_int), ("slot", C.c_int),
                ("version", C.c_int)]


class pb_consume(C.Structure):
    _fields_ = [("mini", C.c_int), ("stage", C.c_int), ("slot", C.c_int),
                ("version", C.c_int)]


class pb_interval(C.Structure):
    _fields_ = [("version", C.c_int), ("from_slot", C.c_int),
                ("freed_slot", C.c_int)]


class pb_restored_stage(C.Structure):
    _fields_ = [("stage_id", C.c_int), ("first_layer", C.c_int), ("n_layers", C.c_int),
                ("version", C.c_int), ("loss", C.c_int), ("epoch", C.c_int),
                ("n_values", C.c_int64)]


class pb_net_spec(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("widths", C.POINTER(C.c_int)),
                ("activations", C.POINTER(C.c_int)), ("loss", C.c_int)]


_lib = None


def lib() -> C.CDLL:
    """Load the native library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `make -C "
                f"{_HERE}` or __graft_entry__.build(); there is no CPU fallback")
        _lib = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        _declare(_lib)
    return _lib


def _declare(L: C.CDLL) -> None:
    i, p, d, f, u64, i64 = C.c_int, C.c_void_p, C.c_double, C.c_float, C.c_uint64, C.c_int64
    P = C.POINTER
    sig = {
        "pb_last_error": (i, [C.c_char_p, i]),
        "pb_last_error_field": (i, [C.c_char_p, i]),
        "pb_last_error_stage_epoch": (i, [P(i), P(i)]),
        "pb_version": (C.c_char_p, []),
        "pb_validate_config": (i, [P(pb_sim_config)]),
        "pb_schedule_build": (i, [P(pb_sim_config), i, P(i), P(pb_task), i]),
        "pb_schedule_document": (i, [P(pb_sim_config), i, C.c_char_p, C.c_int64,
                                     P(C.c_int64)]),
        "pb_schedule_validate": (i, [P(pb_sim_config), i, P(pb_task), i, P(i), P(i), i,
                                     C.c_char_p, i]),
        "pb_assign_versions": (i, [P(pb_sim_config), i, P(pb_task), i, P(pb_commit),
                                   P(pb_pin), P(pb_consume), P(i), P(i)]),
        "pb_measure_version_difference": (i, [P(pb_sim_config), P(i), i, P(i)]),
        "pb_closed_form_v": (i, [i, i, P(i)]),
        "pb_forward_span": (i, [i, i, i, P(i)]),
        "pb_backward_span": (i, [i, P(i)]),
        "pb_overlap_condition": (i, [i, i, P(i)]),
        "pb_decompose_sequences": (i, [P(pb_sim_config), P(i), i, P(i), P(i), P(i), P(i)]),
        "pb_retention_timeline": (i, [P(pb_sim_config), i, P(pb_task), i, P(pb_pin),
                                      P(pb_interval), P(i)]),
        "pb_staleness": (i, [P(pb_sim_config), P(pb_commit), P(pb_consume), P(i)]),
        "pb_partition_model": (i, [P(pb_net_spec), i, P(i), P(i)]),
        "pb_param_count": (i64, [P(pb_net_spec)]),
        "pb_init_network_params": (i, [P(pb_net_spec), u64, P(d), i64]),
        "pb_make_synthetic_task": (i, [i, u64, P(d), P(d)]),
        "pb_params_digest": (i, [P(d), i64, C.c_char_p]),
        "pb_checkpoint_stage": (i, [i, i, i, P(i), i, P(d), i64, i, i, C.c_char_p]),
        "pb_restore_stage": (i, [C.c_char_p, i, i, P(pb_restored_stage), P(i), i, P(d), i64]),
        "pb_device_count": (i, [P(i)]),
        "pb_set_device": (i, [i]),
        "pb_synchronize": (i, []),
        "pb_linear_fwd": (i, [p, p, i, i, i, p, i, i, p, i, p, i, p, i]),
        "pb_linear_bwd_dx": (i, [p, p, i, i, i, p, i, i, p, i, i, p, i]),
        "pb_linear_bwd_dw_sgd": (i, [p, p, i, i, i, p, i, i, p, p, i, p, i, f]),
        "pb_linear_bwd_dw_sgd_split": (i, [p, p, i, i, i, p, i, i, p, p, p, p, i, f]),
        "pb_split_master": (i, [p, p, i, i, i, p, p, i]),
        "pb_join_master": (i, [p, p, p, i, i, i, p, i]),
        "pb_bias_sgd": (i, [p, p, i, i, i, p, p, p, f]),
        "pb_loss_fwd_bwd": (i, [p, p, i, i, i, p, i, i, i, f, p, i, p]),
        "pb_conv_fwd": (i, [p, p, i, i, i, i, p, i, i, p, i, p]),
        "pb_conv_bwd_dx": (i, [p, p, i, i, i, i, p, i, i, p, i, p]),
        "pb_conv_bwd_dw_sgd": (i, [p, p, i, i, i, i, p, i, p, p, i, p, i, f]),
        "pb_maxpool2_fwd": (i, [p, p, i, i, i, i, p]),
        "pb_maxpool2_bwd": (i, [p, p, p, p, i, i, i, i, p]),
        "pb_im2col_first": (i, [p, p, i, i, i, i, i, p, i]),
        "pb_convert_f64_to_bf16": (i, [p, p, i, i, i, p, i]),
        "pb_convert_f32_to_bf16": (i, [p, p, i, i, i, p, i]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    for name, (res, args) in _late_signatures().items():
        if hasattr(L, name):
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args


def _late_signatures():
    from . import _session_abi  # session entry points, declared next to their structs
    return _session_abi.signatures()


def last_error() -> str:
    buf = C.create_string_buffer(4096)
    lib().pb_last_error(buf, 4096)
    return buf.value.decode(errors="replace")


def check(status: int) -> None:
    """Raise the Python mirror of the reference exception for a status."""
    if status == PB_OK:
        return
    msg = last_error()
    L = lib()
    if status == 1:
        buf = C.create_string_buffer(256)
        L.pb_last_error_field(buf, 256)
        raise DomainError(msg, buf.value.decode())
    if status == 2:
        raise StructuralError(msg)
    if status == 3:
        raise InsufficientHorizonError(msg)
    if status == 4:
        st, ep = C.c_int(), C.c_int()
        L.pb_last_error_stage_epoch(C.byref(st), C.byref(ep))
        raise IntegrityError(msg, st.value, ep.value)
    if status == 5:
        raise IoError(msg)
    if status == 6:
        raise CudaError(msg)
    if status == 7:
        raise CapacityError(msg)
    if status == 8:
        raise ValueError(msg)
    raise PipesimError(msg)


EXPORTED_SYMBOLS = None  # filled by tests from include/pipesim_b200.h
