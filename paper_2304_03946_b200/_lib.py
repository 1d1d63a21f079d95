"""ctypes binding of `libflexmoe_b200.so` (declared in include/flexmoe_b200.h).

The native library is the product; this module only loads it, declares the
C signatures and maps status codes onto exceptions that mirror the
reference's C++ exception classes. There is no fallback:
a missing library is an ImportError.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# FLEXMOE_B200_LIB: load another build of the same library (A/B measurements)
_LIB_PATH = Path(os.environ.get("FLEXMOE_B200_LIB") or Path(__file__).resolve().parent / "libflexmoe_b200.so")

FM_OK = 0
FM_ERR_INVALID_ARGUMENT = 1
FM_ERR_LOGIC = 2
FM_ERR_RUNTIME = 3
FM_ERR_OUT_OF_RANGE = 4
FM_ERR_CUDA = 5

FM_GEMM_FWD_BIAS_RELU = 0
FM_GEMM_FWD_BIAS = 1
FM_GEMM_DGRAD_RELU_MASK = 2
FM_GEMM_DGRAD = 3
FM_GEMM_WGRAD = 4


class FlexMoEError(RuntimeError):
    """Base class; `status` holds the C status code."""

    status = FM_ERR_RUNTIME


class InvalidArgument(FlexMoEError, ValueError):
    """std::invalid_argument in the reference."""

    status = FM_ERR_INVALID_ARGUMENT


class LogicError(FlexMoEError):
    """std::logic_error in the reference (broken invariant)."""

    status = FM_ERR_LOGIC


class OutOfRange(FlexMoEError, IndexError):
    """std::out_of_range in the reference."""

    status = FM_ERR_OUT_OF_RANGE


class CudaError(FlexMoEError):
    status = FM_ERR_CUDA


_ERRORS = {
    FM_ERR_INVALID_ARGUMENT: InvalidArgument,
    FM_ERR_LOGIC: LogicError,
    FM_ERR_RUNTIME: FlexMoEError,
    FM_ERR_OUT_OF_RANGE: OutOfRange,
    FM_ERR_CUDA: CudaError,
}

_P = C.c_void_p
_I = C.c_int
_I64P = C.POINTER(C.c_int64)
_I32P = C.POINTER(C.c_int32)
_DP = C.POINTER(C.c_double)

# name -> argtypes (all return int status unless listed in _RESTYPES)
_SIGNATURES = {
    "fm_route_counts": [_P, _P, _I, _I, _P],
    "fm_route_counts_device": [_P, _P, _I, _I, _P, _P, _P],
    "fm_received_matrix": [_P, _I, _I, _P],
    "fm_per_gpu_received": [_P, _I, _I, _P],
    "fm_balance_ratio": [_P, _I, _I, _DP],
    "fm_largest_remainder_round": [_P, _I, C.c_int64, _P],
    "fm_static_ep_kept": [_P, _I, _I, C.c_double, _P, _I64P],
    "fm_trace_save": [C.c_char_p, _P, _P, _I, _I, _I],
    "fm_trace_load": [C.c_char_p, _I, _I, _P, C.c_int64, _P, _P, _P],
    "fm_static_ep_kept_device": [_P, _I, _I, C.c_double, _P, _P, _P],
    "fm_layer_set_capacity_factor": [_P, C.c_double],
    "fm_grouped_gemm": [_I, _P, _P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P],
    "fm_set_gemm_cta_group": [_I],
    "fm_layer_create": [_P, _P, C.POINTER(_P)],
    "fm_layer_destroy": [_P],
    "fm_layer_set_placement": [_P, _P],
    "fm_layer_set_placement_async": [_P, _P, _P, _P],
    "fm_layer_set_operand_slots": [_P, _P, _I, _P],
    "fm_layer_local_experts": [_P, C.POINTER(_I), _P],
    "fm_layer_side_jobs": [_P, C.POINTER(_I)],
    "fm_layer_set_side_jobs": [_P, _I],
    "fm_layer_forward": [_P, _P, _I, _P, _P, _P, _P, _P, _P, _P],
    "fm_layer_backward": [_P] * 9,
    "fm_layer_copy_out": [_P, _I, _P, C.c_size_t, C.POINTER(C.c_size_t)],
    "fm_layer_copy_out_async": [_P, _I, _P, C.c_size_t, C.POINTER(C.c_size_t), _P],
    "fm_layer_set_timing": [_P, _I],
    "fm_profile_reference_default": [_I, _I, _P],
    "fm_step_cost": [_P, _P, _I, _P, _P, _P],
    "fm_make_scheduling_plan": [_P, _P, _I, _P, _I, _P, _I, _P],
    "fm_plan_migrations": [_P, _I, _P, _I, _P, _I, _P],
    "fm_placement_apply": [_P, _I, _P, _P, _P, _P],
    "fm_scheduler_create": [_P, _P, _I, _P],
    "fm_scheduler_destroy": [_P],
    "fm_scheduler_step": [_P, _P, _P],
    "fm_scheduler_begin_step": [_P, _P],
    "fm_scheduler_finish_step": [_P, _P, _P],
    "fm_scheduler_ops": [_P, _I, _P, _I, _P],
    "fm_scheduler_placement": [_P, _I, _P, _P],
    "fm_scheduler_reset": [_P, _P],
    "fm_scheduler_join_policy": [_P, _P],
    "fm_baseline_create": [_P, _P, _I, _P],
    "fm_baseline_destroy": [_P],
    "fm_baseline_step": [_P, _P, _P, _P, _P, _P],
    "fm_baseline_placement": [_P, _P, _P, _P],
    "fm_layer_gate": [_P, _P, _I, _P, _P, _P],
    "fm_layer_route": [_P, _P, _P, _P, _P],
    "fm_layer_dispatch": [_P, _P, _P, _P],
    "fm_layer_expert_forward": [_P] * 8,
    "fm_layer_combine": [_P] * 4,
    "fm_layer_combine_backward": [_P] * 5,
    "fm_layer_expert_backward": [_P] * 10,
    "fm_layer_unpermute_backward": [_P] * 7,
    "fm_layer_read_timing": [_P, _P, _P],
    "fm_layer_enable_p2p": [_P],
    "fm_layer_p2p_handle": [_P, _P],
    "fm_layer_p2p_open_peer": [_P, _I, _P],
    "fm_layer_p2p_link_peer": [_P, _I, _P],
    "fm_layer_p2p_status": [_P, _P],
    "fm_layer_route_p2p": [_P, _P, _P],
    "fm_layer_dispatch_p2p": [_P, _P, _P],
    "fm_layer_expert_forward_p2p": [_P] * 6,
    "fm_layer_combine_p2p": [_P, _P, _P],
    "fm_layer_combine_backward_p2p": [_P, _P, _P],
    "fm_layer_expert_backward_p2p": [_P] * 9,
    "fm_layer_unpermute_backward_p2p": [_P] * 5,
    "fm_layer_p2p_bind_dx": [_P] * 3,
    "fm_pool_create": [_I, _I, _I, _I, C.POINTER(_P)],
    "fm_pool_destroy": [_P],
    "fm_pool_info": [_P, _P, _P],
    "fm_pool_slot_ptr": [_P, _I, C.POINTER(_P)],
    "fm_pool_ipc_handle": [_P, _P],
    "fm_pool_open_peer": [_P, _I, _P],
    "fm_pool_link_peer": [_P, _I, _P],
    "fm_pool_migrate": [_P, _P, _I, _P, _I, _P, _P, _P, _P, _P],
    "fm_pool_set_operand_layout": [_P, _I],
    "fm_pool_wait_ready": [_P, _P],
    "fm_pool_pack": [_P, _P, _I, _P, _P, _P, _P, _P],
    "fm_pool_adam": [_P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P],
    "fm_pool_migration_stats": [_P, _P, _P, _P],
}
_RESTYPES = {"fm_last_error": C.c_char_p, "fm_version": C.c_char_p, "fm_kernel_launches": C.c_ulonglong}

_lib = None


def lib() -> C.CDLL:
    """Loads the native library (once). Raises ImportError if it was not built."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise ImportError(
                f"{_LIB_PATH} is missing: run `python -m paper_2304_03946_b200.build` "
                "(or __graft_entry__.build()); there is no fallback path"
            )
        handle = C.CDLL(str(_LIB_PATH))
        for name, res in _RESTYPES.items():
            if hasattr(handle, name):
                getattr(handle, name).restype = res
                getattr(handle, name).argtypes = []
        for name, args in _SIGNATURES.items():
            if hasattr(handle, name):
                fn = getattr(handle, name)
                fn.argtypes = args
                fn.restype = C.c_int
        _lib = handle
    return _lib


def release(destroy_fn: str, handle) -> None:
    """Calls `destroy_fn(handle)` unless the handle is empty or the library is
    already gone (interpreter shutdown clears module globals before __del__)."""
    lib_ = _lib
    if lib_ is None or handle is None or not handle.value:
        return
    getattr(lib_, destroy_fn)(handle)


def exported_symbols() -> list[str]:
    return sorted(set(_SIGNATURES) | set(_RESTYPES))


def check(status: int) -> None:
    if status != FM_OK:
        msg = lib().fm_last_error().decode(errors="replace")
        raise _ERRORS.get(status, FlexMoEError)(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))


def ptr(t) -> int | None:
    """Raw address of a torch tensor / numpy array (None for None)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def stream_ptr(stream=None) -> int | None:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream
