"""ctypes binding of librnnwave_sm100.so (include/rnnwave_sm100.h).

There is no fallback: if the library is missing or fails to load, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

_F = C.POINTER(C.c_float)
_PF = C.POINTER(_F)

RW_OK, RW_EINVAL, RW_ECUDA, RW_ENOMEM, RW_ENCCL, RW_ESTATE = range(6)
RW_PREC_BF16, RW_PREC_FP32 = 0, 1
RW_SCHED_AUTO, RW_SCHED_STEPWISE, RW_SCHED_PERSISTENT, RW_SCHED_CLUSTER, RW_SCHED_LAYERSEQ = 0, 1, 2, 3, 4
RW_TAPE_X0, RW_TAPE_H, RW_TAPE_C, RW_TAPE_GATES, RW_TAPE_TANH_C, RW_TAPE_DGW, RW_TAPE_Y, RW_TAPE_ZRH, RW_TAPE_DGR = range(9)

class rw_trace_record(C.Structure):
    _fields_ = [("task_id", C.c_int32), ("layer", C.c_int32), ("block", C.c_int32), ("step_k", C.c_int32),
                ("phase", C.c_int32), ("worker", C.c_int32), ("start_ns", C.c_int64), ("end_ns", C.c_int64)]


# every symbol include/rnnwave_sm100.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "rw_create", "rw_destroy", "rw_last_error", "rw_create_error", "rw_set_params", "rw_forward",
    "rw_backward_data", "rw_weight_update", "rw_get_tape", "rw_upload_inputs", "rw_run_pass",
    "rw_sync", "rw_set_profiling", "rw_read_outputs", "rw_launch_count", "rw_params_updated",
    "rw_nccl_unique_id", "rw_comm_init", "rw_allreduce_grads", "rw_comm_overlap", "rw_phase_times", "rw_describe", "rw_describe_variants",
    "rw_describe_precision", "rw_flop_count_cell",
    "rw_test_gemm", "rw_test_gemm_last_ms", "rw_pp_export", "rw_pp_link", "rw_pp_set_next_w",
    "rw_train_step", "rw_train_wait", "rw_trace_enable", "rw_trace_records", "rw_gemm", "rw_ladder_pass",
    "rw_pointwise_forward", "rw_pointwise_backward",
]


class rw_config(C.Structure):
    _fields_ = [("layers", C.c_int), ("hidden", C.c_int), ("input", C.c_int), ("batch", C.c_int),
                ("steps", C.c_int), ("cell_kind", C.c_int), ("opt_level", C.c_int),
                ("batch_steps", C.c_int), ("workers", C.c_int), ("seed", C.c_uint64),
                ("precision", C.c_int), ("schedule", C.c_int)]


class rw_pp_ring(C.Structure):
    _fields_ = [("handle", (C.c_char * 64) * 5), ("offset", C.c_uint64 * 5), ("ptr", C.c_uint64 * 5),
                ("pid", C.c_int64), ("device", C.c_int), ("ko", C.c_int),
                ("mode", C.c_int)]


_lib = None


def lib_path() -> str:
    return _build.LIB


def _nccl_hint() -> None:
    """Point the library's lazy NCCL dlopen at the NCCL PyTorch links (the nvidia-nccl wheel), so
    both share one libnccl.so.2 in a process (runtime.cu nccl())."""
    if os.environ.get("RW_NCCL_PATH"):
        return
    try:
        import importlib.util
        spec = importlib.util.find_spec("nvidia.nccl")
        for d in (spec.submodule_search_locations or []) if spec else []:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                os.environ["RW_NCCL_PATH"] = p
                return
    except (ImportError, ValueError):
        pass


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building first if needed and possible) the sm_100a library."""
    global _lib
    _nccl_hint()
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path) or not _build.up_to_date():
        if not build_if_missing:
            raise FileNotFoundError(f"{path} is missing: run __graft_entry__.build()")
        _build.build()
    L = C.CDLL(path)
    vp = C.c_void_p
    L.rw_create.argtypes = [C.POINTER(rw_config), C.c_int, C.POINTER(vp)]
    L.rw_destroy.argtypes = [vp]
    L.rw_destroy.restype = None
    L.rw_last_error.argtypes = [vp]
    L.rw_last_error.restype = C.c_char_p
    L.rw_create_error.argtypes = []
    L.rw_create_error.restype = C.c_char_p
    L.rw_set_params.argtypes = [vp, C.c_int, _F, _F, _F]
    L.rw_forward.argtypes = [vp, _F, C.c_int, _PF, _PF, _F, C.POINTER(C.c_uint64)]
    L.rw_backward_data.argtypes = [vp, C.c_uint64, _F, _F, _PF, _PF]
    L.rw_weight_update.argtypes = [vp, C.c_uint64, _PF, _PF, _PF]
    L.rw_get_tape.argtypes = [vp, C.c_int, C.c_int, _F]
    L.rw_upload_inputs.argtypes = [vp, _F, _F]
    L.rw_run_pass.argtypes = [vp, C.c_int, vp]
    L.rw_sync.argtypes = [vp]
    L.rw_set_profiling.argtypes = [vp, C.c_int]
    L.rw_phase_times.argtypes = [vp, C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_int, C.c_int]
    L.rw_describe.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                              C.POINTER(C.c_int)]
    L.rw_describe_variants.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.rw_describe_precision.argtypes = [vp, C.POINTER(C.c_int)]
    L.rw_read_outputs.argtypes = [vp, _F, _F, _PF, _PF, _PF]
    L.rw_launch_count.argtypes = [vp, C.POINTER(C.c_longlong), C.c_int]
    L.rw_params_updated.argtypes = [vp]
    L.rw_nccl_unique_id.argtypes = [C.c_char_p]
    L.rw_comm_init.argtypes = [vp, C.c_int, C.c_int, C.c_char_p]
    L.rw_allreduce_grads.argtypes = [vp, vp]
    L.rw_comm_overlap.argtypes = [vp, C.c_int]
    L.rw_flop_count_cell.argtypes = [C.c_int, C.c_int, C.c_int]
    L.rw_flop_count_cell.restype = C.c_int64
    L.rw_test_gemm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp,
                               C.c_longlong, vp, C.c_longlong, vp, C.c_longlong, C.c_int]
    L.rw_pp_export.argtypes = [vp, C.c_int, C.POINTER(rw_pp_ring)]
    L.rw_pp_link.argtypes = [vp, C.c_int, C.POINTER(rw_pp_ring), _F]
    L.rw_pp_set_next_w.argtypes = [vp, _F]
    L.rw_pp_debug.argtypes = [vp, C.POINTER(C.c_longlong)]
    L.rw_train_step.argtypes = [vp, _F, _F, _F, _F, _PF, _PF, _PF]
    L.rw_train_wait.argtypes = [vp]
    L.rw_trace_enable.argtypes = [vp, C.c_int]
    L.rw_ladder_pass.argtypes = [vp, C.c_int, vp]
    L.rw_gemm.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, _F, C.c_longlong, _F,
                          C.c_longlong, C.c_float, _F, C.c_longlong]
    L.rw_pointwise_forward.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int] + [_F] * 10
    L.rw_pointwise_backward.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int] + [_F] * 13
    L.rw_trace_records.argtypes = [vp, C.c_int, C.POINTER(rw_trace_record), C.c_int, C.POINTER(C.c_int)]
    L.rw_test_gemm_last_ms.argtypes = []
    L.rw_test_gemm_last_ms.restype = C.c_float
    _lib = L
    return L
