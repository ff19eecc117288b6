"""ctypes binding of ``libdear.so`` (the C ABI declared in include/dear.h).

There is no fallback: if the native library is missing or fails to load,
importing the runtime raises. Build it with ``python -m
paper_2302_12445_b200.build`` (``__graft_entry__.build()`` does this).
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# DEAR_LIB selects an alternative in-tree build (kernel-variant experiments).
LIB_PATH = os.path.join(PKG, os.environ.get("DEAR_LIB", "libdear.so"))

DEAR_OK, DEAR_EINVAL, DEAR_EINTERNAL = 0, 1, 2
POLICIES = {"WFBP": 0, "WFBP_FUSED": 1, "PRIORITY_PARTITION": 2, "DEAR": 3, "DEAR_FUSED": 4}


class DearError(RuntimeError):
    """A non-zero return from the C ABI (code 1 = invalid argument, 2 = CUDA/NCCL)."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidArgument(DearError, ValueError):
    pass


class DearCfg(C.Structure):
    _fields_ = [
        ("policy", C.c_int32),
        ("fusion_buffer_bytes", C.c_int64),
        ("dear_group_dependency", C.c_int32),
        ("lr", C.c_double),
        ("momentum", C.c_double),
        ("dampening", C.c_double),
        ("weight_decay", C.c_double),
        ("nesterov", C.c_int32),
        ("defer_allgather", C.c_int32),
        ("partition_bytes", C.c_int64),
    ]


_P = C.c_void_p
_SIGNATURES = {
    "dear_plan_build": [C.POINTER(C.c_int64), C.c_int32, C.c_int64, C.POINTER(C.c_int32),
                        C.POINTER(C.c_int32), C.POINTER(C.c_int32)],
    "dear_chunk_layout": [C.c_int64, C.c_int32, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "dear_comm_unique_id": [C.c_char_p],
    "dear_comm_init": [C.POINTER(_P), C.c_int32, C.c_char_p, C.c_int32],
    "dear_comm_destroy": [_P],
    "dear_local_group_create": [C.c_int32, C.POINTER(_P)],
    "dear_local_group_destroy": [_P],
    "dear_local_group_create_ex": [C.c_int32, C.c_int32, C.POINTER(_P)],
    "dear_local_group_connect": [_P, C.c_int32],
    "dear_create": [_P, C.c_int32, C.c_int32, _P, C.POINTER(DearCfg), C.POINTER(_P)],
    "dear_create_local": [_P, C.c_int32, _P, C.POINTER(DearCfg), C.POINTER(_P)],
    "dear_register_tensor": [_P, C.c_int32, _P, _P, C.c_int64],
    "dear_register_shadow": [_P, C.c_int32, _P],
    "dear_finalize": [_P],
    "dear_grad_ready": [_P, C.c_int32, _P],
    "dear_param_wait": [_P, C.c_int32, _P],
    "dear_step": [_P, _P],
    "dear_set_comm_order": [_P, C.POINTER(C.c_int32), C.c_int32],
    "dear_join": [_P, _P],
    "dear_synchronize": [_P],
    "dear_destroy": [_P],
    "dear_set_lr": [_P, C.c_double],
    "dear_num_buckets": [_P, C.POINTER(C.c_int32)],
    "dear_bucket_info": [_P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                         C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
    "dear_trace": [_P, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)],
    "dear_set_timing": [_P, C.c_int32],
    "dear_get_timings": [_P, C.POINTER(C.c_float), C.c_int32],
    "dear_check_replicas": [_P, C.POINTER(C.c_int32)],
    "dear_peer_handle": [_P, C.c_char_p],
    "dear_get_timeline": [_P, _P, C.POINTER(C.c_float), C.c_int32],
    "dear_peer_connect": [_P, C.c_char_p, C.c_int32],
    "dear_peer_zero_copy": [_P, C.POINTER(C.c_int32)],
    "dear_bench_stage": [_P, C.c_int32, C.c_int32, _P],
    "dear_nvls_supported": [C.c_int32, C.POINTER(C.c_int32)],
    "dear_symm_create": [C.c_int32, C.c_int32, C.c_int64, C.POINTER(_P), C.POINTER(C.c_int64),
                         C.POINTER(C.c_int64)],
    "dear_symm_join": [_P, C.c_int64, C.c_int64],
    "dear_symm_bind": [_P],
    "dear_symm_ptr": [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(C.c_int64)],
    "dear_symm_destroy": [_P],
    "dear_nvls_connect": [_P, _P],
    "dear_nvls_enabled": [_P, C.POINTER(C.c_int32)],
    "dear_comm_error": [_P, C.POINTER(C.c_int32)],
    "dear_set_comm_trace": [_P, C.c_int64],
    "dear_comm_trace_count": [C.POINTER(C.c_int64)],
}
DEAR_PEER_HANDLE_BYTES = 256

_lib = None


def lib() -> C.CDLL:
    """Load libdear.so once (RTLD_GLOBAL so its NCCL resolves to the one torch loaded)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the native DeAR runtime with "
                "`python -m paper_2302_12445_b200.build` (there is no CPU fallback)")
        try:
            import torch  # noqa: F401  (load torch's libnccl/libcudart first)
        except ImportError:
            pass
        L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, argtypes in _SIGNATURES.items():
            f = getattr(L, name)
            f.argtypes = argtypes
            f.restype = C.c_int
        L.dear_last_error.restype = C.c_char_p
        L.dear_last_error.argtypes = []
        L.dear_slot_stride.restype = C.c_int64
        L.dear_slot_stride.argtypes = [C.c_int64, C.c_int32]
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != DEAR_OK:
        msg = lib().dear_last_error().decode(errors="replace")
        if rc == DEAR_EINVAL:
            raise InvalidArgument(rc, msg)
        raise DearError(rc, msg)


GEMM_SYMBOLS = ["dear_gemm_plan_create", "dear_gemm_run", "dear_gemm_run_group",
                "dear_gemm_plan_info", "dear_gemm_plan_cluster", "dear_gemm_plan_pair",
                "dear_gemm_plan_set_flags", "dear_gemm_plan_set_tile", "dear_gemm_plan_set_splits",
                "dear_gemm_set_trace",
                "dear_gemm_plan_destroy"]  # bound in gemm.py


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES) + ["dear_last_error", "dear_slot_stride"] + GEMM_SYMBOLS
