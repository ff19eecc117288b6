"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/*.h declares; argument validation that needs no GPU behaves."""
import ctypes as C
import glob
import os
import re

import pytest

from paper_2302_12445_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names |= set(re.findall(r"\b(dear_[a-z0-9_]+)\s*\(", src))
    return names


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _declared()
    assert len(declared) >= 25
    missing = [n for n in sorted(declared) if not hasattr(L, n)]
    assert not missing, missing
    # and the Python binding knows the signature of each of them
    assert set(_lib.exported_symbols()) == declared


def test_dynamic_symbol_table():
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    exported = set(re.findall(r" T (dear_\w+)", out))
    assert _declared() <= exported


def test_sm100a_cubin_embedded():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_invalid_arguments_without_gpu():
    L = _lib.lib()
    assert L.dear_plan_build(None, 0, 0, None, None, None) == _lib.DEAR_EINVAL
    assert L.dear_chunk_layout(5, 0, None, None) == _lib.DEAR_EINVAL
    assert "workers must be >= 1" in L.dear_last_error().decode()
    assert L.dear_finalize(None) == _lib.DEAR_EINVAL
    assert L.dear_slot_stride(-1, 2) == -1
    cfg = _lib.DearCfg(1, 0, 0, 0.1, 0, 0, 0, 0, 0)  # WFBP_FUSED without a buffer
    ctx = C.c_void_p()
    assert L.dear_create(None, 0, 1, None, C.byref(cfg), C.byref(ctx)) == _lib.DEAR_EINVAL
    assert "requires fusion_buffer_bytes > 0" in L.dear_last_error().decode()
    cfg = _lib.DearCfg(2, 1, 0, 0.1, 0, 0, 0, 0, 0, 0)  # PRIORITY_PARTITION without parts
    assert L.dear_create(None, 0, 1, None, C.byref(cfg), C.byref(ctx)) == _lib.DEAR_EINVAL
    assert "PRIORITY_PARTITION requires partition_bytes > 0" in L.dear_last_error().decode()
    cfg = _lib.DearCfg(3, 0, 0, 0.1, 0, 0, 0, 0, 0)
    assert L.dear_create(None, 0, 2, None, C.byref(cfg), C.byref(ctx)) == _lib.DEAR_EINVAL
    assert "NCCL communicator is required" in L.dear_last_error().decode()
    # zero-copy query and the bench hook validate their context first
    on = C.c_int32(7)
    assert L.dear_peer_zero_copy(None, C.byref(on)) == _lib.DEAR_EINVAL
    assert L.dear_bench_stage(None, 0, 1, None) == _lib.DEAR_EINVAL
    assert L.dear_peer_connect(None, None, 0) == _lib.DEAR_EINVAL


def test_runtime_rejects_unknown_policy():
    from paper_2302_12445_b200 import Runtime

    with pytest.raises(ValueError, match="unknown policy"):
        Runtime(policy="BYTESCHEDULER")


def test_python_transport_validation_without_gpu():
    """Host-side argument checks of the transports (no CUDA call is made)."""
    import paper_2302_12445_b200 as dear

    with pytest.raises(ValueError, match="transport"):
        dear.LocalGroup(2, "bogus")
    with pytest.raises(ValueError, match="needs a SymmetricHeap"):
        dear.Runtime(None, 0, 1, backend="nvls")
    with pytest.raises(ValueError, match="backend must be"):
        dear.Runtime(None, 0, 1, backend="gloo")
    L = _lib.lib()
    # PRIORITY_PARTITION is a runtime policy now (validated like policy.cpp:58-61)
    cfg = _lib.DearCfg(2, 0, 0, 0.1, 0, 0, 0, 0, 0, -5)
    ctx = C.c_void_p()
    assert L.dear_create(None, 0, 1, None, C.byref(cfg), C.byref(ctx)) == _lib.DEAR_EINVAL
    # local-group / heap entry points validate their handles first
    assert L.dear_local_group_connect(None, 1) == _lib.DEAR_EINVAL
    assert L.dear_nvls_connect(None, None) == _lib.DEAR_EINVAL
    assert L.dear_symm_join(None, 0, 0) == _lib.DEAR_EINVAL
    assert L.dear_symm_bind(None) == _lib.DEAR_EINVAL
    g = C.c_void_p()
    assert L.dear_local_group_create_ex(2, 7, C.byref(g)) == _lib.DEAR_EINVAL
    assert L.dear_local_group_create_ex(17, 1, C.byref(g)) == _lib.DEAR_EINVAL
