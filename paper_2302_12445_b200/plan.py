"""Host partitioner and shard layout (pure host; calls the native library).

Mirrors the reference's value-type API:
  * :func:`build_fusion_plan` <- ``build_fusion_plan`` / ``per_layer_plan``
    (proj/src/fusion.cpp:29-70)
  * :func:`chunk_ranges`      <- ``chunk_ranges`` (proj/src/collective.cpp:39-57)
  * :func:`chunk_owner`       <- owner ``(c - 1) mod P`` (collective.cpp:94)
"""
from __future__ import annotations

import ctypes as C

from ._lib import check, lib


def build_fusion_plan(layer_bytes, buffer_bytes: int) -> list[tuple[int, int]]:
    """Groups ``(low_layer, high_layer)`` in backprop issue order.

    ``layer_bytes[0]`` is layer 1; ``buffer_bytes == 0`` gives the per-layer
    plan. Raises ``ValueError`` with the reference's messages (e.g.
    ``"build_fusion_plan: empty model"``).
    """
    L = len(layer_bytes)
    arr = (C.c_int64 * max(L, 1))(*[int(x) for x in layer_bytes])
    lo = (C.c_int32 * max(L, 1))()
    hi = (C.c_int32 * max(L, 1))()
    n = C.c_int32(0)
    check(lib().dear_plan_build(arr, L, int(buffer_bytes), lo, hi, C.byref(n)))
    return [(lo[g], hi[g]) for g in range(n.value)]


def chunk_ranges(d: int, P: int) -> list[tuple[int, int]]:
    """``[begin, end)`` of chunk c for c = 0..P-1; the first ``d % P`` are one longer."""
    b = (C.c_int64 * (P + 1))() if P >= 1 else None
    s = C.c_int64(0)
    check(lib().dear_chunk_layout(int(d), int(P), b, C.byref(s)))
    return [(b[c], b[c + 1]) for c in range(P)]


def chunk_owner(c: int, P: int) -> int:
    """Rank holding chunk c fully reduced after reduce-scatter: (c - 1) mod P."""
    return (c - 1) % P


def slot_chunk(r: int, P: int) -> int:
    """Chunk carried by NCCL slot r (rank r's shard): (r + 1) mod P."""
    return (r + 1) % P


def slot_stride(d: int, P: int) -> int:
    """Elements between rank slots in a bucket buffer (ceil(d/P) -> multiple of 64)."""
    v = lib().dear_slot_stride(int(d), int(P))
    if v < 0:
        raise ValueError("slot_stride: need d >= 0 and P >= 1")
    return v
