"""B200-native DeAR: decoupled all-reduce (reduce-scatter -> shard update ->
all-gather) with per-bucket forward gating, over NCCL on NVLink/NVSwitch.

Public API
----------
* :func:`init`, :class:`DistOptim`            — PyTorch integration
* :class:`Runtime`, :class:`Communicator`,
  :class:`LocalGroup`                          — the native runtime (include/dear.h)
* :func:`build_fusion_plan`, :func:`chunk_ranges`,
  :func:`chunk_owner`                          — host partitioner / layout (bit-exact
                                                 with proj/src/fusion.cpp, collective.cpp)
"""
from ._lib import DearError, InvalidArgument
from .optim import DistOptim, init
from .plan import build_fusion_plan, chunk_owner, chunk_ranges, slot_chunk, slot_stride
from .runtime import Communicator, LocalGroup, Runtime, SymmetricHeap, nvls_supported

__all__ = [
    "DearError", "InvalidArgument", "DistOptim", "init", "build_fusion_plan", "chunk_owner",
    "chunk_ranges", "slot_chunk", "slot_stride", "Communicator", "LocalGroup", "Runtime",
    "SymmetricHeap", "nvls_supported",
]
