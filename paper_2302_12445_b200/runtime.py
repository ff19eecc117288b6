"""Python face of the native DeAR runtime (one context per GPU / rank).

This is a thin object wrapper over the C ABI in ``include/dear.h``; every
call goes to ``libdear.so`` and errors surface as :class:`DearError`
(``ValueError`` subclass for invalid arguments). Reference counterparts:

==========================  ===============================================
``Runtime.register``        LayerSpec / ModelSpec (model.hpp:26-45)
``Runtime.finalize``        build_fusion_plan / per_layer_plan (fusion.cpp)
``Runtime.grad_ready``      RS_g <- BP of g's layers (task_graph.cpp:148-194)
``Runtime.step``            BARRIER + AG issue (task_graph.cpp:195-206)
``Runtime.param_wait``      FF_l <- AG_g(l) (task_graph.cpp:207)
``Runtime.check_replicas``  "replica divergence" check (collective.cpp:172)
==========================  ===============================================
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import torch

from ._lib import DEAR_PEER_HANDLE_BYTES, POLICIES, DearCfg, DearError, check, lib


def _dist_ready() -> bool:
    import torch.distributed as dist

    return dist.is_available() and dist.is_initialized()


def _stream_ptr(stream: Optional[torch.cuda.Stream]) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class Communicator:
    """An NCCL communicator (one rank per process / GPU) over NVLink/NVSwitch."""

    def __init__(self, rank: int, world_size: int, unique_id: bytes):
        if len(unique_id) != 128:
            raise ValueError("NCCL unique id must be 128 bytes")
        self.rank, self.world_size = rank, world_size
        self._comm = C.c_void_p()
        check(lib().dear_comm_init(C.byref(self._comm), world_size, unique_id, rank))

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().dear_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def from_torch_distributed(cls, group=None) -> "Communicator":
        """Bootstrap over an initialised torch.distributed group (any backend):
        rank 0 creates the NCCL id, every rank receives it via broadcast."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        return cls(rank, world, obj[0])

    @property
    def handle(self) -> int:
        return self._comm.value or 0

    def close(self) -> None:
        if self._comm.value:
            check(lib().dear_comm_destroy(self._comm))
            self._comm = C.c_void_p()


class LocalGroup:
    """P ranks in one process on one device.

    ``transport="ring"``: ring-order collective kernels over all ranks'
    buffers (the reference's ring rounds, collective.cpp:59-152). Drive the P
    contexts in lock-step: every rank makes the same sequence of calls, and
    all ranks finish an iteration's ``step`` before any rank starts the next
    forward.

    ``transport="peer"``: the multi-GPU NVLink peer kernels (zero-copy or slot
    reduce-scatter + update, all-gather) against each other's memory on the
    one device — the N > 1 data path on one GPU. Each collective runs as one
    cooperative launch over every rank's data once all ranks reached it (same
    lock-step rule). Call :meth:`connect` after every rank's ``finalize``."""

    TRANSPORTS = {"ring": 0, "peer": 1}

    def __init__(self, P: int, transport: str = "ring"):
        if transport not in self.TRANSPORTS:
            raise ValueError("transport must be 'ring' or 'peer'")
        self.P = P
        self.transport = transport
        self._g = C.c_void_p()
        check(lib().dear_local_group_create_ex(P, self.TRANSPORTS[transport], C.byref(self._g)))

    def connect(self, zero_copy: bool = True) -> None:
        """Peer transport: map the ranks onto each other (dear_local_group_connect)."""
        check(lib().dear_local_group_connect(self._g, int(zero_copy)))

    @property
    def handle(self) -> int:
        return self._g.value

    def close(self) -> None:
        if self._g.value:
            check(lib().dear_local_group_destroy(self._g))
            self._g = C.c_void_p()


def nvls_supported(device: Optional[int] = None) -> bool:
    """The GPU supports NVLink SHARP multicast objects (NVSwitch systems)."""
    ok = C.c_int32(0)
    dev = torch.cuda.current_device() if device is None else device
    check(lib().dear_nvls_supported(dev, C.byref(ok)))
    return bool(ok.value)


class _CudaBuffer:
    """__cuda_array_interface__ view of raw device bytes (kept alive by the heap)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


class SymmetricHeap:
    """Device memory mapped on every rank through one NVLS multicast object
    (dear_symm_*). Collective over torch.distributed (or a single rank
    without it). ``tensor()`` carves 256-byte aligned tensors in call order —
    identical offsets on every rank when every rank makes the same calls."""

    def __init__(self, nbytes: int, rank: Optional[int] = None, world_size: Optional[int] = None):
        dist_on = _dist_ready()
        if dist_on:
            import torch.distributed as dist

            rank, world_size = dist.get_rank(), dist.get_world_size()
        rank = 0 if rank is None else rank
        world_size = 1 if world_size is None else world_size
        self.rank, self.world_size = rank, world_size
        self._h = C.c_void_p()
        pid, fd = C.c_int64(-1), C.c_int64(-1)
        check(lib().dear_symm_create(rank, world_size, int(nbytes), C.byref(self._h),
                                     C.byref(pid), C.byref(fd)))
        pair = [(pid.value, fd.value)]
        if dist_on and world_size > 1:
            import torch.distributed as dist

            dist.broadcast_object_list(pair, 0)
        check(lib().dear_symm_join(self._h, pair[0][0], pair[0][1]))
        if dist_on and world_size > 1:
            torch.distributed.barrier()  # every GPU added before any memory is bound
        check(lib().dear_symm_bind(self._h))
        if dist_on and world_size > 1:
            torch.distributed.barrier()
        loc, mc, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        check(lib().dear_symm_ptr(self._h, C.byref(loc), C.byref(mc), C.byref(n)))
        self.local, self.multicast, self.nbytes = loc.value, mc.value, n.value
        self._bytes = torch.as_tensor(_CudaBuffer(self.local, self.nbytes), device="cuda")
        self._cursor = 0

    @property
    def handle(self) -> int:
        return self._h.value

    def tensor(self, numel: int, dtype=torch.float32) -> torch.Tensor:
        esz = torch.empty((), dtype=dtype).element_size()
        nb = max(int(numel), 1) * esz
        at = (self._cursor + 255) // 256 * 256
        if at + nb > self.nbytes:
            raise MemoryError(f"symmetric heap exhausted ({at + nb} > {self.nbytes} bytes)")
        self._cursor = at + nb
        return self._bytes[at:at + nb].view(dtype)[:numel]

    def close(self) -> None:
        if self._h.value:
            if _dist_ready() and self.world_size > 1:
                torch.cuda.synchronize()
                torch.distributed.barrier()
            self._bytes = None
            check(lib().dear_symm_destroy(self._h))
            self._h = C.c_void_p()


class Runtime:
    """One DeAR context: registered tensors, fusion buckets, comm stream."""

    def __init__(self, comm=None, rank: int = 0, world_size: int = 1, *,
                 policy: str = "DEAR_FUSED", fusion_buffer_bytes: int = 25_000_000,
                 lr: float = 0.05, momentum: float = 0.0, dampening: float = 0.0,
                 weight_decay: float = 0.0, nesterov: bool = False,
                 dear_group_dependency: bool = False, defer_allgather: bool = False,
                 backend: str = "auto", stream: Optional[torch.cuda.Stream] = None,
                 heap: Optional[SymmetricHeap] = None, partition_bytes: int = 0):
        if policy not in POLICIES:
            raise ValueError(f"unknown policy kind {policy!r}; expected one of "
                             f"{', '.join(POLICIES)}")
        if backend not in ("auto", "nccl", "peer", "nvls"):
            raise ValueError("backend must be 'auto', 'nccl', 'peer' or 'nvls'")
        if backend == "nvls" and heap is None:
            raise ValueError("the nvls backend needs a SymmetricHeap holding the tensors")
        if heap is not None and backend == "auto":
            backend = "nvls"
        if isinstance(comm, LocalGroup):
            # A local group's transport decides the collectives: "local" (the
            # ring-order emulation kernels) or "peer" (the NVLink peer kernels).
            if comm.transport == "peer":
                if backend == "nccl":
                    raise ValueError("a LocalGroup(transport='peer') runs the peer kernels")
                backend = "peer"
            else:
                if backend == "peer":
                    raise ValueError("use LocalGroup(P, transport='peer') for the peer kernels "
                                     "on one device")
                backend = "local"
        elif backend == "auto":
            # The NVLink peer path (fused RS+update / AG+unpack kernels) when
            # several processes share torch.distributed; NCCL otherwise.
            backend = "peer" if (isinstance(comm, Communicator) and comm.world_size > 1
                                 and _dist_ready()) else "nccl"
        self.policy = policy
        self.backend = backend
        self._group = comm if isinstance(comm, LocalGroup) else None
        self._comm_obj = comm if isinstance(comm, Communicator) else None
        self._heap = heap
        cfg = DearCfg(POLICIES[policy], int(fusion_buffer_bytes) if "FUSED" in policy else 0,
                      int(dear_group_dependency), float(lr),
                      float(momentum), float(dampening), float(weight_decay), int(nesterov),
                      int(defer_allgather), int(partition_bytes))
        self._ctx = C.c_void_p()
        sp = _stream_ptr(stream)
        if isinstance(comm, LocalGroup):
            self.rank, self.world_size = rank, comm.P
            check(lib().dear_create_local(comm.handle, rank, sp, C.byref(cfg),
                                          C.byref(self._ctx)))
        else:
            if isinstance(comm, Communicator):
                rank, world_size, handle = comm.rank, comm.world_size, comm.handle
            else:
                handle = 0
            self.rank, self.world_size = rank, world_size
            check(lib().dear_create(handle or None, rank, world_size, sp, C.byref(cfg),
                                    C.byref(self._ctx)))
        self._keep = []  # tensors whose storage the runtime points at

    # -- registration ----------------------------------------------------
    def register(self, layer: int, param: torch.Tensor, grad: torch.Tensor,
                 shadow: Optional[torch.Tensor] = None) -> None:
        for name, t in (("param", param), ("grad", grad)):
            if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} of layer {layer} must be a contiguous CUDA fp32 tensor")
        if param.numel() != grad.numel():
            raise ValueError(f"param/grad size mismatch for layer {layer}")
        check(lib().dear_register_tensor(self._ctx, layer, param.data_ptr(), grad.data_ptr(),
                                         param.numel()))
        self._keep += [param, grad]
        if shadow is not None:
            if shadow.dtype != torch.bfloat16 or shadow.numel() < param.numel():
                raise ValueError(f"shadow of layer {layer} must be bf16 with >= numel elements")
            check(lib().dear_register_shadow(self._ctx, layer, shadow.data_ptr()))
            self._keep.append(shadow)

    def finalize(self) -> None:
        check(lib().dear_finalize(self._ctx))
        if self.backend == "nvls":
            check(lib().dear_nvls_connect(self._ctx, self._heap.handle))
        elif self.backend == "peer" and self.world_size > 1 and self._group is None:
            self._connect_peers()

    @property
    def zero_copy(self) -> bool:
        """The peer backend took the zero-copy path (dear_peer_zero_copy)."""
        if not self._ctx.value:
            return False
        on = C.c_int32()
        check(lib().dear_peer_zero_copy(self._ctx, C.byref(on)))
        return bool(on.value)

    @property
    def push_rs(self) -> bool:
        """The zero-copy path runs the push reduce-scatter (DEAR_PUSH_RS=1)."""
        if not self._ctx.value:
            return False
        on = C.c_int32()
        check(lib().dear_peer_zero_copy(self._ctx, C.byref(on)))
        return on.value == 2

    def _connect_peers(self) -> None:
        """Exchange arena IPC handles over torch.distributed and map the peers."""
        import torch.distributed as dist

        buf = C.create_string_buffer(DEAR_PEER_HANDLE_BYTES)
        check(lib().dear_peer_handle(self._ctx, buf))
        handles = [None] * self.world_size
        dist.all_gather_object(handles, buf.raw)
        check(lib().dear_peer_connect(self._ctx, b"".join(handles), self.world_size))
        dist.barrier()

    # -- schedule hooks ----------------------------------------------------
    def grad_ready(self, layer: int, stream=None) -> None:
        check(lib().dear_grad_ready(self._ctx, layer, _stream_ptr(stream)))

    def param_wait(self, layer: int, stream=None) -> None:
        check(lib().dear_param_wait(self._ctx, layer, _stream_ptr(stream)))

    def step(self, stream=None) -> None:
        check(lib().dear_step(self._ctx, _stream_ptr(stream)))

    def set_comm_order(self, seq) -> None:
        """Comm-stream dispatch sequence (dear_set_comm_order). DEAR with
        dear_group_dependency: +g = RS of bucket g, -g = AG of bucket g, 1-based
        plan order. PRIORITY_PARTITION: every part g once, in dispatch order.
        [] restores the default."""
        seq = [int(v) for v in seq]
        arr = (C.c_int32 * max(1, len(seq)))(*seq)
        check(lib().dear_set_comm_order(self._ctx, arr, len(seq)))

    def join(self, stream=None) -> None:
        check(lib().dear_join(self._ctx, _stream_ptr(stream)))

    def synchronize(self) -> None:
        try:
            check(lib().dear_synchronize(self._ctx))
        except DearError as e:
            if "communicator aborted" in str(e) and self._comm_obj is not None:
                self._comm_obj._comm = C.c_void_p()  # freed by ncclCommAbort
            raise

    def comm_failed(self) -> bool:
        """The NCCL communicator reported an asynchronous error (dear_comm_error)."""
        bad = C.c_int32(0)
        check(lib().dear_comm_error(self._ctx, C.byref(bad)))
        return bool(bad.value)

    def set_lr(self, lr: float) -> None:
        check(lib().dear_set_lr(self._ctx, float(lr)))

    # -- introspection -------------------------------------------------------
    def buckets(self) -> list[dict]:
        n = C.c_int32(0)
        check(lib().dear_num_buckets(self._ctx, C.byref(n)))
        out = []
        for g in range(n.value):
            lo, hi, d, s = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64()
            check(lib().dear_bucket_info(self._ctx, g, C.byref(lo), C.byref(hi), C.byref(d),
                                         C.byref(s)))
            out.append({"low": lo.value, "high": hi.value, "elems": d.value,
                        "slot_stride": s.value})
        return out

    def trace(self) -> list[str]:
        need = C.c_int64(0)
        check(lib().dear_trace(self._ctx, None, 0, C.byref(need)))
        buf = C.create_string_buffer(int(need.value))
        check(lib().dear_trace(self._ctx, buf, need.value, C.byref(need)))
        return [x for x in buf.value.decode().split("\n") if x]

    def bench_stage(self, stage: str, reps: int = 1, stream=None) -> None:
        """Measurement hook (dear_bench_stage): `reps` rounds of one bucket
        kernel over every bucket, outside the schedule (graph-capturable)."""
        k = {"pack": 0, "update": 1, "unpack": 2, "direct": 3}[stage]
        check(lib().dear_bench_stage(self._ctx, k, int(reps), _stream_ptr(stream)))

    def set_timing(self, enable: bool) -> None:
        check(lib().dear_set_timing(self._ctx, int(enable)))

    def timings(self) -> list[dict]:
        """Per bucket (plan order) milliseconds of pack/rs/update/ag/unpack; None
        where the stage did not run in the last timed iteration."""
        n = len(self.buckets())
        arr = (C.c_float * (5 * n))()
        check(lib().dear_get_timings(self._ctx, arr, n))
        keys = ("pack", "rs", "update", "ag", "unpack")
        return [{k: (arr[5 * g + i] if arr[5 * g + i] >= 0 else None)
                 for i, k in enumerate(keys)} for g in range(n)]

    STAMPS = ("pack0", "pack1", "rs1", "update1", "ag0", "ag1", "unpack1")

    def timeline(self, base_event: "torch.cuda.Event") -> list[dict]:
        """Per bucket: ms from `base_event` to each comm-stream stamp of the last
        timed iteration (None where the stage did not run)."""
        n = len(self.buckets())
        arr = (C.c_float * (7 * n))()
        check(lib().dear_get_timeline(self._ctx, C.c_void_p(base_event.cuda_event), arr, n))
        return [{k: (arr[7 * g + i] if arr[7 * g + i] >= 0 else None)
                 for i, k in enumerate(self.STAMPS)} for g in range(n)]

    def check_replicas(self) -> bool:
        ok = C.c_int32(0)
        check(lib().dear_check_replicas(self._ctx, C.byref(ok)))
        return bool(ok.value)

    def close(self) -> None:
        """Destroy the context. On the multi-process peer backend this is
        collective: peers may still read this rank's arena / tensors through
        their mappings, so every rank drains its comm stream and meets the
        others at a barrier before any unmaps or frees."""
        if self._ctx.value:
            if self.backend in ("peer", "nvls") and self.world_size > 1 \
                    and self._group is None and _dist_ready():
                import torch.distributed as dist

                check(lib().dear_synchronize(self._ctx))
                dist.barrier()
            check(lib().dear_destroy(self._ctx))
            self._ctx = C.c_void_p()
            self._keep = []

    def __del__(self):
        # Best effort at interpreter teardown (no barrier: peers may be gone).
        try:
            if self._ctx.value:
                check(lib().dear_destroy(self._ctx))
                self._ctx = C.c_void_p()
        except Exception:
            pass
