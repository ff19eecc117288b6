"""Python binding of the sm_100a tcgen05/TMA GEMM (include/dear_gemm.h).

Used for the synthetic per-layer compute (feed-forward, data-gradient and
weight-gradient contractions) that the DeAR collectives overlap with. No
fallback: the plan calls the native kernel or raises.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

from ._lib import check, lib

_bound = False


def _bind():
    global _bound
    if _bound:
        return lib()
    L = lib()
    P = C.c_void_p
    L.dear_gemm_plan_create.argtypes = [P, C.c_int64, P, C.c_int64, C.c_int32, P, C.c_int64,
                                        C.c_int32, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_int32, C.c_int32, C.POINTER(P)]
    L.dear_gemm_run.argtypes = [P, P]
    L.dear_gemm_run_group.argtypes = [C.POINTER(P), C.c_int32, P]
    L.dear_gemm_plan_info.argtypes = [P] + [C.POINTER(C.c_int32)] * 4
    L.dear_gemm_plan_destroy.argtypes = [P]
    L.dear_gemm_plan_cluster.argtypes = [P] + [C.POINTER(C.c_int32)] * 3
    L.dear_gemm_plan_pair.argtypes = [P, C.POINTER(C.c_int32)]
    L.dear_gemm_plan_set_flags.argtypes = [P, C.c_int32]
    L.dear_gemm_plan_set_tile.argtypes = [P, C.c_int32, C.c_int32]
    L.dear_gemm_plan_set_splits.argtypes = [P, C.c_int32]
    L.dear_gemm_set_trace.argtypes = [P]
    for f in ("dear_gemm_plan_create", "dear_gemm_run", "dear_gemm_run_group",
              "dear_gemm_plan_info", "dear_gemm_plan_cluster", "dear_gemm_plan_pair",
              "dear_gemm_plan_set_flags", "dear_gemm_plan_set_tile", "dear_gemm_plan_set_splits",
              "dear_gemm_set_trace",
              "dear_gemm_plan_destroy"):
        getattr(L, f).restype = C.c_int
    _bound = True
    return L


def set_trace(buf: "torch.Tensor | None") -> None:
    """Profiling: per-CTA %globaltimer phase stamps of every later launch go to
    `buf` (int64 CUDA tensor, >= 8 x 148 entries); None disables."""
    check(_bind().dear_gemm_set_trace(buf.data_ptr() if buf is not None else None))


class GemmPlan:
    """D[M,N] (+)= A[M,K] @ B^T, bf16 inputs, fp32 accumulation.

    a: [M, K] bf16 (K contiguous). b: [N, K] bf16 (``b_mn_major=False``) or
    [K, N] bf16 (``b_mn_major=True``). d: [M, ldd] fp32 / bf16 view or a flat
    tensor (``d_limit`` = number of valid flat elements, for partial rows).
    ``early_operands=True`` asserts that A and B are not written by any kernel
    that may still run when this GEMM starts (DEAR_GEMM_EARLY_OPERANDS): the
    operand stream then starts under the preceding kernel's tail.
    """

    def __init__(self, a: torch.Tensor, b: torch.Tensor, d: torch.Tensor, M: int, N: int,
                 K: int, *, b_mn_major: bool = False, lda: int | None = None,
                 ldb: int | None = None, ldd: int | None = None, d_limit: int = -1,
                 accumulate: bool = False, split_k: int = 0, early_operands: bool = False):
        L = _bind()
        for t in (a, b):
            if t.dtype != torch.bfloat16 or not t.is_cuda:
                raise ValueError("GEMM operands must be CUDA bf16 tensors")
        if d.dtype not in (torch.float32, torch.bfloat16):
            raise ValueError("D must be fp32 or bf16")
        lda = lda if lda is not None else a.stride(0)
        ldb = ldb if ldb is not None else b.stride(0)
        ldd = ldd if ldd is not None else (d.stride(0) if d.dim() == 2 else N)
        self._keep = (a, b, d)
        self._plan = C.c_void_p()
        check(L.dear_gemm_plan_create(a.data_ptr(), lda, b.data_ptr(), ldb, int(b_mn_major),
                                      d.data_ptr(), ldd, int(d.dtype == torch.float32), M, N,
                                      K, d_limit, int(accumulate), split_k,
                                      C.byref(self._plan)))
        self._flags = 1 if early_operands else 0
        if self._flags:
            check(L.dear_gemm_plan_set_flags(self._plan, self._flags))
        self.M, self.N, self.K = M, N, K

    def run(self, stream: torch.cuda.Stream | None = None) -> None:
        s = (stream or torch.cuda.current_stream()).cuda_stream
        check(_bind().dear_gemm_run(self._plan, s))

    def info(self) -> dict:
        v = [C.c_int32() for _ in range(4)]
        check(_bind().dear_gemm_plan_info(self._plan, *[C.byref(x) for x in v]))
        out = dict(zip(("bn", "n_tiles", "m_tiles", "splits"), (x.value for x in v)))
        c = [C.c_int32() for _ in range(3)]
        check(_bind().dear_gemm_plan_cluster(self._plan, *[C.byref(x) for x in c]))
        out.update(zip(("cm", "cn", "resident_clusters"), (x.value for x in c)))
        pr = C.c_int32()
        check(_bind().dear_gemm_plan_pair(self._plan, C.byref(pr)))
        out["pair"] = pr.value
        return out

    @property
    def flops(self) -> int:
        return 2 * self.M * self.N * self.K

    def set_tile(self, bn: int, pair: bool) -> None:
        """Override the cost model's tile choice (dear_gemm_plan_set_tile)."""
        check(_bind().dear_gemm_plan_set_tile(self._plan, int(bn), int(bool(pair))))

    def set_red_add(self, on: bool) -> None:
        """fp32 accumulate via per-thread red.add (True) or TMA reduce (False)."""
        self._flags = (self._flags & ~2) | (2 if on else 0)
        check(_bind().dear_gemm_plan_set_flags(self._plan, self._flags))

    def set_splits(self, split_k: int) -> None:
        """Override the split-K count of an accumulating plan."""
        check(_bind().dear_gemm_plan_set_splits(self._plan, int(split_k)))

    @staticmethod
    def run_group(plans: "list[GemmPlan]", stream: torch.cuda.Stream | None = None) -> None:
        """One persistent launch computing up to two independent plans."""
        s = (stream or torch.cuda.current_stream()).cuda_stream
        arr = (C.c_void_p * len(plans))(*[p._plan.value for p in plans])
        check(_bind().dear_gemm_run_group(arr, len(plans), s))

    def close(self) -> None:
        if self._plan.value:
            check(_bind().dear_gemm_plan_destroy(self._plan))
            self._plan = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# Plan-time autotuning of the tile configuration.
#
# The cost model inside dear_gemm_plan_create assumes isolated launches; in a
# chain of early-operand launches the next GEMM streams its operands under the
# previous one's tail, which favours fewer, wider tiles (profiles/r01_gemm_tiles.md).
# The chain is measured instead: each candidate (bn, pair) is timed as a
# CUDA-graph-captured run of back-to-back launches, once per distinct shape,
# outside any timed region.

def tile_candidates(M: int, N: int, mn_major: bool) -> list[tuple[int, int]]:
    # DEAR_GEMM_MAX_BN: for library builds with narrower TMEM accumulators
    # (DEAR_GEMM_BN_MAX, e.g. three CTAs per SM at BN <= 128).
    max_bn = int(os.environ.get("DEAR_GEMM_MAX_BN", "256"))
    out = []
    for pair in (0, 1):
        if pair and M <= 128:
            continue
        for bn in range(64, max_bn + 1, 16):
            if pair and mn_major and bn not in (128, 256):
                continue
            nt = -(-N // bn)
            if nt > 1 and (nt - 1) * bn >= N:  # a fully padded last tile
                continue
            out.append((bn, pair))
    return out


def time_chain(launch, n: int, stream: torch.cuda.Stream, reps: int = 3) -> float:
    """Device µs per call of launch(i), i = 0..n-1 captured in one CUDA graph."""
    with torch.cuda.stream(stream):
        for i in range(2):
            launch(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(n):
            launch(i)
    with torch.cuda.stream(stream):
        g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
    torch.cuda.synchronize()
    del g
    return e0.elapsed_time(e1) * 1e3 / (reps * n)


def autotune(plans: "list[GemmPlan]", candidates, n: int = 16,
             stream: torch.cuda.Stream | None = None) -> list[tuple[float, int, int]]:
    """Time a chain of `plans` (same shape, outputs that may be clobbered) for
    every (bn, pair) candidate; leaves the best one set and returns
    [(µs per launch, bn, pair)] sorted."""
    stream = stream or torch.cuda.Stream()
    res = []
    for bn, pair in candidates:
        for p in plans:
            p.set_tile(bn, pair)
        us = time_chain(lambda i: plans[i % len(plans)].run(stream), n, stream)
        res.append((us, bn, pair))
    res.sort()
    for p in plans:
        p.set_tile(res[0][1], res[0][2])
    return res


def autotune_group(first: "list[GemmPlan]", second: "list[GemmPlan]", top_first, top_second,
                   n: int = 16, stream: torch.cuda.Stream | None = None):
    """Joint choice for grouped launches (run_group([first[i], second[i]])) among
    the given per-plan candidates; leaves the best pair of configs set."""
    stream = stream or torch.cuda.Stream()
    res = []
    for c0 in top_first:
        for c1 in top_second:
            for p in first:
                p.set_tile(*c0)
            for p in second:
                p.set_tile(*c1)
            us = time_chain(lambda i: GemmPlan.run_group(
                [first[i % len(first)], second[i % len(second)]], stream), n, stream)
            res.append((us, c0, c1))
    res.sort(key=lambda r: r[0])
    for p in first:
        p.set_tile(*res[0][1])
    for p in second:
        p.set_tile(*res[0][2])
    return res
