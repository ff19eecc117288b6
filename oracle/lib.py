"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the oracle libraries.

See ``oracle/__init__.py`` for who may import this.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATED_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdearsim_ref.so")
REF_SRC = "/root/reference/proj/src/collective.cpp"

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


def build(ref: bool | None = None) -> None:
    """Compile the restatement (and the reference build when its sources exist)."""
    target = ["all"] if ref is None else (["restate", "ref"] if ref else ["restate"])
    subprocess.run(["make", "-s", "-C", HERE, *target], check=True)


def have_reference_build() -> bool:
    return os.path.exists(REF_SO)


class Restated:
    """The plain-C restatement (oracle/dear_oracle.c)."""

    def __init__(self, path: str = RESTATED_SO):
        if not os.path.exists(path):
            build(ref=False)
        lib = C.CDLL(path)
        lib.or_random_vectors.argtypes = [C.c_int, C.c_int64, C.c_uint64, _f64p]
        lib.or_random_vectors_f32.argtypes = [C.c_int, C.c_int64, C.c_uint64, _f32p]
        lib.or_preset_params.argtypes = [C.c_char_p, C.c_int, _i64p, C.c_int]
        lib.or_build_fusion_plan.argtypes = [_i64p, C.c_int, C.c_int64, _i32p, _i32p]
        lib.or_chunk_ranges.argtypes = [C.c_int64, C.c_int, _i64p]
        lib.or_chunk_owner.argtypes = [C.c_int, C.c_int]
        lib.or_ring_reduce_scatter.argtypes = [C.c_int, C.c_int64, _f64p, _f64p]
        lib.or_all_reduce_average.argtypes = [C.c_int, C.c_int64, _f64p, _f64p]
        lib.or_sgd_step.argtypes = [C.c_int, C.c_int64, C.c_double, _f64p, _f64p]
        lib.or_sgd_step_momentum.argtypes = [
            C.c_int, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int,
            _f64p, _f64p, C.POINTER(C.c_int), _f64p]
        lib.or_ring_reduce_scatter_f32.argtypes = [C.c_int, C.c_int64, _f32p, _f32p]
        lib.or_sgd_step_f32.argtypes = [
            C.c_int, C.c_int64, C.c_float, C.c_float, C.c_float, C.c_float, C.c_int,
            _f32p, _f32p, C.POINTER(C.c_int), _f32p, C.c_int]
        self.lib = lib

    def random_vectors(self, P: int, d: int, seed: int) -> np.ndarray:
        out = np.empty(P * d, np.float64)
        self.lib.or_random_vectors(P, d, seed, out)
        return out.reshape(P, d)

    def random_vectors_f32(self, P: int, d: int, seed: int) -> np.ndarray:
        """random_vectors(P, d, seed).astype(float32) without the fp64 array."""
        out = np.empty(P * d, np.float32)
        self.lib.or_random_vectors_f32(P, d, seed, out)
        return out.reshape(P, d)

    def preset_params(self, name: str, profile: int = 0) -> np.ndarray:
        out = np.zeros(1024, np.int64)
        n = self.lib.or_preset_params(name.encode(), profile, out, 1024)
        if n < 0:
            raise ValueError(f"unknown preset {name!r}")
        return out[:n].copy()

    def build_fusion_plan(self, layer_bytes, buffer_bytes: int):
        lb = np.ascontiguousarray(layer_bytes, np.int64)
        lo = np.zeros(len(lb) + 1, np.int32)
        hi = np.zeros(len(lb) + 1, np.int32)
        n = self.lib.or_build_fusion_plan(lb, len(lb), buffer_bytes, lo, hi)
        if n < 0:
            raise ValueError("invalid fusion-plan input")
        return [(int(lo[g]), int(hi[g])) for g in range(n)]

    def chunk_ranges(self, d: int, P: int) -> np.ndarray:
        b = np.zeros(P + 1, np.int64)
        if self.lib.or_chunk_ranges(d, P, b) != 0:
            raise ValueError("invalid chunk_ranges input")
        return b

    def chunk_owner(self, c: int, P: int) -> int:
        return self.lib.or_chunk_owner(c, P)

    def ring_reduce_scatter(self, vecs: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(vecs, np.float64)
        out = np.empty(v.shape[1], np.float64)
        self.lib.or_ring_reduce_scatter(v.shape[0], v.shape[1], v.reshape(-1), out)
        return out

    def all_reduce_average(self, vecs: np.ndarray) -> np.ndarray:
        v = np.ascontiguousarray(vecs, np.float64)
        out = np.empty(v.shape[1], np.float64)
        self.lib.or_all_reduce_average(v.shape[0], v.shape[1], v.reshape(-1), out)
        return out

    def sgd_step(self, w: np.ndarray, grads: np.ndarray, lr: float) -> np.ndarray:
        w = np.array(w, np.float64, copy=True)
        g = np.ascontiguousarray(grads, np.float64)
        self.lib.or_sgd_step(g.shape[0], g.shape[1], lr, w, g.reshape(-1))
        return w

    def sgd_step_momentum(self, w, buf, has_buf: bool, grads, lr, momentum=0.0,
                          dampening=0.0, weight_decay=0.0, nesterov=False):
        w = np.array(w, np.float64, copy=True)
        buf = np.array(buf, np.float64, copy=True)
        hb = C.c_int(1 if has_buf else 0)
        g = np.ascontiguousarray(grads, np.float64)
        self.lib.or_sgd_step_momentum(g.shape[0], g.shape[1], lr, momentum, dampening,
                                      weight_decay, int(nesterov), w, buf, C.byref(hb),
                                      g.reshape(-1))
        return w, buf, bool(hb.value)

    def sgd_step_f32(self, w, buf, has_buf: bool, grads, lr, momentum=0.0, dampening=0.0,
                     weight_decay=0.0, nesterov=False, prescale=False):
        w = np.array(w, np.float32, copy=True)
        buf = np.array(buf, np.float32, copy=True)
        hb = C.c_int(1 if has_buf else 0)
        g = np.ascontiguousarray(grads, np.float32)
        self.lib.or_sgd_step_f32(g.shape[0], g.shape[1], lr, momentum, dampening,
                                 weight_decay, int(nesterov), w, buf, C.byref(hb),
                                 g.reshape(-1), int(prescale))
        return w, buf, bool(hb.value)


class Reference:
    """The reference's own code (oracle/_ref/libdearsim_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            if not os.path.exists(REF_SRC):
                raise FileNotFoundError(
                    "oracle/_ref is not built and /root/reference is absent")
            build(ref=True)
        lib = C.CDLL(path)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_preset_params.argtypes = [C.c_char_p, C.c_int, _i64p, C.c_int]
        lib.ref_build_plan.argtypes = [_i64p, C.c_int, C.c_int, C.c_int64, _i32p, _i32p]
        lib.ref_chunk_ranges.argtypes = [C.c_int64, C.c_int, _i64p, _i64p]
        lib.ref_random_vectors.argtypes = [C.c_int, C.c_int64, C.c_uint64, _f64p]
        lib.ref_ring_reduce_scatter.argtypes = [C.c_int, C.c_int64, _f64p, _f64p,
                                                C.POINTER(C.c_int)]
        lib.ref_all_reduce.argtypes = [C.c_int, C.c_int64, _f64p, _f64p, C.c_int]
        lib.ref_sgd_step.argtypes = [C.c_int, C.c_int64, C.c_double, _f64p, _f64p, _f64p]
        lib.ref_sgd_step_replicas.argtypes = [C.c_int, C.c_int64, C.c_double, _f64p, _f64p,
                                              _f64p]
        lib.ref_simulate_json.restype = C.c_void_p
        lib.ref_simulate_json.argtypes = [_i64p, C.c_int, _f64p, _f64p, C.c_int, C.c_int64,
                                          C.c_int, C.c_int, C.c_double, C.c_double]
        lib.ref_simulate_json_ex.restype = C.c_void_p
        lib.ref_simulate_json_ex.argtypes = [_i64p, C.c_int, _f64p, _f64p, C.c_int, C.c_int64,
                                             C.c_int, C.c_int, C.c_double, C.c_double,
                                             C.c_int64, C.c_int, C.c_int]
        lib.ref_free.argtypes = [C.c_void_p]
        lib.ref_time_sgd_steps.argtypes = [_i64p, C.c_int, C.c_int, C.c_int, C.c_int,
                                           C.c_uint64, C.c_double, _f64p]
        D = C.POINTER(C.c_double)
        lib.ref_calibrate.argtypes = [_f64p, _f64p, C.c_int, C.c_int, D, D, C.POINTER(C.c_int)]
        lib.ref_costs.argtypes = [C.c_double, C.c_int, C.c_double, C.c_double, D, D]
        lib.ref_theory.argtypes = [C.c_double] * 4 + [C.c_int, D, D, D]
        lib.ref_gp.argtypes = [_f64p, _f64p, C.c_int, _f64p, C.c_int, _f64p, _f64p, _f64p]
        lib.ref_tune_quadratic.argtypes = [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int,
                                           _f64p, _f64p, C.POINTER(C.c_int)]
        self.lib = lib

    def _check(self, rc):
        if rc < 0:
            raise ValueError(self.lib.ref_last_error().decode())
        return rc

    def preset_params(self, name: str, profile: int = 0) -> np.ndarray:
        out = np.zeros(1024, np.int64)
        n = self._check(self.lib.ref_preset_params(name.encode(), profile, out, 1024))
        return out[:n].copy()

    def build_plan(self, counts, buffer_bytes: int, bytes_per_elem: int = 4):
        c = np.ascontiguousarray(counts, np.int64)
        lo = np.zeros(len(c) + 1, np.int32)
        hi = np.zeros(len(c) + 1, np.int32)
        n = self._check(self.lib.ref_build_plan(c, len(c), bytes_per_elem, buffer_bytes, lo, hi))
        return [(int(lo[g]), int(hi[g])) for g in range(n)]

    def chunk_ranges(self, d: int, P: int):
        b = np.zeros(P, np.int64)
        e = np.zeros(P, np.int64)
        self._check(self.lib.ref_chunk_ranges(d, P, b, e))
        return b, e

    def random_vectors(self, P: int, d: int, seed: int) -> np.ndarray:
        out = np.empty(P * d, np.float64)
        self.lib.ref_random_vectors(P, d, seed, out)
        return out.reshape(P, d)

    def ring_reduce_scatter(self, vecs):
        v = np.ascontiguousarray(vecs, np.float64)
        out = np.empty(v.shape[1], np.float64)
        rounds = C.c_int(0)
        self._check(self.lib.ref_ring_reduce_scatter(v.shape[0], v.shape[1], v.reshape(-1),
                                                     out, C.byref(rounds)))
        return out, rounds.value

    def all_reduce(self, vecs, average: bool):
        v = np.ascontiguousarray(vecs, np.float64)
        out = np.empty_like(v)
        self._check(self.lib.ref_all_reduce(v.shape[0], v.shape[1], v.reshape(-1),
                                            out.reshape(-1), int(average)))
        return out

    def sgd_step(self, w, grads, lr: float) -> np.ndarray:
        w = np.ascontiguousarray(w, np.float64)
        g = np.ascontiguousarray(grads, np.float64)
        out = np.empty_like(g)
        self._check(self.lib.ref_sgd_step(g.shape[0], g.shape[1], lr, w, g.reshape(-1),
                                          out.reshape(-1)))
        return out

    def sgd_step_replicas(self, ws, grads, lr: float) -> np.ndarray:
        ws = np.ascontiguousarray(ws, np.float64)
        g = np.ascontiguousarray(grads, np.float64)
        out = np.empty_like(g)
        self._check(self.lib.ref_sgd_step_replicas(g.shape[0], g.shape[1], lr, ws.reshape(-1),
                                                   g.reshape(-1), out.reshape(-1)))
        return out

    POLICY = {"WFBP": 0, "WFBP_FUSED": 1, "PRIORITY_PARTITION": 2, "DEAR": 3, "DEAR_FUSED": 4}

    def simulate(self, counts, t_ff, t_bp, policy: str, fusion_buffer_bytes: int = 0,
                 group_dependency: bool = False, workers: int = 2, alpha: float = 0.0,
                 beta: float = 0.0, partition_bytes: int = 0, negotiation_rounds: int = 1,
                 negotiation_floating: bool = False) -> dict:
        c = np.ascontiguousarray(counts, np.int64)
        tf = np.ascontiguousarray(t_ff, np.float64)
        tb = np.ascontiguousarray(t_bp, np.float64)
        p = self.lib.ref_simulate_json_ex(c, len(c), tf, tb, self.POLICY[policy],
                                          fusion_buffer_bytes, int(group_dependency), workers,
                                          alpha, beta, int(partition_bytes),
                                          int(negotiation_rounds), int(negotiation_floating))
        if not p:
            raise ValueError(self.lib.ref_last_error().decode())
        try:
            return json.loads(C.string_at(p).decode())
        finally:
            self.lib.ref_free(p)

    def calibrate(self, measurements, workers: int) -> dict:
        b = np.ascontiguousarray([m[0] for m in measurements], np.float64)
        t = np.ascontiguousarray([m[1] for m in measurements], np.float64)
        a, be, cl = C.c_double(), C.c_double(), C.c_int()
        self._check(self.lib.ref_calibrate(b, t, len(b), workers, C.byref(a), C.byref(be),
                                           C.byref(cl)))
        return {"alpha": a.value, "beta": be.value, "clamped": bool(cl.value)}

    def costs(self, nbytes: float, workers: int, alpha: float, beta: float):
        rs, ar = C.c_double(), C.c_double()
        self._check(self.lib.ref_costs(nbytes, workers, alpha, beta, C.byref(rs), C.byref(ar)))
        return rs.value, ar.value

    def theory(self, t_ff, t_bp, t_rs, t_ag, workers):
        d, b, s = C.c_double(), C.c_double(), C.c_double()
        self._check(self.lib.ref_theory(t_ff, t_bp, t_rs, t_ag, workers, C.byref(d), C.byref(b),
                                        C.byref(s)))
        return {"dear": d.value, "baseline": b.value, "smax": s.value}

    def gp(self, obs, queries):
        xb = np.ascontiguousarray([o[0] for o in obs], np.float64)
        ty = np.ascontiguousarray([o[1] for o in obs], np.float64)
        q = np.ascontiguousarray(queries, np.float64)
        m, v, e = (np.zeros(len(q)) for _ in range(3))
        self._check(self.lib.ref_gp(xb, ty, len(xb), q, len(q), m, v, e))
        return m, v, e

    def tune_quadratic(self, opt_mb, width_mb, peak, max_trials=20, measure_steps=1):
        b = np.zeros(max_trials + 2)
        t = np.zeros(max_trials + 2)
        n = C.c_int(0)
        self._check(self.lib.ref_tune_quadratic(opt_mb, width_mb, peak, max_trials,
                                                measure_steps, b, t, C.byref(n)))
        return b[:n.value].copy(), t[:n.value].copy()

    def time_sgd_steps(self, bucket_elems, P: int, threads: int, steps: int,
                       seed: int = 1, lr: float = 0.05) -> np.ndarray:
        b = np.ascontiguousarray(bucket_elems, np.int64)
        out = np.zeros(steps, np.float64)
        self._check(self.lib.ref_time_sgd_steps(b, len(b), P, threads, steps, seed, lr, out))
        return out
