"""Bayesian-optimisation fusion-buffer tuner (DeAR-BO, §IV).

Restates the reference's GP + expected-improvement tuner so it can drive the
LIVE B200 objective (measured samples/s of the DeAR runtime at a buffer size):

  * GpPosterior           proj/src/gp.cpp:46-158   RBF kernel on buffer bytes
                          normalised to [0, 1], standardised outputs, Cholesky
                          with jitter escalation, variance snap 1e-12
  * expected_improvement  proj/src/gp.cpp:160-183  in standardised space, xi margin
  * suggest_next          proj/src/tuner.cpp:135-174  512-point grid + golden-section
                          refinement (60 iterations); all-zero EI -> max variance
  * tune / random_search / grid_search   proj/src/tuner.cpp:176-227, with the
                          SearchLog protocol (:79-132): whole-byte buffers,
                          measure_steps averaged calls, failed evaluations
                          recorded as NaN, three consecutive failures abort.
Defaults are the reference's TunerConfig (tuner.hpp:28-37): 1-100 MB, xi = 0.1,
first trial 25 MB, 10 measured steps, 20 trials. Pinned against the reference
build in tests/test_tuner.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np

_INV_SQRT_2PI = 0.39894228040143268
_VARIANCE_SNAP = 1e-12


@dataclass
class GpHyperParams:
    lengthscale: float = 0.2
    signal_variance: float = 1.0
    noise_variance: float = 1e-6


@dataclass
class TunerConfig:
    lower_bytes: float = 1e6
    upper_bytes: float = 1e8
    xi: float = 0.1
    init_buffer_bytes: float = 2.5e7
    measure_steps: int = 10
    max_trials: int = 20
    seed: int = 0
    gp: GpHyperParams = field(default_factory=GpHyperParams)

    def validate(self) -> None:
        if not (self.lower_bytes < self.upper_bytes) or not (self.lower_bytes > 0.0):
            raise ValueError("tuner: need 0 < lower_bytes < upper_bytes")
        if self.xi < 0.0:
            raise ValueError("tuner: xi must be >= 0")
        if self.init_buffer_bytes < self.lower_bytes or self.init_buffer_bytes > self.upper_bytes:
            raise ValueError("tuner: init_buffer_bytes out of bounds")
        if self.measure_steps < 1:
            raise ValueError("tuner: measure_steps must be >= 1")
        if self.max_trials < 1:
            raise ValueError("tuner: max_trials must be >= 1")


def _cholesky(k: np.ndarray):
    n = k.shape[0]
    L = np.zeros_like(k)
    for j in range(n):
        d = k[j, j] - float(np.dot(L[j, :j], L[j, :j]))
        if not d > 0.0:
            return None
        ljj = math.sqrt(d)
        L[j, j] = ljj
        for i in range(j + 1, n):
            L[i, j] = (k[i, j] - float(np.dot(L[i, :j], L[j, :j]))) / ljj
    return L


def _forward(L: np.ndarray, b: np.ndarray) -> np.ndarray:
    x = np.zeros_like(b)
    for i in range(len(b)):
        x[i] = (b[i] - float(np.dot(L[i, :i], x[:i]))) / L[i, i]
    return x


def _backward_t(L: np.ndarray, y: np.ndarray) -> np.ndarray:
    n = len(y)
    x = np.zeros_like(y)
    for i in range(n - 1, -1, -1):
        x[i] = (y[i] - float(np.dot(L[i + 1:, i], x[i + 1:]))) / L[i, i]
    return x


class GpPosterior:
    def __init__(self, observations, hyper: GpHyperParams, lower: float, upper: float):
        if not observations:
            raise ValueError("gp_fit: need at least one observation")
        if not lower < upper:
            raise ValueError("gp_fit: lower bound must be < upper bound")
        if not (hyper.lengthscale > 0 and hyper.signal_variance > 0 and hyper.noise_variance >= 0):
            raise ValueError("gp_fit: bad hyperparameters")
        if hyper.noise_variance == 0.0:
            for i, (xi_, yi) in enumerate(observations):
                for xj, yj in observations[i + 1:]:
                    if xi_ == xj and yi != yj:
                        raise ValueError("gp_fit: inconsistent noise-free observations "
                                         "(same buffer, different throughput)")
        self.obs = list(observations)
        self.hyper, self.lower, self.upper = hyper, float(lower), float(upper)
        n = len(self.obs)
        self.x = np.array([self.normalize(o[0]) for o in self.obs], np.float64)
        y = np.array([o[1] for o in self.obs], np.float64)
        self.y_mean = float(y.sum() / n)
        sd = math.sqrt(float(((y - self.y_mean) ** 2).sum()) / n)
        self.y_scale = sd if sd > 1e-15 * max(1.0, abs(self.y_mean)) else 1.0
        y_std = (y - self.y_mean) / self.y_scale
        k = np.array([[self.kernel(a, b) for b in self.x] for a in self.x], np.float64)
        k[np.diag_indices(n)] += hyper.noise_variance
        for jitter in (0.0, 1e-10, 1e-9, 1e-8, 1e-7, 1e-6):
            kj = k.copy()
            if jitter > 0.0:
                kj[np.diag_indices(n)] += jitter
            L = _cholesky(kj)
            if L is not None:
                self.L = L
                self.w = _backward_t(L, _forward(L, y_std))
                return
        raise RuntimeError("gp_fit: kernel matrix not positive definite after jitter escalation")

    def normalize(self, b: float) -> float:
        return (b - self.lower) / (self.upper - self.lower)

    def kernel(self, a: float, b: float) -> float:
        r = (a - b) / self.hyper.lengthscale
        return self.hyper.signal_variance * math.exp(-0.5 * r * r)

    def _kstar(self, b: float) -> np.ndarray:
        x = self.normalize(b)
        return np.array([self.kernel(x, xi) for xi in self.x], np.float64)

    def normalized_variance(self, b: float) -> float:
        v = _forward(self.L, self._kstar(b))
        var = self.hyper.signal_variance - float(np.dot(v, v))
        return 0.0 if var < _VARIANCE_SNAP else var

    def predict_standardized(self, b: float):
        return float(np.dot(self._kstar(b), self.w)), self.normalized_variance(b)

    def predict(self, b: float):
        m, v = self.predict_standardized(b)
        return m * self.y_scale + self.y_mean, v * self.y_scale * self.y_scale

    def best_throughput(self) -> float:
        return max(o[1] for o in self.obs)


def expected_improvement_value(mean: float, sigma: float, best: float, xi: float) -> float:
    if xi < 0.0:
        raise ValueError("expected_improvement: xi >= 0")
    if not sigma >= 0.0:
        raise ValueError("expected_improvement: sigma >= 0")
    gain = mean - best - xi
    if sigma == 0.0:
        return max(0.0, gain)
    z = gain / sigma
    cdf = 0.5 * math.erfc(-z / math.sqrt(2.0))
    pdf = _INV_SQRT_2PI * math.exp(-0.5 * z * z)
    return max(0.0, gain * cdf + sigma * pdf)


def expected_improvement(gp: GpPosterior, b: float, best: float, xi: float) -> float:
    m, v = gp.predict_standardized(b)
    best_std = (best - gp.y_mean) / gp.y_scale
    return expected_improvement_value(m, math.sqrt(v), best_std, xi)


_GRID = 512
_REFINE = 60
_INV_PHI = 0.6180339887498949


def _golden(gp, cfg, best, lo, hi):
    a, b = lo, hi
    c = b - _INV_PHI * (b - a)
    d = a + _INV_PHI * (b - a)
    fc = expected_improvement(gp, c, best, cfg.xi)
    fd = expected_improvement(gp, d, best, cfg.xi)
    for _ in range(_REFINE):
        if fc >= fd:
            b, d, fd = d, c, fc
            c = b - _INV_PHI * (b - a)
            fc = expected_improvement(gp, c, best, cfg.xi)
        else:
            a, c, fc = c, d, fd
            d = a + _INV_PHI * (b - a)
            fd = expected_improvement(gp, d, best, cfg.xi)
    return c if fc >= fd else d


def suggest_next(gp: GpPosterior, cfg: TunerConfig) -> float:
    cfg.validate()
    lo, hi = cfg.lower_bytes, cfg.upper_bytes
    best = gp.best_throughput()
    step = (hi - lo) / (_GRID - 1)
    best_i, best_ei, best_ei_var, best_var, var_i = 0, -1.0, -1.0, -1.0, 0
    for i in range(_GRID):
        x = lo + step * i
        ei = expected_improvement(gp, x, best, cfg.xi)
        var = gp.normalized_variance(x)
        if ei > best_ei or (ei == best_ei and var > best_ei_var):
            best_ei, best_ei_var, best_i = ei, var, i
        if var > best_var:
            best_var, var_i = var, i
    if best_ei <= 0.0:
        return lo + step * var_i
    cell_lo = lo + step * max(0, best_i - 1)
    cell_hi = lo + step * min(_GRID - 1, best_i + 1)
    refined = _golden(gp, cfg, best, cell_lo, cell_hi)
    return refined if expected_improvement(gp, refined, best, cfg.xi) > best_ei \
        else lo + step * best_i


@dataclass
class TrialRecord:
    trial: int
    buffer_bytes: float
    throughput: float
    ok: bool
    cumulative_best: float


class _Log:
    def __init__(self, cfg: TunerConfig):
        self.cfg, self.trace, self.obs = cfg, [], []
        self.best, self.fails = -math.inf, 0

    def evaluate(self, objective: Callable[[float], float], b: float) -> bool:
        x = min(max(float(np.round(b)), self.cfg.lower_bytes), self.cfg.upper_bytes)
        try:
            tot = 0.0
            for _ in range(self.cfg.measure_steps):
                tot += objective(x)
            thr, ok = tot / self.cfg.measure_steps, True
        except Exception:
            thr, ok = math.nan, False
        if ok:
            self.obs.append((x, thr))
            self.best = max(self.best, thr)
            self.fails = 0
        else:
            self.fails += 1
        self.trace.append(TrialRecord(len(self.trace) + 1, x, thr, ok, self.best))
        return ok

    def finish(self):
        if not self.obs:
            raise RuntimeError("tuner: no successful observations")
        best_b = next(b for b, t in self.obs if t == self.best)
        return {"best_buffer_bytes": best_b, "best_throughput": self.best, "trace": self.trace}


def tune(objective: Callable[[float], float], cfg: TunerConfig | None = None) -> dict:
    cfg = cfg or TunerConfig()
    cfg.validate()
    log = _Log(cfg)
    log.evaluate(objective, cfg.init_buffer_bytes)
    span = cfg.upper_bytes - cfg.lower_bytes
    fallback = [0.5 * (cfg.lower_bytes + cfg.upper_bytes), cfg.lower_bytes + 0.75 * span,
                cfg.lower_bytes + 0.25 * span]
    fb = 0
    for _ in range(cfg.max_trials):
        if log.fails >= 3:
            break
        if not log.obs:
            nxt = fallback[fb % 3]
            fb += 1
        else:
            gp = GpPosterior(log.obs, cfg.gp, cfg.lower_bytes, cfg.upper_bytes)
            nxt = suggest_next(gp, cfg)
        log.evaluate(objective, nxt)
    return log.finish()


def grid_search(objective, cfg: TunerConfig | None = None) -> dict:
    cfg = cfg or TunerConfig()
    cfg.validate()
    log = _Log(cfg)
    width = (cfg.upper_bytes - cfg.lower_bytes) / cfg.max_trials
    for i in range(cfg.max_trials):
        if log.fails >= 3:
            break
        log.evaluate(objective, cfg.lower_bytes + (i + 0.5) * width)
    return log.finish()
