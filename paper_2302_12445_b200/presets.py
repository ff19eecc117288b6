"""Benchmark model presets: per-tensor parameter counts.

Restates ``preset_model`` (proj/src/model.cpp:80-168): the tensor counts and
parameter totals of Table I, spread uniformly over tensors with the
first ``total % count`` tensors one larger (``spread_uniform``, :90-98), or the
"imbalanced" profile with 80% of the parameters in the last
``max(1, round(0.2 n))`` tensors (:138-152). Bit-exact with the reference
(tests/test_presets.py against tests/golden/plans.json).

``mlp4x1024`` is BASELINE config 1: four W[1024,1024] + b[1024] layers.
"""
from __future__ import annotations

PRESETS = {
    "resnet50": (161, 25_600_000),
    "densenet201": (604, 20_000_000),
    "inceptionv4": (449, 42_700_000),
    "bert_base": (206, 110_100_000),
    "bert_large": (398, 336_200_000),
}


def _spread(count: int, total: int) -> list[int]:
    if count <= 0:
        return []
    base, extra = divmod(total, count)
    return [base + (1 if i < extra else 0) for i in range(count)]


def _round_half_away(x: float) -> int:
    # std::llround semantics (halves away from zero)
    import math

    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def preset_param_counts(name: str, profile: str = "uniform") -> list[int]:
    """Per-tensor parameter counts, layer 1 (input side) first."""
    if name == "mlp4x1024":
        return [1024 * 1024 + 1024] * 4
    if name not in PRESETS:
        raise ValueError(f"unknown preset model '{name}'; valid presets: "
                         + ", ".join([*PRESETS, "mlp4x1024"]))
    n, total = PRESETS[name]
    if profile == "uniform":
        return _spread(n, total)
    if profile != "imbalanced":
        raise ValueError("profile must be 'uniform' or 'imbalanced'")
    tail = max(1, _round_half_away(0.2 * n))
    head = n - tail
    tail_params = total if head == 0 else _round_half_away(0.8 * total)
    return _spread(head, total - tail_params) + _spread(tail, tail_params)
