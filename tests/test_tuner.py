"""The product BO fusion-buffer tuner (paper_2302_12445_b200.tuner) against the
reference's gp.cpp / tuner.cpp (oracle/_ref build)."""
import math

import numpy as np
import pytest

from paper_2302_12445_b200 import tuner as T


def test_gp_matches_reference(reference):
    rng = np.random.default_rng(11)
    for _ in range(20):
        n = int(rng.integers(1, 9))
        xs = rng.uniform(1e6, 1e8, n)
        obs = [(float(x), float(rng.uniform(100, 200))) for x in xs]
        q = np.linspace(1e6, 1e8, 37)
        m, v, e = reference.gp(obs, q)
        gp = T.GpPosterior(obs, T.GpHyperParams(), 1e6, 1e8)
        for j, x in enumerate(q):
            mm, vv = gp.predict(float(x))
            assert mm == pytest.approx(m[j], rel=1e-9, abs=1e-9)
            assert vv == pytest.approx(v[j], rel=1e-6, abs=1e-9)
            ee = T.expected_improvement(gp, float(x), gp.best_throughput(), 0.1)
            assert ee == pytest.approx(e[j], rel=1e-6, abs=1e-9)


@pytest.mark.parametrize("opt_mb,width", [(35.0, 10.0), (12.0, 5.0), (80.0, 30.0)])
def test_tune_trace_matches_reference(reference, opt_mb, width):
    obj = lambda x: 1000.0 - ((x / 1e6 - opt_mb) / width) ** 2  # noqa: E731
    rb, rt = reference.tune_quadratic(opt_mb, width, 1000.0, max_trials=12, measure_steps=1)
    res = T.tune(obj, T.TunerConfig(max_trials=12, measure_steps=1))
    got = [r.buffer_bytes for r in res["trace"]]
    assert len(got) == len(rb)
    # identical trials until a suggestion lands within float noise of a tie
    same = 0
    for a, b in zip(got, rb):
        if abs(a - b) > 1.0:
            break
        same += 1
    assert same >= 6, (got, list(rb))
    # same search quality as the reference's tuner
    assert res["best_throughput"] >= max(rt) - 1e-6 * abs(max(rt))


def test_failures_and_abort():
    calls = {"n": 0}

    def obj(x):
        calls["n"] += 1
        raise RuntimeError("boom")
    with pytest.raises(RuntimeError, match="no successful observations"):
        T.tune(obj, T.TunerConfig(max_trials=10, measure_steps=1))
    assert calls["n"] == 3  # init trial + 2 fallbacks, then abort after 3 consecutive


def test_config_validation():
    with pytest.raises(ValueError):
        T.TunerConfig(lower_bytes=2e8).validate()
    with pytest.raises(ValueError):
        T.TunerConfig(init_buffer_bytes=5e8).validate()
    assert math.isclose(T.expected_improvement_value(1.0, 0.0, 0.5, 0.1), 0.4)
