"""The product's prediction layer (paper_2302_12445_b200.costmodel) against the
reference build: alpha-beta costs, calibration, Eq. 6-8, and the simulated
DeAR / WFBP iteration times of the golden scenarios."""
import json
import os

import numpy as np
import pytest

from paper_2302_12445_b200 import costmodel as cm

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_costs_match_reference(reference):
    rng = np.random.default_rng(5)
    for _ in range(200):
        d, P = float(rng.uniform(0, 1e9)), int(rng.integers(1, 65))
        a, b = float(rng.uniform(0, 1e-4)), float(rng.uniform(0, 2e-9))
        rs, ar = reference.costs(d, P, a, b)
        assert cm.reduce_scatter_time(d, P, a, b) == rs
        assert cm.all_reduce_time(d, P, a, b) == ar
        assert cm.reduce_scatter_time(d, P, a, b) + cm.all_gather_time(d, P, a, b) == ar


def test_calibration_matches_reference(reference):
    # the paper's two points (test_cost_model.cpp:33-34)
    pts = [(1e6, 4.5e-3), (5e5, 3.9e-3)]
    got, ref = cm.calibrate_alpha_beta(pts, 64), reference.calibrate(pts, 64)
    assert got["alpha"] == pytest.approx(ref["alpha"], rel=1e-9)
    assert got["beta"] == pytest.approx(ref["beta"], rel=1e-9)
    assert got["alpha"] == pytest.approx(2.6190476e-5, rel=1e-6)
    rng = np.random.default_rng(9)
    for _ in range(50):
        P = int(rng.integers(2, 9))
        a, b = float(rng.uniform(1e-6, 1e-4)), float(rng.uniform(1e-12, 1e-9))
        sizes = np.exp(rng.uniform(np.log(6.4e4), np.log(2.6e8), 8))
        pts = [(s, cm.all_reduce_time(s, P, a, b) * float(rng.uniform(0.95, 1.05))) for s in sizes]
        got, ref = cm.calibrate_alpha_beta(pts, P), reference.calibrate(pts, P)
        assert got["alpha"] == pytest.approx(ref["alpha"], rel=1e-6, abs=1e-15)
        assert got["beta"] == pytest.approx(ref["beta"], rel=1e-6, abs=1e-21)
    with pytest.raises(ValueError):
        cm.calibrate_alpha_beta([(1e6, 1e-3), (1e6, 2e-3)], 4)


def test_theory_matches_reference(reference):
    rng = np.random.default_rng(3)
    for _ in range(100):
        v = [float(x) for x in rng.uniform(0, 1e-2, 4)]
        P = int(rng.integers(1, 65))
        ref = reference.theory(*v, P)
        t = cm.theoretical_times(*v)
        assert t["dear"] == ref["dear"] and t["baseline"] == ref["baseline"]
        assert cm.max_speedup(*v, P) == pytest.approx(ref["smax"], rel=1e-15)


def test_predicted_iterations_match_reference_simulator():
    with open(os.path.join(GOLD, "schedules.json")) as f:
        scen = json.load(f)["scenarios"]
    for s in scen:
        got = cm.predict_iteration([4 * c for c in s["counts"]], s["t_ff"], s["t_bp"],
                                   s["policy"], s["buffer"], s["P"], s["alpha"], s["beta"])
        assert got["iteration_seconds"] == pytest.approx(s["result"]["iteration_seconds"],
                                                         rel=1e-12), s["name"]


def _labels(order):
    return [("RS g%d" % v) if v > 0 else ("AG g%d" % -v) for v in order]


@pytest.mark.parametrize("gd", [False, True])
@pytest.mark.parametrize("P,alpha,beta", [(2, 1e-4, 1e-9), (4, 5e-5, 4e-9), (8, 2e-5, 1e-8)])
def test_comm_order_is_reference_dispatch_order(gd, P, alpha, beta):
    """The dispatch sequence predict_iteration hands to Runtime.set_comm_order
    is the reference scheduler's Comm dispatch order (oracle restatement of
    task_graph.cpp:181-210 + simulate.cpp:65-159), with and without
    dear_group_dependency."""
    from oracle.schedule import build_graph, comm_dispatch_order, simulate

    rng = np.random.default_rng(P)
    counts = [int(x) for x in rng.integers(1, 400_000, size=40)]
    t_ff = [float(x) for x in rng.uniform(1e-5, 3e-5, size=40)]
    t_bp = [2 * t for t in t_ff]
    lb = [4 * c for c in counts]
    got = cm.predict_iteration(lb, t_ff, t_bp, "DEAR_FUSED", 1_000_000, P, alpha, beta,
                               group_dependency=gd)
    tasks, _ = build_graph(lb, t_ff, t_bp, "DEAR_FUSED", 1_000_000, group_dependency=gd, P=P,
                           alpha=alpha, beta=beta)
    span, makespan = simulate(tasks)
    assert _labels(got["comm_order"]) == comm_dispatch_order(tasks, span)
    assert got["iteration_seconds"] == pytest.approx(makespan, rel=1e-12)


def test_comm_order_with_measured_stage_times():
    """rs_times / ag_times replace the alpha-beta durations per group."""
    counts = [100_000] * 12
    lb = [4 * c for c in counts]
    plan_groups = cm.predict_iteration(lb, [1e-5] * 12, [2e-5] * 12, "DEAR_FUSED", 800_000, 4,
                                       0.0, 0.0)["buckets"]
    slow = cm.predict_iteration(lb, [1e-5] * 12, [2e-5] * 12, "DEAR_FUSED", 800_000, 4, 0.0, 0.0,
                                group_dependency=True, rs_times=[1e-3] * plan_groups,
                                ag_times=[1e-3] * plan_groups)
    fast = cm.predict_iteration(lb, [1e-5] * 12, [2e-5] * 12, "DEAR_FUSED", 800_000, 4, 0.0, 0.0,
                                group_dependency=True, rs_times=[1e-6] * plan_groups,
                                ag_times=[1e-6] * plan_groups)
    # comm-bound: every RS first, then the AGs in feed-forward order
    G = plan_groups
    assert slow["comm_order"] == list(range(1, G + 1)) + [-g for g in range(G, 0, -1)]
    # comm much faster than backprop: each AG right behind its RS
    assert fast["comm_order"] == [v for g in range(1, G + 1) for v in (g, -g)]


def test_priority_partition_matches_reference_build(reference):
    """PRIORITY_PARTITION (task_graph.cpp:215-258): per-layer parts of
    ceil(bytes / partition_bytes), each behind a negotiation (or a floating
    release delay), issued by ascending layer. The restatement's makespan and
    its AR dispatch sequence equal the reference build's on random models."""
    import random

    from paper_2302_12445_b200 import costmodel as cm

    rng = random.Random(5)
    for _ in range(120):
        L = rng.randint(1, 7)
        counts = [rng.choice([0, 1, 50, 700, 5000, 12000]) for _ in range(L)]
        tf = [rng.uniform(0.1, 2) for _ in range(L)]
        tb = [rng.uniform(0.1, 3) for _ in range(L)]
        pb = rng.choice([1000, 4096, 8000, 30000])
        nr, fl = rng.randint(0, 2), rng.random() < 0.5
        P, a, b = rng.choice([2, 4, 8]), rng.choice([0.0, 1e-3]), rng.choice([0.0, 1e-6])
        ref = reference.simulate(counts, tf, tb, "PRIORITY_PARTITION", 0, workers=P, alpha=a,
                                 beta=b, partition_bytes=pb, negotiation_rounds=nr,
                                 negotiation_floating=fl)
        got = cm.predict_iteration([4 * c for c in counts], tf, tb, "PRIORITY_PARTITION", 0, P,
                                   a, b, partition_bytes=pb, negotiation_rounds=nr,
                                   negotiation_floating=fl)
        assert got["iteration_seconds"] == ref["iteration_seconds"]
        ref_ar = [t["label"] for t in sorted(ref["tasks"], key=lambda t: (t["start"], t["id"]))
                  if t["kind"] == "AR"]
        parts = [(l, k + 1) for l, n in cm.partition_plan([4 * c for c in counts], pb)
                 for k in range(n)]
        got_ar = ["AR l%d p%d" % parts[g - 1] for g in got["comm_order"]]
        assert got_ar == ref_ar
