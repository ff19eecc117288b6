"""The schedule restatement (oracle/schedule.py) against the reference's own
build_graph + simulate (golden fixtures from oracle/_ref) and the reference's
golden traces (test_simulate.cpp:52-110, test_task_graph.cpp:79-111). The
runtime's collective issue order is checked against this restatement in
tests/test_runtime_gpu.py::test_trace_is_reference_dispatch_order."""
import json
import os

import pytest

from oracle.schedule import AG, AR, BARRIER, FF, RS, build_graph, comm_dispatch_order, simulate

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _scen():
    with open(os.path.join(GOLD, "schedules.json")) as f:
        return json.load(f)["scenarios"]


@pytest.mark.parametrize("s", _scen(), ids=lambda s: s["name"])
def test_restated_schedule_matches_reference(s):
    tasks, plan = build_graph([4 * c for c in s["counts"]], s["t_ff"], s["t_bp"], s["policy"],
                              s["buffer"], P=s["P"], alpha=s["alpha"], beta=s["beta"])
    ref = s["result"]
    assert len(tasks) == len(ref["tasks"])
    span, makespan = simulate(tasks)
    for t, r in zip(tasks, ref["tasks"]):
        assert t.label == r["label"]
        assert t.issue_order == r["issue_order"]
        assert sorted(t.deps) == sorted(r["deps"])
        assert t.duration == pytest.approx(r["duration"], rel=1e-15, abs=0)
        assert span[t.id][0] == pytest.approx(r["start"], rel=1e-12, abs=1e-15)
        assert span[t.id][1] == pytest.approx(r["end"], rel=1e-12, abs=1e-15)
    assert makespan == pytest.approx(ref["iteration_seconds"], rel=1e-12)
    if ref["groups"]:
        assert [tuple(g) for g in ref["groups"]] == plan


def test_golden_traces():
    # test_simulate.cpp:52-93: two layers, t_ff 1, t_bp 2, collective = alpha = 1
    tasks, _ = build_graph([4, 4], [1, 1], [2, 2], "WFBP", P=2, alpha=1.0)
    span, mk = simulate(tasks)
    assert mk == 8.0
    tasks, _ = build_graph([4, 4], [1, 1], [2, 2], "DEAR", P=2, alpha=1.0)
    span, mk = simulate(tasks)
    ev = {t.label: span[t.id] for t in tasks}
    assert ev["RS g1"] == (2.0, 3.0) and ev["RS g2"] == (4.0, 5.0)
    assert ev["AG g2"] == (5.0, 6.0) and ev["AG g1"] == (6.0, 7.0)
    assert ev["FF l1"][0] == 6.0 and ev["FF l2"][0] == 7.0 and mk == 8.0
    # :95-110 comm-heavy: WFBP 13 vs DEAR 11
    w, _ = build_graph([4] * 3, [1] * 3, [1] * 3, "WFBP", P=2, alpha=1.5)
    d, _ = build_graph([4] * 3, [1] * 3, [1] * 3, "DEAR", P=2, alpha=1.5)
    assert simulate(w)[1] == 13.0 and simulate(d)[1] == 11.0


def test_dear_graph_shape():  # test_task_graph.cpp:79-111
    tasks, _ = build_graph([1_000_000] * 3, [1.0] * 3, [2.0] * 3, "DEAR", P=8, alpha=1e-5,
                           beta=1e-9)
    rs = [t for t in tasks if t.kind == RS]
    ag = [t for t in tasks if t.kind == AG]
    bar = [t for t in tasks if t.kind == BARRIER]
    assert len(rs) == 3 and len(ag) == 3 and len(bar) == 1 and len(bar[0].deps) == 3
    by = {t.label: t for t in tasks}
    assert by["AG g3"].issue_order < by["AG g2"].issue_order < by["AG g1"].issue_order
    assert by["AG g3"].id in by["FF l1"].deps


def test_dispatch_order_contract():
    """RS in plan order during backprop, then AG in feed-forward order (DEAR);
    AR per group in plan order (WFBP)."""
    counts = [1000, 2000, 3000, 4000, 5000]
    tasks, plan = build_graph([4 * c for c in counts], [1.0] * 5, [2.0] * 5, "DEAR_FUSED",
                              30_000, P=4, alpha=1e-3)
    order = comm_dispatch_order(tasks, simulate(tasks)[0])
    G = len(plan)
    assert order == [f"RS g{g}" for g in range(1, G + 1)] + [f"AG g{g}" for g in range(G, 0, -1)]
    tasks, plan = build_graph([4 * c for c in counts], [1.0] * 5, [2.0] * 5, "WFBP", 0, P=4,
                              alpha=1e-3)
    order = comm_dispatch_order(tasks, simulate(tasks)[0])
    assert order == [f"AR l{l}" for l in range(5, 0, -1)]
    assert all(t.kind in (FF, "BP", AR) for t in tasks)
