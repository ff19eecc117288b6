"""Measured-timeline export (paper_2302_12445_b200.timeline): the reference's
Chrome-trace / CSV layout and validate_timeline-style invariants."""
import json

from paper_2302_12445_b200 import timeline as T


def _sample():
    # the reference's iteration: BP_L..BP_1, then the next FF_1..FF_L, each FF
    # gated on its bucket's all-gather (task_graph.cpp:127-146, :207)
    compute = [("BP l2", 0.0, 2.0), ("BP l1", 2.0, 4.0), ("FF l1", 5.2, 6.2), ("FF l2", 7.5, 8.5)]
    buckets = [{"low": 2, "high": 2, "elems": 10, "slot_stride": 64},
               {"low": 1, "high": 1, "elems": 10, "slot_stride": 64}]
    stamps = [dict(pack0=2.1, pack1=2.2, rs1=2.5, update1=2.6, ag0=6.9, ag1=7.2, unpack1=7.4),
              dict(pack0=4.1, pack1=4.2, rs1=4.5, update1=4.6, ag0=4.6, ag1=5.0, unpack1=5.1)]
    return compute, buckets, stamps


def test_trace_schema_and_labels():
    tl = T.build(*_sample(), "DEAR_FUSED")
    tr = T.chrome_trace(tl)
    names = {e["args"]["name"] for e in tr["traceEvents"] if e["ph"] == "M"}
    assert {"Compute", "Comm"} <= names
    labels = {e["name"] for e in tr["traceEvents"] if e["ph"] == "X"}
    assert {"FF l1", "BP l2", "RS g1", "AG g2", "PACK g1"} <= labels
    assert all(e["dur"] >= 0 for e in tr["traceEvents"] if e["ph"] == "X")
    json.loads(T.dumps(tl))
    assert T.csv(tl).startswith("task_id,label,resource,start_seconds,end_seconds\n")
    assert tl["ff_ms"] == 2.0 and tl["bp_ms"] == 4.0
    assert abs(tl["exposed_comm_ms"] - (8.5 - 6.0)) < 1e-9
    assert tl["violations"] == []


def test_wfbp_labels_and_violations():
    c, b, s = _sample()
    tl = T.build(c, b, s, "WFBP")
    labels = {e["label"] for e in tl["events"] if e["resource"] == "Comm"}
    assert labels == {"AR l2", "AR l1"}
    # a reduction that starts before its bucket's last backprop is flagged
    s[0]["pack0"] = 1.0
    assert any("before BP l2" in v for v in T.validate(c, b, s, "DEAR_FUSED"))
    # a forward that starts before its bucket's all-gather (+ unpack) ended
    c3 = list(c)
    c3[3] = ("FF l2", 7.0, 8.0)
    s[0]["pack0"] = 2.1
    assert T.validate(c, b, s, "DEAR_FUSED") == []
    assert any("FF l2 starts before AG g1" in v for v in T.validate(c3, b, s, "DEAR_FUSED"))
    assert any("FF l2 starts before AR g1" in v for v in T.validate(c3, b, s, "WFBP"))
    # fused peer kernels: no unpack stamp, the all-gather ends at ag1
    s2 = [dict(x, unpack1=None, update1=None) for x in s]
    assert any("FF l2 starts before AG g1" in v for v in T.validate(c3, b, s2, "DEAR_FUSED"))
    c2 = [("FF l1", 0.0, 2.0), ("FF l2", 1.0, 3.0)]
    assert any("overlaps" in v for v in T.validate(c2, [], [], "DEAR"))
