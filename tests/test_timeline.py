"""Measured-timeline export (paper_2302_12445_b200.timeline): the reference's
Chrome-trace / CSV layout and validate_timeline-style invariants."""
import json

from paper_2302_12445_b200 import timeline as T


def _sample():
    compute = [("FF l1", 0.0, 1.0), ("FF l2", 1.5, 2.5), ("BP l2", 2.5, 4.5), ("BP l1", 4.5, 6.5)]
    buckets = [{"low": 2, "high": 2, "elems": 10, "slot_stride": 64},
               {"low": 1, "high": 1, "elems": 10, "slot_stride": 64}]
    stamps = [dict(pack0=4.6, pack1=4.7, rs1=5.0, update1=5.1, ag0=7.0, ag1=7.3, unpack1=7.4),
              dict(pack0=6.6, pack1=6.7, rs1=7.0, update1=7.1, ag0=6.9, ag1=7.0, unpack1=7.1)]
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
    assert abs(tl["exposed_comm_ms"] - (7.4 - 6.0)) < 1e-9


def test_wfbp_labels_and_violations():
    c, b, s = _sample()
    tl = T.build(c, b, s, "WFBP")
    labels = {e["label"] for e in tl["events"] if e["resource"] == "Comm"}
    assert labels == {"AR l2", "AR l1"}
    # a reduction that starts before its bucket's last backprop is flagged
    s[0]["pack0"] = 3.0
    assert any("before BP l2" in v for v in T.validate(c, b, s, "DEAR_FUSED"))
    c2 = [("FF l1", 0.0, 2.0), ("FF l2", 1.0, 3.0)]
    assert any("overlaps" in v for v in T.validate(c2, [], [], "DEAR"))
