"""Measured iteration timelines in the reference's trace schema.

The reference exports simulated timelines as a Chrome trace (thread 0
"Compute", thread 1 "Comm", microseconds, task labels such as "FF l1",
"BP l3", "RS g2", "AG g2", "AR g1"; proj/src/trace_export.cpp:84-127,
task_label task_graph.cpp:51-58) and checks them with validate_timeline
(simulate.cpp:161-210). This module does the same for a *measured* B200
iteration: compute-stream CUDA events around every layer's FF / BP, and the
runtime's comm-stream stamps per bucket (``Runtime.timeline``).
"""
from __future__ import annotations

import json


def _first(st: dict, *keys):
    for k in keys:
        if st.get(k) is not None:
            return st[k]
    return None


def build(compute: list[tuple[str, float, float]], buckets: list[dict], stamps: list[dict],
          policy: str) -> dict:
    """compute: (label, start_ms, end_ms) for "BP l.." / "FF l.." in issue
    order — the reference's iteration is BP_L..BP_1 then FF_1..FF_L
    (task_graph.cpp:127-146), the feed-forward gated on the all-gathers;
    buckets: Runtime.buckets(); stamps: Runtime.timeline(base) (the fused
    peer kernels have no separate update / unpack stamps: the reduce-scatter
    ends at rs1, the all-gather at ag1).
    Returns {"events": [...], "iteration_ms", "ff_ms", "bp_ms",
    "exposed_comm_ms", "violations": [...]}."""
    dear = policy.startswith("DEAR")
    fused = policy.endswith("_FUSED")
    events = []
    for label, s, e in compute:
        events.append({"label": label, "resource": "Compute", "start": s, "end": e})
    for g, (b, st) in enumerate(zip(buckets, stamps), start=1):
        subj = f"g{g}" if (dear or fused) else f"l{b['high']}"
        ag_end = _first(st, "unpack1", "ag1")
        if dear:
            if st["pack0"] is not None and st["rs1"] is not None:
                events.append({"label": f"RS {subj}", "resource": "Comm", "start": st["pack0"],
                               "end": st["rs1"]})
            if st["ag0"] is not None and ag_end is not None:
                events.append({"label": f"AG {subj}", "resource": "Comm", "start": st["ag0"],
                               "end": ag_end})
        elif st["pack0"] is not None and ag_end is not None:
            events.append({"label": f"AR {subj}", "resource": "Comm", "start": st["pack0"],
                           "end": ag_end})
        for name, a, z in (("PACK", "pack0", "pack1"), ("UPDATE", "rs1", "update1"),
                           ("UNPACK", "ag1", "unpack1")):
            if st[a] is not None and st[z] is not None:
                events.append({"label": f"{name} {subj}", "resource": "CommKernels",
                               "start": st[a], "end": st[z]})
    events.sort(key=lambda e: (e["start"], e["resource"], e["label"]))
    ff = sum(e - s for lab, s, e in compute if lab.startswith("FF"))
    bp = sum(e - s for lab, s, e in compute if lab.startswith("BP"))
    t0 = min(e["start"] for e in events)
    t1 = max(e["end"] for e in events)
    out = {"events": events, "iteration_ms": t1 - t0, "ff_ms": ff, "bp_ms": bp,
           "exposed_comm_ms": max(0.0, (t1 - t0) - ff - bp)}
    out["violations"] = validate(compute, buckets, stamps, policy)
    return out


def validate(compute, buckets, stamps, policy: str, tol_ms: float = 1e-3) -> list[str]:
    """validate_timeline's invariants on measured events: no overlap on the
    compute stream; RS_g / AR_g start after the BP of the bucket's last layer
    (its lowest index, task_graph.cpp:148-154); FF_l starts after its bucket's
    all-gather + unpack (task_graph.cpp:207)."""
    bad = []
    prev_end = None
    for label, s, e in compute:
        if e < s - tol_ms:
            bad.append(f"{label}: negative duration")
        if prev_end is not None and s < prev_end - tol_ms:
            bad.append(f"{label}: overlaps the previous compute task")
        prev_end = e
    bp_end = {int(l.split("l")[1]): e for l, _, e in compute if l.startswith("BP")}
    ff_start = {int(l.split("l")[1]): s for l, s, _ in compute if l.startswith("FF")}
    kind = "AG" if policy.startswith("DEAR") else "AR"
    for g, (b, st) in enumerate(zip(buckets, stamps), start=1):
        low = b["low"]
        if st["pack0"] is not None and low in bp_end and st["pack0"] < bp_end[low] - tol_ms:
            bad.append(f"bucket g{g}: reduction starts before BP l{low} ends")
        # FF_l <- AG_{g(l)} (DeAR) / AR_{g(l)} (WFBP), the parameters' last
        # writer being the all-gather's unpack (task_graph.cpp:170-171, :207)
        ag_end = _first(st, "unpack1", "ag1")
        if ag_end is None:
            continue
        for l in range(b["low"], b["high"] + 1):
            if l in ff_start and ff_start[l] < ag_end - tol_ms:
                bad.append(f"FF l{l} starts before {kind} g{g} (+ unpack) ends")
    return bad


def chrome_trace(tl: dict) -> dict:
    """The reference's Chrome-trace layout (trace_export.cpp:84-110), µs."""
    tids = {"Compute": 0, "Comm": 1, "CommKernels": 2}
    ev = [{"name": "thread_name", "ph": "M", "pid": 0, "tid": t, "args": {"name": n}}
          for n, t in tids.items()]
    t0 = min(e["start"] for e in tl["events"])
    for e in tl["events"]:
        ev.append({"name": e["label"], "ph": "X", "ts": (e["start"] - t0) * 1e3,
                   "dur": (e["end"] - e["start"]) * 1e3, "pid": 0, "tid": tids[e["resource"]]})
    return {"traceEvents": ev, "displayTimeUnit": "ms"}


def csv(tl: dict) -> str:
    """timeline_csv layout (trace_export.cpp:117-127), seconds."""
    t0 = min(e["start"] for e in tl["events"])
    rows = ["task_id,label,resource,start_seconds,end_seconds"]
    for i, e in enumerate(tl["events"]):
        rows.append(f"{i},{e['label']},{e['resource']},{(e['start'] - t0) / 1e3:.9g},"
                    f"{(e['end'] - t0) / 1e3:.9g}")
    return "\n".join(rows) + "\n"


def dumps(tl: dict) -> str:
    return json.dumps(chrome_trace(tl))
