"""alpha-beta collective cost model, DeAR/WFBP schedule prediction and the
paper's analysis bounds — the reference's prediction layer, fed with what the
B200 runtime measures.

Restates (tested against the reference build in tests/test_costmodel.py):
  * reduce_scatter_time / all_gather_time / all_reduce_time
        proj/src/cost_model.cpp:34-48      (P-1)(alpha + (d/P) beta), AR = RS + AG
  * calibrate_alpha_beta                 proj/src/cost_model.cpp:79-133
  * theoretical_times (Eq. 7 / Eq. 8), max_speedup (Eq. 6), breakdown
        proj/src/analysis.cpp:34-101
  * predict_iteration: build_graph (task_graph.cpp:127-210) + the two-stream
    list scheduler (simulate.cpp:65-159) on measured per-layer times.
"""
from __future__ import annotations

import heapq

import numpy as np

from .plan import build_fusion_plan


def reduce_scatter_time(nbytes: float, P: int, alpha: float, beta: float) -> float:
    if not (nbytes >= 0) or P < 1 or alpha < 0 or beta < 0:
        raise ValueError("message_bytes must be finite and >= 0; P >= 1; alpha, beta >= 0")
    return (P - 1.0) * (alpha + (nbytes / P) * beta)


def all_gather_time(nbytes: float, P: int, alpha: float, beta: float) -> float:
    return reduce_scatter_time(nbytes, P, alpha, beta)


def all_reduce_time(nbytes: float, P: int, alpha: float, beta: float) -> float:
    return reduce_scatter_time(nbytes, P, alpha, beta) + all_gather_time(nbytes, P, alpha, beta)


def calibrate_alpha_beta(measurements, workers: int) -> dict:
    """Least-squares fit of t = 2(P-1) alpha + 2(P-1)(d/P) beta to measured
    all-reduce times [(bytes, seconds)], size column rescaled for conditioning,
    negative coefficients clamped to 0."""
    if workers < 2:
        raise ValueError("calibrate_alpha_beta: workers must be >= 2")
    if len(measurements) < 2:
        raise ValueError("calibrate_alpha_beta: need at least 2 measurements")
    d = np.array([m[0] for m in measurements], np.float64)
    t = np.array([m[1] for m in measurements], np.float64)
    if not np.all(np.isfinite(d)) or not np.all(np.isfinite(t)) or np.any(d < 0):
        raise ValueError("calibrate_alpha_beta: measurements must be finite, sizes >= 0")
    if np.all(d == d[0]):
        raise ValueError("rank-deficient calibration: all message sizes are identical")
    p = float(workers)
    c = 2.0 * (p - 1.0)
    scale = d.max() if d.max() > 0 else 1.0
    A = np.stack([np.full_like(d, c), c * (d / p) / scale], axis=1)
    x, *_ = np.linalg.lstsq(A, t, rcond=None)
    alpha, beta = float(x[0]), float(x[1] / scale)
    clamped = False
    if alpha < 0:
        alpha, clamped = 0.0, True
    if beta < 0:
        beta, clamped = 0.0, True
    return {"alpha": alpha, "beta": beta, "clamped": clamped}


def theoretical_times(t_ff, t_bp, t_rs, t_ag) -> dict:
    """Eq. 7 (DeAR) and Eq. 8 (all-reduce baseline) bounds."""
    for v in (t_ff, t_bp, t_rs, t_ag):
        if not (v >= 0) or not np.isfinite(v):
            raise ValueError("times must be finite and >= 0")
    return {"dear": max(t_ff, t_ag) + max(t_bp, t_rs), "baseline": t_ff + max(t_bp, t_rs + t_ag)}


def max_speedup(t_ff, t_bp, t_rs, t_ag, workers: int) -> float:
    """Eq. 6: S_max = P (t_ff + t_bp) / (max(t_ff, t_ag) + max(t_bp, t_rs))."""
    den = max(t_ff, t_ag) + max(t_bp, t_rs)
    if not den > 0:
        raise ValueError("max_speedup: denominator is zero")
    return workers * (t_ff + t_bp) / den


def exposed_comm(iteration: float, t_ff_total: float, t_bp_total: float) -> float:
    """breakdown (analysis.cpp:85-101): iteration - sum(t_ff) - sum(t_bp), >= 0."""
    return max(0.0, iteration - t_ff_total - t_bp_total)


def partition_plan(layer_bytes, partition_bytes: int):
    """PRIORITY_PARTITION parts (task_graph.cpp:215-258): layer l (L down to 1)
    in ceil(bytes / partition_bytes) parts (one part for an empty layer);
    returns [(layer, parts)] in that order."""
    if partition_bytes <= 0:
        raise ValueError("PRIORITY_PARTITION requires partition_bytes > 0")
    out = []
    for l in range(len(layer_bytes), 0, -1):
        b = int(layer_bytes[l - 1])
        out.append((l, 1 if b == 0 else (b + partition_bytes - 1) // partition_bytes))
    return out


def predict_iteration(layer_bytes, t_ff, t_bp, policy: str, buffer_bytes: int, P: int,
                      alpha: float, beta: float, group_dependency: bool = False,
                      rs_times=None, ag_times=None, partition_bytes: int = 0,
                      negotiation_rounds: int = 1, negotiation_floating: bool = False,
                      ar_times=None) -> dict:
    """Simulated steady-state iteration (seconds) of one worker: BP_L..BP_1 and
    FF_1..FF_L on the compute stream, RS/AG/AR on the comm stream, issue order
    and dependencies of task_graph.cpp:127-210, non-preemptive list
    scheduling by (issue_order, id) as simulate.cpp:65-159.

    rs_times / ag_times (seconds per fusion group, plan order) replace the
    alpha-beta durations, e.g. with the runtime's measured per-bucket stage
    times. Also returns the comm stream's dispatch sequence ("comm_order":
    +g = RS / AR of group g, -g = AG of group g, 1-based), the input of
    Runtime.set_comm_order."""
    L = len(layer_bytes)
    tasks = []  # (kind, subject, duration, deps, order, resource, release, part)

    def add(kind, subj, dur, deps, order, release=0.0, part=0):
        tasks.append([kind, subj, dur, list(deps), order, 0 if kind in ("FF", "BP") else 1,
                      release, part])
        return len(tasks) - 1

    bp, ff, order = [0] * (L + 2), [0] * (L + 2), 0
    for l in range(L, 0, -1):
        bp[l] = add("BP", l, t_bp[l - 1], [bp[l + 1]] if l < L else [], order)
        order += 1
    for l in range(1, L + 1):
        ff[l] = add("FF", l, t_ff[l - 1], [ff[l - 1]] if l > 1 else [], order)
        order += 1
    fused = policy.endswith("_FUSED")
    plan = build_fusion_plan(list(layer_bytes), buffer_bytes if fused else 0)
    gbytes = [sum(layer_bytes[lo - 1:hi]) for lo, hi in plan]
    deps_bp = [[bp[l] for l in range(hi, lo - 1, -1)] for lo, hi in plan]
    order = 0
    part_ids = {}  # PRIORITY_PARTITION: AR task id -> 1-based part bucket (plan order)
    if policy == "PRIORITY_PARTITION":
        # add_priority_partition (task_graph.cpp:215-258): per layer, parts in
        # issue priority (l-1)*stride + k (ascending layer = feed-forward order),
        # each after a negotiation (on the comm stream, or as a release delay
        # when floating).
        parts = partition_plan(layer_bytes, partition_bytes)
        stride = max(n for _, n in parts) + 1
        neg = float(negotiation_rounds) * 2.0 * (float(P) - 1.0) * alpha
        g = 0
        for l, n in parts:
            part_b = float(layer_bytes[l - 1]) / n
            for k in range(n):
                g += 1
                issue = (l - 1) * stride + k
                dur = (ar_times[g - 1] if ar_times is not None
                       else all_reduce_time(part_b, P, alpha, beta))
                if negotiation_floating:
                    t = add("AR", l, dur, [bp[l]], issue, release=neg, part=k + 1)
                else:
                    nt = add("NEGOTIATE", l, neg, [bp[l]], issue, part=k + 1)
                    t = add("AR", l, dur, [nt], issue, part=k + 1)
                part_ids[t] = g
                tasks[ff[l]][3].append(t)
        plan = [(l, l) for l, _ in parts]
    elif policy.startswith("WFBP"):
        for gi, (lo, hi) in enumerate(plan):
            # measured stage times: the all-reduce is RS + AG
            t_ar = (rs_times[gi] + ag_times[gi] if rs_times is not None and ag_times is not None
                    else all_reduce_time(gbytes[gi], P, alpha, beta))
            t = add("AR", gi + 1, t_ar, deps_bp[gi], order)
            order += 1
            for l in range(lo, hi + 1):
                tasks[ff[l]][3].append(t)
    elif policy.startswith("DEAR"):
        rs = []
        for gi in range(len(plan)):
            t_rs = (rs_times[gi] if rs_times is not None
                    else reduce_scatter_time(gbytes[gi], P, alpha, beta))
            rs.append(add("RS", gi + 1, t_rs, deps_bp[gi], order))
            order += 1
        bar = -1
        if not group_dependency:
            bar = add("BARRIER", 0, 0.0, rs, order)
            order += 1
        for gi in range(len(plan) - 1, -1, -1):
            lo, hi = plan[gi]
            t_ag = (ag_times[gi] if ag_times is not None
                    else all_gather_time(gbytes[gi], P, alpha, beta))
            t = add("AG", gi + 1, t_ag, [bar] if bar >= 0 else [rs[gi]], order)
            order += 1
            for l in range(lo, hi + 1):
                tasks[ff[l]][3].append(t)
    else:
        raise ValueError(f"unknown policy {policy!r}")
    n = len(tasks)
    remaining = [len(t[3]) for t in tasks]
    finish = [0.0] * n
    dependents = [[] for _ in range(n)]
    for i, t in enumerate(tasks):
        for d in t[3]:
            dependents[d].append(i)
    ev = [(tasks[i][6], 1, i) for i in range(n) if not tasks[i][3]]
    heapq.heapify(ev)
    ready, running, end_at = [[], []], [-1, -1], [0.0] * n
    done = 0
    dispatched = []
    while ev:
        now = ev[0][0]
        while ev and ev[0][0] == now:
            _, typ, i = heapq.heappop(ev)
            if typ == 0:
                running[tasks[i][5]] = -1
                done += 1
                for j in dependents[i]:
                    finish[j] = max(finish[j], now)
                    remaining[j] -= 1
                    if remaining[j] == 0:
                        heapq.heappush(ev, (finish[j] + tasks[j][6], 1, j))
            else:
                heapq.heappush(ready[tasks[i][5]], (tasks[i][4], i))
        for r in (0, 1):
            if running[r] == -1 and ready[r]:
                _, i = heapq.heappop(ready[r])
                running[r] = i
                if r == 1 and tasks[i][0] == "AR" and part_ids:
                    dispatched.append(part_ids[i])
                elif r == 1 and tasks[i][0] not in ("BARRIER", "NEGOTIATE"):
                    dispatched.append(-tasks[i][1] if tasks[i][0] == "AG" else tasks[i][1])
                end_at[i] = now + tasks[i][2]
                heapq.heappush(ev, (end_at[i], 0, i))
    if done != n:
        raise RuntimeError("simulate: cycle detected")
    it = max(end_at)
    labels = {}
    for i, t in enumerate(tasks):
        if t[0] in ("AR", "NEGOTIATE") and t[7] > 0:
            labels[i] = f"{t[0]} l{t[1]} p{t[7]}"
    return {"iteration_seconds": it, "buckets": len(part_ids) if part_ids else len(plan),
            "start": [end_at[i] - tasks[i][2] for i in range(n)], "part_labels": labels,
            "exposed_comm_seconds": exposed_comm(it, float(sum(t_ff)), float(sum(t_bp))),
            "comm_order": dispatched}
