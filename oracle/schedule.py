"""TEST INFRASTRUCTURE ONLY — restatement of the reference's schedule rules.

Pure-Python (small integer/ordering work) restatement of
  * GraphBuilder::add_compute_chains  (task_graph.cpp:127-146)
  * GraphBuilder::add_wfbp            (task_graph.cpp:163-176)
  * GraphBuilder::add_dear            (task_graph.cpp:181-210)
  * task_label                        (task_graph.cpp:51-58)
  * simulate                          (simulate.cpp:65-159): one Compute and one
    Comm stream, non-preemptive, ready set ordered by (issue_order, id),
    completions processed before readiness at equal times.
  * reduce/all-gather/all-reduce time (cost_model.cpp:34-48)
It is pinned against oracle/_ref's build_graph+simulate on golden fixtures
(tests/golden/schedules.json) and the reference's golden traces
(test_simulate.cpp:52-110). PRIORITY_PARTITION is out of scope.

It is the checker for the runtime's collective issue order: the order in
which the runtime enqueues RS/AG/AR on its comm stream must equal the order
in which this simulator dispatches them on the Comm resource.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field

FF, BP, RS, AG, AR, BARRIER = "FF", "BP", "RS", "AG", "AR", "BARRIER"
COMPUTE, COMM = 0, 1


@dataclass
class Task:
    id: int
    kind: str
    subject: int
    group_subject: bool
    duration: float
    deps: list = field(default_factory=list)
    issue_order: int = 0

    @property
    def resource(self) -> int:
        return COMPUTE if self.kind in (FF, BP) else COMM

    @property
    def label(self) -> str:
        if self.kind == BARRIER:
            return "BARRIER"
        return f"{self.kind} {'g' if self.group_subject else 'l'}{self.subject}"


def rs_time(nbytes: float, P: int, alpha: float, beta: float) -> float:
    return (P - 1.0) * (alpha + (nbytes / P) * beta)


def ar_time(nbytes: float, P: int, alpha: float, beta: float) -> float:
    return rs_time(nbytes, P, alpha, beta) + rs_time(nbytes, P, alpha, beta)


def fusion_plan(layer_bytes, buffer_bytes: int):
    """build_fusion_plan / per_layer_plan (fusion.cpp:29-70)."""
    L = len(layer_bytes)
    if L == 0:
        raise ValueError("build_fusion_plan: empty model")
    if buffer_bytes == 0:
        return [(l, l) for l in range(L, 0, -1)]
    groups, high, acc = [], L, layer_bytes[L - 1]
    for l in range(L - 1, 0, -1):
        nxt = layer_bytes[l - 1]
        if acc + nxt <= buffer_bytes:
            acc += nxt
        else:
            groups.append((l + 1, high))
            high, acc = l, nxt
    groups.append((1, high))
    return groups


def build_graph(layer_bytes, t_ff, t_bp, policy: str, buffer_bytes: int = 0,
                group_dependency: bool = False, P: int = 2, alpha: float = 0.0,
                beta: float = 0.0):
    L = len(layer_bytes)
    tasks: list[Task] = []

    def add(kind, subject, group_subject, duration, deps, order):
        tasks.append(Task(len(tasks), kind, subject, group_subject, duration, list(deps), order))
        return tasks[-1].id

    bp_id, ff_id, order = [0] * (L + 1), [0] * (L + 1), 0
    for l in range(L, 0, -1):
        bp_id[l] = add(BP, l, False, t_bp[l - 1], [bp_id[l + 1]] if l < L else [], order)
        order += 1
    for l in range(1, L + 1):
        ff_id[l] = add(FF, l, False, t_ff[l - 1], [ff_id[l - 1]] if l > 1 else [], order)
        order += 1

    fused = policy in ("WFBP_FUSED", "DEAR_FUSED")
    plan = fusion_plan(layer_bytes, buffer_bytes if fused else 0)
    gbytes = [sum(layer_bytes[lo - 1:hi]) for lo, hi in plan]
    bp_deps = [[bp_id[l] for l in range(hi, lo - 1, -1)] for lo, hi in plan]
    order = 0
    if policy in ("WFBP", "WFBP_FUSED"):
        for gi, (lo, hi) in enumerate(plan):
            subj = gi + 1 if fused else hi
            tid = add(AR, subj, fused, ar_time(gbytes[gi], P, alpha, beta), bp_deps[gi], order)
            order += 1
            for l in range(lo, hi + 1):
                tasks[ff_id[l]].deps.append(tid)
    elif policy in ("DEAR", "DEAR_FUSED"):
        rs_ids = []
        for gi in range(len(plan)):
            rs_ids.append(add(RS, gi + 1, True, rs_time(gbytes[gi], P, alpha, beta),
                              bp_deps[gi], order))
            order += 1
        barrier = -1
        if not group_dependency:
            barrier = add(BARRIER, 0, False, 0.0, rs_ids, order)
            order += 1
        for gi in range(len(plan) - 1, -1, -1):
            lo, hi = plan[gi]
            dep = [barrier] if barrier >= 0 else [rs_ids[gi]]
            tid = add(AG, gi + 1, True, rs_time(gbytes[gi], P, alpha, beta), dep, order)
            order += 1
            for l in range(lo, hi + 1):
                tasks[ff_id[l]].deps.append(tid)
    else:
        raise ValueError(f"policy {policy!r} out of scope")
    return tasks, plan


def simulate(tasks):
    """Two-stream list scheduler; returns {task id: (start, end)}, makespan."""
    n = len(tasks)
    remaining = [len(t.deps) for t in tasks]
    dep_finish = [0.0] * n
    dependents = [[] for _ in range(n)]
    for t in tasks:
        for d in t.deps:
            dependents[d].append(t.id)
    events = []  # (time, type 0=complete 1=ready, task)
    for t in tasks:
        if not t.deps:
            heapq.heappush(events, (0.0, 1, t.id))
    ready = [[], []]  # heaps of (issue_order, id)
    running = [-1, -1]
    span = {}
    while events:
        now = events[0][0]
        while events and events[0][0] == now:
            _, typ, tid = heapq.heappop(events)
            if typ == 0:
                running[tasks[tid].resource] = -1
                for nx in dependents[tid]:
                    dep_finish[nx] = max(dep_finish[nx], now)
                    remaining[nx] -= 1
                    if remaining[nx] == 0:
                        heapq.heappush(events, (dep_finish[nx], 1, nx))
            else:
                heapq.heappush(ready[tasks[tid].resource], (tasks[tid].issue_order, tid))
        for r in (0, 1):
            if running[r] != -1 or not ready[r]:
                continue
            _, tid = heapq.heappop(ready[r])
            end = now + tasks[tid].duration
            running[r] = tid
            span[tid] = (now, end)
            heapq.heappush(events, (end, 0, tid))
    if len(span) != n:
        raise RuntimeError("simulate: cycle detected")
    return span, max(e for _, e in span.values())


def comm_dispatch_order(tasks, span):
    """Labels of Comm-resource tasks (excluding the zero-length BARRIER) in the
    order the simulator dispatches them — the runtime's enqueue contract."""
    comm = [t for t in tasks if t.resource == COMM and t.kind != BARRIER]
    comm.sort(key=lambda t: (span[t.id][0], t.issue_order, t.id))
    return [t.label for t in comm]
