"""Shared test harness: drive the DeAR runtime on seeded inputs and compute the
oracle's expectation for the same inputs (tests only)."""
from __future__ import annotations

import numpy as np

from oracle.lib import Restated
from oracle.schedule import fusion_plan


def bucket_plan(numels, policy: str, buffer_bytes: int):
    fused = "FUSED" in policy
    return fusion_plan([4 * n for n in numels], buffer_bytes if fused else 0)


def bucket_ranges(o: Restated, numels, policy: str, buffer_bytes: int, partition_bytes: int = 0):
    """Flat element ranges [a, b) of the buckets, plan order. PRIORITY_PARTITION:
    every layer (L down to 1) in ceil(bytes / partition_bytes) balanced parts
    (task_graph.cpp:215-258; the split follows chunk_ranges)."""
    offs = np.concatenate([[0], np.cumsum(numels)]).astype(np.int64)
    if policy == "PRIORITY_PARTITION":
        out = []
        for l in range(len(numels), 0, -1):
            n = int(numels[l - 1])
            parts = 1 if n == 0 else (4 * n + partition_bytes - 1) // partition_bytes
            b = o.chunk_ranges(n, parts)
            out += [(int(offs[l - 1] + b[k]), int(offs[l - 1] + b[k + 1])) for k in range(parts)]
        return out
    return [(int(offs[lo - 1]), int(offs[hi])) for lo, hi in bucket_plan(numels, policy,
                                                                           buffer_bytes)]


def seeded_grads(o: Restated, P: int, numels, step: int, seed0: int = 1000) -> np.ndarray:
    """Rank-major [P, D] fp32 gradients, U(-1,1) from the reference tests'
    generator (mt19937_64 + uniform_real_distribution), one seed per step."""
    D = int(sum(numels))
    return o.random_vectors(P, D, seed0 + step).astype(np.float32)


def initial_weights(o: Restated, numels, seed: int = 77) -> np.ndarray:
    D = int(sum(numels))
    return o.random_vectors(1, D, seed)[0].astype(np.float32)


def oracle_run(o: Restated, numels, P: int, steps: int, policy: str, buffer_bytes: int,
               lr: float, momentum=0.0, dampening=0.0, weight_decay=0.0, nesterov=False,
               f32: bool = True, seed0: int = 1000, wseed: int = 77, w0=None, grads_fn=None,
               lr_schedule=None, partition_bytes: int = 0):
    """Apply the oracle's S-SGD step per fusion bucket (chunk layout is per
    bucket), for `steps` steps. f32=True uses the fp32 ring-order
    restatement (bit-exact target for the local group); f32=False the fp64
    restatement of collective.cpp (tolerance target)."""
    offs = np.concatenate([[0], np.cumsum(numels)]).astype(np.int64)
    w = initial_weights(o, numels, wseed) if w0 is None else w0
    w = np.array(w, dtype=np.float32 if f32 else np.float64)
    bufs = {}
    ranges = bucket_ranges(o, numels, policy, buffer_bytes, partition_bytes)
    prescale = (P & (P - 1)) == 0
    for s in range(steps):
        g = grads_fn(s) if grads_fn is not None else seeded_grads(o, P, numels, s, seed0)
        if lr_schedule is not None:
            lr = lr_schedule[s]
        for a, b in ranges:
            if b == a:
                continue
            gb = g[:, a:b]
            key = (a, b)
            if f32:
                buf, has = bufs.get(key, (np.zeros(b - a, np.float32), False))
                nw, nbuf, nhas = o.sgd_step_f32(w[a:b], buf, has, gb, lr, momentum, dampening,
                                                weight_decay, nesterov, prescale)
            else:
                buf, has = bufs.get(key, (np.zeros(b - a, np.float64), False))
                if momentum == 0.0 and weight_decay == 0.0:
                    nw = o.sgd_step(w[a:b], gb.astype(np.float64), lr)
                    nbuf, nhas = buf, has
                else:
                    nw, nbuf, nhas = o.sgd_step_momentum(w[a:b], buf, has, gb.astype(np.float64),
                                                         lr, momentum, dampening, weight_decay,
                                                         nesterov)
            w[a:b] = nw
            bufs[key] = (nbuf, nhas)
    return w


def run_local(numels, P: int, steps: int, policy: str, buffer_bytes: int, lr: float,
              momentum=0.0, dampening=0.0, weight_decay=0.0, nesterov=False,
              defer_allgather=False, seed0: int = 1000, wseed: int = 77, shadow: bool = False,
              comm_order=None, transport: str = "ring", flat: bool = False,
              zero_copy: bool = True, w0=None, grads_fn=None, lr_schedule=None,
              partition_bytes: int = 0):
    """Drive P local-group ranks in lock-step through `steps` iterations of
    backward (layers L..1) + step + forward waits. Returns (params [P, D],
    shadows or None, traces, runtimes-closed).

    transport="ring": ring-order emulation kernels; "peer": the multi-GPU
    NVLink peer kernels on one device (each rank on its own stream). flat=True
    lays every rank's parameters / gradients out as 64-element aligned views
    of one tensor each (the zero-copy peer layout). w0: initial fp32 weights
    (default: the seeded generator); grads_fn(step) -> [P, D] fp32 gradients
    (default: seeded_grads). lr_schedule: per-step learning rates (set_lr
    before each step's backward)."""
    import torch

    from paper_2302_12445_b200 import LocalGroup, Runtime

    o = Restated()
    dev = torch.device("cuda")
    L = len(numels)
    offs = np.concatenate([[0], np.cumsum(numels)]).astype(np.int64)
    if w0 is None:
        w0 = initial_weights(o, numels, wseed)
    group = LocalGroup(P, transport)
    peer = transport == "peer"
    streams = [torch.cuda.Stream() for _ in range(P)] if peer else [None] * P
    rts, params, grads, shadows = [], [], [], []
    aoffs = [0]
    for n in numels:
        aoffs.append(aoffs[-1] + (n + 63) // 64 * 64)
    for r in range(P):
        rt = Runtime(group, r, P, policy=policy, fusion_buffer_bytes=buffer_bytes, lr=lr,
                     momentum=momentum, dampening=dampening, weight_decay=weight_decay,
                     nesterov=nesterov, defer_allgather=defer_allgather,
                     dear_group_dependency=comm_order is not None and policy.startswith("DEAR"),
                     stream=streams[r], partition_bytes=partition_bytes)
        ps, gs, ss = [], [], []
        if flat:
            pflat = torch.zeros(aoffs[-1] + 64, device=dev)
            gflat = torch.zeros_like(pflat)
        for l in range(1, L + 1):
            a, b = offs[l - 1], offs[l]
            src = torch.from_numpy(np.ascontiguousarray(w0[a:b], np.float32)).to(dev)
            if flat:
                p = pflat[aoffs[l - 1]:aoffs[l - 1] + (b - a)]
                p.copy_(src)
                g = gflat[aoffs[l - 1]:aoffs[l - 1] + (b - a)]
            else:
                p, g = src, torch.zeros_like(src)
            sh = torch.zeros(max(b - a, 1), dtype=torch.bfloat16, device=dev) if shadow else None
            rt.register(l, p, g, sh)
            ps.append(p)
            gs.append(g)
            ss.append(sh)
        rts.append(rt)
        params.append(ps)
        grads.append(gs)
        shadows.append(ss)
    torch.cuda.synchronize()
    for rt in rts:
        rt.finalize()
        if comm_order is not None:
            rt.set_comm_order(comm_order)
    if peer:
        group.connect(zero_copy)
    traces = []
    for s in range(steps):
        G = grads_fn(s) if grads_fn is not None else seeded_grads(o, P, numels, s, seed0)
        if lr_schedule is not None:
            for rt in rts:
                rt.set_lr(lr_schedule[s])
        # forward of iteration s: wait for each layer's bucket (flushes AGs)
        for l in range(1, L + 1):
            for r in range(P):
                rts[r].param_wait(l, streams[r])
        for l in range(L, 0, -1):
            a, b = offs[l - 1], offs[l]
            for r in range(P):
                with torch.cuda.stream(streams[r] or torch.cuda.current_stream()):
                    grads[r][l - 1].copy_(torch.from_numpy(np.ascontiguousarray(G[r, a:b])).to(dev))
                rts[r].grad_ready(l, streams[r])
        for r in range(P):
            rts[r].step(streams[r])
        traces.append([rt.trace() for rt in rts])
    for rt in rts:
        rt.synchronize()
    torch.cuda.synchronize()
    out = np.stack([np.concatenate([p.cpu().numpy() for p in params[r]]) if L else np.zeros(0)
                    for r in range(P)])
    sh_out = None
    if shadow:
        sh_out = np.stack([np.concatenate([s[: numels[i]].float().cpu().numpy()
                                           for i, s in enumerate(shadows[r])]) for r in range(P)])
    same = [rt.check_replicas() for rt in rts]
    run_local.zero_copy = [rt.zero_copy for rt in rts]
    for rt in rts:
        rt.close()
    group.close()
    return out, sh_out, traces, same
