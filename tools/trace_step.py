#!/usr/bin/env python
"""Measured timeline of one DeAR / WFBP iteration (eager, events per layer),
exported in the reference's Chrome-trace / CSV schema with its invariants
checked (paper_2302_12445_b200.timeline).

    torchrun --nproc-per-node P tools/trace_step.py [--workload bert_large]
        [--policy DEAR_FUSED] [--out profiles/trace]

Rank 0 writes <out>_<policy>_P<P>.json (chrome://tracing) and .csv, and prints
a JSON summary: iteration / FF / BP / exposed-comm ms, per-stage comm totals,
and how long forward layers stalled on their bucket's all-gather.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bert_large")
    ap.add_argument("--policy", default="DEAR_FUSED")
    ap.add_argument("--buffer", type=int, default=25_000_000)
    ap.add_argument("--backend", default="nccl")
    ap.add_argument("--out", default="profiles/trace")
    ap.add_argument("--iters", type=int, default=4)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    import paper_2302_12445_b200 as dear
    from paper_2302_12445_b200 import timeline as T
    from paper_2302_12445_b200.presets import preset_param_counts
    from paper_2302_12445_b200.synthetic import SyntheticModel

    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    lr_ = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(lr_)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", lr_))
        comm = dear.init()
    wl = bench.WORKLOADS[a.workload]
    model = SyntheticModel(preset_param_counts(wl["preset"]), wl["hidden"],
                           wl["batch"] * wl["tokens_per_sample"], seed=1234)
    s = torch.cuda.Stream()
    rt = dear.Runtime(comm, rank, world, policy=a.policy, fusion_buffer_bytes=a.buffer, lr=0.01,
                      backend=a.backend, stream=s)
    for l in range(1, model.L + 1):
        rt.register(l, model.params[l - 1], model.grads[l - 1], model.shadows[l - 1])
    rt.finalize()
    rt.set_timing(True)
    mk = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for it in range(a.iters):
        base = mk()
        evs = []
        with torch.cuda.stream(s):
            base.record(s)
            model.set_input(None)
            for l in range(1, model.L + 1):
                rt.param_wait(l, s)
                e0, e1 = mk(), mk()
                e0.record(s)
                model.forward_layer(l, s)
                e1.record(s)
                evs.append((f"FF l{l}", e0, e1))
            model.zero_grad()
            for l in range(model.L, 0, -1):
                e0, e1 = mk(), mk()
                e0.record(s)
                model.backward_layer(l, s)
                e1.record(s)
                evs.append((f"BP l{l}", e0, e1))
                rt.grad_ready(l, s)
            rt.step(s)
        rt.synchronize()
        torch.cuda.synchronize()
    compute = [(lab, base.elapsed_time(e0), base.elapsed_time(e1)) for lab, e0, e1 in evs]
    # This iteration's all-gathers ran in the NEXT forward; the stamps read now
    # belong to the last completed ones (recorded before this iteration's FF).
    stamps = rt.timeline(base)
    tl = T.build(compute, rt.buckets(), stamps, a.policy)
    rt.close()
    if rank == 0:
        tag = f"{a.out}_{a.workload}_{a.policy}_{a.backend}_P{world}"
        os.makedirs(os.path.dirname(tag) or ".", exist_ok=True)
        with open(tag + ".json", "w") as f:
            f.write(T.dumps(tl))
        with open(tag + ".csv", "w") as f:
            f.write(T.csv(tl))
        comm_tot = {}
        for e in tl["events"]:
            k = e["label"].split()[0]
            comm_tot[k] = comm_tot.get(k, 0.0) + (e["end"] - e["start"])
        ff_first = min(s_ for lab, s_, _ in compute if lab.startswith("FF"))
        bp_first = min(s_ for lab, s_, _ in compute if lab.startswith("BP"))
        ff_span = max(e_ for lab, _, e_ in compute if lab.startswith("FF")) - ff_first
        bp_span = max(e_ for lab, _, e_ in compute if lab.startswith("BP")) - bp_first
        print(json.dumps({"workload": a.workload, "policy": a.policy, "P": world,
                          "iteration_ms": tl["iteration_ms"], "ff_ms": tl["ff_ms"],
                          "bp_ms": tl["bp_ms"], "ff_span_ms": ff_span, "bp_span_ms": bp_span,
                          "ff_stall_ms": ff_span - tl["ff_ms"], "bp_stall_ms": bp_span - tl["bp_ms"],
                          "exposed_comm_ms": tl["exposed_comm_ms"], "stage_totals_ms": comm_tot,
                          "violations": tl["violations"][:5], "trace": tag + ".json"}), flush=True)
    if comm:
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
