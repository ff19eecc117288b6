#!/usr/bin/env python
"""BASELINE config 3: DeAR vs WFBP (same kernels) across fusion-buffer sizes.

    torchrun --nproc-per-node P tools/sweep_buffers.py [--workload bert_base]
        [--buffers-mb 0,1,2,5,10,25,50,100] [--backend nccl|peer]

buffer 0 = per-layer (unfused DEAR vs WFBP). Every point: CUDA-graph replay of
one training iteration over the synthetic preset-shaped layers (bench.py's
step), --steps timed after --warmup; max over ranks. Rank 0 prints one JSON
line per buffer, and a summary line with the best buffer for each policy.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bert_base")
    ap.add_argument("--buffers-mb", default="0,1,2,5,10,25,50,100")
    ap.add_argument("--backend", default="nccl")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--batch", type=int, default=0)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    import paper_2302_12445_b200 as dear
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
    batch = a.batch or wl["batch"]
    model = SyntheticModel(preset_param_counts(wl["preset"]), wl["hidden"],
                           batch * wl["tokens_per_sample"], seed=1234)
    stream = torch.cuda.Stream()
    # compute-only reference (same kernels, no runtime)
    run = bench.make_runner(bench.Step(model, None, stream), True, stream)
    t_comp = bench.time_loop(run, a.steps, a.warmup, stream, world > 1)
    results = []
    for mb in [float(x) for x in a.buffers_mb.split(",")]:
        buf = int(mb * 1e6)
        row = {"workload": a.workload, "P": world, "buffer_mb": mb, "backend": a.backend,
               "compute_only_ms": t_comp}
        for pol in ("DEAR", "WFBP"):
            policy = pol + ("_FUSED" if buf > 0 else "")
            rt = dear.Runtime(comm, rank, world, policy=policy, fusion_buffer_bytes=buf,
                              lr=0.01, defer_allgather=True, backend=a.backend, stream=stream)
            for l in range(1, model.L + 1):
                rt.register(l, model.params[l - 1], model.grads[l - 1], model.shadows[l - 1])
            rt.finalize()
            run = bench.make_runner(bench.Step(model, rt, stream), True, stream)
            ms = bench.time_loop(run, a.steps, a.warmup, stream, world > 1)
            rt.synchronize()
            row[pol.lower() + "_ms"] = ms
            row[pol.lower() + "_samples_per_s"] = batch * world / (ms / 1e3)
            row["buckets"] = len(rt.buckets())
            rt.close()
        row["dear_over_wfbp"] = row["wfbp_ms"] / row["dear_ms"]
        row["dear_exposed_pct"] = max(0.0, 100 * (row["dear_ms"] - t_comp) / row["dear_ms"])
        row["wfbp_exposed_pct"] = max(0.0, 100 * (row["wfbp_ms"] - t_comp) / row["wfbp_ms"])
        results.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)
    if rank == 0:
        bd = min(results, key=lambda r: r["dear_ms"])
        bw = min(results, key=lambda r: r["wfbp_ms"])
        print(json.dumps({"summary": True, "best_dear_buffer_mb": bd["buffer_mb"],
                          "best_dear_ms": bd["dear_ms"], "best_wfbp_buffer_mb": bw["buffer_mb"],
                          "best_wfbp_ms": bw["wfbp_ms"],
                          "best_vs_best": bw["wfbp_ms"] / bd["dear_ms"]}), flush=True)
    if comm:
        comm.close()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
