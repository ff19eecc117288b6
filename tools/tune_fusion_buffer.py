#!/usr/bin/env python
"""DeAR-BO on the live B200 step: the reference's GP +
expected-improvement tuner (paper_2302_12445_b200.tuner, pinned to
proj/src/{gp,tuner}.cpp) picks fusion-buffer sizes; each trial builds the
runtime at that size and times graph-replayed steps of the synthetic model.

    torchrun --nproc-per-node P tools/tune_fusion_buffer.py [--workload bert_base]
        [--policy DEAR_FUSED] [--trials 10] [--backend auto]

The objective (samples/s) is the max-over-ranks step time, so every rank's GP
sees identical observations and proposes identical trials. Rank 0 prints one
JSON line: the trial trace, the best buffer and the 25 MB default for comparison.
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bert_base")
    ap.add_argument("--policy", default="DEAR_FUSED")
    ap.add_argument("--trials", type=int, default=10)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--backend", default="auto")
    ap.add_argument("--group-dependency", type=int, default=0)
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    import paper_2302_12445_b200 as dear
    from paper_2302_12445_b200 import tuner
    from paper_2302_12445_b200.presets import preset_param_counts
    from paper_2302_12445_b200.synthetic import SyntheticModel

    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    lr_ = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(lr_)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{lr_}"))
        comm = dear.init()
    wl = bench.WORKLOADS[a.workload]
    batch = wl["batch"]
    model = SyntheticModel(preset_param_counts(wl["preset"]), wl["hidden"],
                           batch * wl["tokens_per_sample"], seed=1234)
    stream = torch.cuda.Stream()

    def measure(buffer_bytes, policy=a.policy):
        ns = argparse.Namespace(group_dependency=a.group_dependency, buffer=int(buffer_bytes),
                                lr=0.05, momentum=0.0, backend=a.backend, contention=1.0,
                                order_search=0)
        rt = bench.make_runtime(ns, model, comm, rank, world, stream, policy, True)
        run = bench.make_runner(bench.Step(model, rt, stream), True, stream)
        ms = bench.time_loop(run, a.steps, 3, stream, world > 1)
        rt.synchronize()
        rt.close()
        del run
        return batch * world / (ms / 1e3), ms

    evals = []

    def objective(b):
        sps, ms = measure(b)
        evals.append({"buffer_bytes": int(b), "samples_per_s": sps, "ms": ms})
        return sps

    cfg = tuner.TunerConfig(lower_bytes=1e6, upper_bytes=1e8, init_buffer_bytes=2.5e7,
                            measure_steps=1, max_trials=a.trials)
    res = tuner.tune(objective, cfg)
    wfbp_sps, wfbp_ms = measure(res["best_buffer_bytes"], "WFBP_FUSED")
    wfbp25_sps, wfbp25_ms = measure(25_000_000, "WFBP_FUSED")
    out = {"workload": wl["config"], "P": world, "policy": a.policy,
           "backend": a.backend, "group_dependency": a.group_dependency,
           "best_buffer_bytes": res["best_buffer_bytes"],
           "best_samples_per_s": res["best_throughput"],
           "default_25MB": evals[0],
           "wfbp_at_best_buffer": {"samples_per_s": wfbp_sps, "ms": wfbp_ms},
           "wfbp_at_25MB": {"samples_per_s": wfbp25_sps, "ms": wfbp25_ms},
           "trials": evals}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
