#!/usr/bin/env python
"""BASELINE config 5: reduce-scatter / all-gather bucket-size sweep through the
DeAR runtime (in-place NCCL RS/AG of one bucket buffer on the comm stream).

    torchrun --nproc-per-node P tools/sweep_collectives.py [--min-kb 64] [--max-mb 256]

For each bucket size (x2 from 64 KB to 256 MB, fp32) one tensor is registered,
`--reps` DeAR iterations run with comm-stream event timing, and rank 0 prints
one JSON line per size with the median RS / AG time and bus bandwidth
(nccl-tests convention: busbw = (P-1) * slot_bytes / t), plus a final line
with the alpha-beta fit (paper_2302_12445_b200.costmodel.calibrate_alpha_beta,
restating proj/src/cost_model.cpp:79-133) of the measured all-reduce = RS + AG.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-kb", type=int, default=64)
    ap.add_argument("--max-mb", type=int, default=256)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "peer"],
                    help="peer: fused RS+update / AG+unpack NVLink kernels (times include "
                         "the update / unpack they fuse)")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2302_12445_b200 as dear
    from paper_2302_12445_b200.costmodel import calibrate_alpha_beta

    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    comm = dear.init()
    s = torch.cuda.Stream()
    size = a.min_kb * 1024
    points = []
    while size <= a.max_mb * 1024 * 1024:
        n = size // 4
        p = torch.zeros(n, device="cuda")
        g = torch.ones(n, device="cuda")
        rt = dear.Runtime(comm, rank, P, policy="DEAR", lr=0.0, stream=s, backend=a.backend)
        rt.register(1, p, g)
        rt.finalize()
        rt.set_timing(True)
        rs, ag = [], []
        for it in range(a.warmup + a.reps):
            with torch.cuda.stream(s):
                rt.param_wait(1, s)
                rt.grad_ready(1, s)
                rt.step(s)
            rt.synchronize()
            if it >= a.warmup:
                t = rt.timings()[0]
                rs.append(t["rs"])
                ag.append(t["ag"])
        stride = rt.buckets()[0]["slot_stride"]
        rt.close()
        t_rs = torch.tensor([statistics.median(rs)], device="cuda")
        t_ag = torch.tensor([statistics.median(ag)], device="cuda")
        dist.all_reduce(t_rs, op=dist.ReduceOp.MAX)
        dist.all_reduce(t_ag, op=dist.ReduceOp.MAX)
        bus = (P - 1) * stride * 4
        pt = {"backend": a.backend, "bytes": size, "P": P, "rs_ms": t_rs.item(), "ag_ms": t_ag.item(),
              "rs_busbw_gbs": bus / (t_rs.item() / 1e3) / 1e9,
              "ag_busbw_gbs": bus / (t_ag.item() / 1e3) / 1e9}
        points.append(pt)
        if rank == 0:
            print(json.dumps(pt), flush=True)
        size *= 2
    if rank == 0:
        cal = calibrate_alpha_beta([(p["bytes"], (p["rs_ms"] + p["ag_ms"]) / 1e3) for p in points], P)
        print(json.dumps({"backend": a.backend, "calibration": cal, "P": P,
                          "link_GBps_from_beta": (1 / cal["beta"] / 1e9) if cal["beta"] else None}),
              flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
