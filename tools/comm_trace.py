#!/usr/bin/env python
"""Where the zero-copy comm kernels spend their time inside the real step.

    torchrun --nproc-per-node P tools/comm_trace.py [--workload bert_large]
        [--policy DEAR_FUSED] [--compute-only-ref]

Runs the bench step (CUDA graph, default peer transport) and, for one replay,
has every reduce-scatter / all-gather CTA stamp %globaltimer at entry, when
all peers had arrived, and at exit (dear_set_comm_trace). Per launch: wait =
last CTA released - first CTA start (the rank ran ahead of a peer), move =
last CTA end - last CTA released (data movement + update). Rank 0 prints one
JSON line per rank with the sums over the step and the achieved per-launch
NVLink rate of the move phase.
"""
import argparse
import collections
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bert_large")
    ap.add_argument("--policy", default="DEAR_FUSED")
    ap.add_argument("--group-dependency", type=int, default=1)
    ap.add_argument("--buffer", type=int, default=25_000_000)
    a = ap.parse_args()
    import numpy as np
    import torch
    import torch.distributed as dist

    import bench
    import paper_2302_12445_b200 as dear
    from paper_2302_12445_b200._lib import check, lib
    from paper_2302_12445_b200.presets import preset_param_counts
    from paper_2302_12445_b200.synthetic import SyntheticModel

    world, rank = int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0))
    lr = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{lr}"))
    comm = dear.init()
    wl = bench.WORKLOADS[a.workload]
    model = SyntheticModel(preset_param_counts(wl["preset"]), wl["hidden"],
                           wl["batch"] * wl["tokens_per_sample"], seed=1234)
    stream = torch.cuda.Stream()
    ns = argparse.Namespace(group_dependency=a.group_dependency, buffer=a.buffer, lr=0.05,
                            momentum=0.0, backend="auto", contention=1.0, order_search=1)
    rt = bench.make_runtime(ns, model, comm, rank, world, stream, a.policy, True)
    buckets = rt.buckets()
    run = bench.make_runner(bench.Step(model, rt, stream), True, stream)
    ms = bench.time_loop(run, 10, 5, stream, True)
    cap = 1 << 17
    buf = torch.zeros(cap * 5, dtype=torch.int64, device="cuda")  # 40-byte records
    torch.cuda.synchronize()
    dist.barrier()
    check(lib().dear_set_comm_trace(C.c_void_p(buf.data_ptr()), cap))
    run()
    torch.cuda.synchronize()
    n = C.c_int64()
    check(lib().dear_comm_trace_count(C.byref(n)))
    check(lib().dear_set_comm_trace(None, 0))
    recs = buf[: 5 * min(n.value, cap)].cpu().numpy().view(np.uint64).reshape(-1, 5)
    t0, t1, t2 = recs[:, 0].astype(np.int64), recs[:, 1].astype(np.int64), recs[:, 2].astype(np.int64)
    meta = recs[:, 3]
    kind = (meta & 0xffffffff).astype(np.int64)
    tag = (meta >> 32).astype(np.int64)
    launches = collections.defaultdict(list)
    for i in range(len(recs)):
        launches[(int(kind[i]), int(tag[i]))].append(i)
    base = int(t0.min()) if len(recs) else 0
    out = {"rank": rank, "P": world, "workload": a.workload, "policy": a.policy,
           "step_ms": ms, "records": int(n.value), "launches": len(launches)}
    # bytes moved over NVLink per rank and launch ((P-1)/P of the bucket each way)
    bucket_bytes = sorted(b["elems"] * 4 for b in buckets)
    med_bytes = bucket_bytes[len(bucket_bytes) // 2] if bucket_bytes else 0
    for k, name in ((0, "rs"), (1, "ag")):
        rows = [v for (kk, _), v in launches.items() if kk == k]
        waits, moves, spans, starts = [], [], [], []
        for idx in rows:
            first = t0[idx].min()
            released = t1[idx].max()
            end = t2[idx].max()
            waits.append((released - first) / 1e3)
            moves.append((end - released) / 1e3)
            spans.append((end - first) / 1e3)
            starts.append((first - base) / 1e3)
        if not rows:
            continue
        out[name] = {"launches": len(rows), "wait_us_sum": float(np.sum(waits)),
                     "move_us_sum": float(np.sum(moves)), "span_us_sum": float(np.sum(spans)),
                     "wait_us_median": float(np.median(waits)),
                     "move_us_median": float(np.median(moves)),
                     "move_gbs_median": (world - 1) / world * med_bytes /
                     (np.median(moves) * 1e-6) / 1e9 if np.median(moves) > 0 else None,
                     "first_start_us": float(min(starts)), "last_start_us": float(max(starts))}
    allout = [None] * world
    dist.all_gather_object(allout, out)
    if rank == 0:
        for o in allout:
            print(json.dumps(o), flush=True)
    rt.synchronize()
    rt.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
