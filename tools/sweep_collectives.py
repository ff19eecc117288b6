#!/usr/bin/env python
"""BASELINE config 5: reduce-scatter / all-gather bucket-size sweep through the
DeAR runtime, per collective transport:

  nccl  in-place ncclReduceScatter / ncclAllGather of one bucket buffer (the
        pack / update / unpack kernels around them timed separately)
  zc    zero-copy NVLink peer kernels (RS pulls every rank's gradients, sums
        in ring order and applies the update; AG pulls the owners' parameters)
  slot  peer kernels over IPC-mapped bucket slots (pack, RS+update, AG+unpack)
  nvls  NVLink SHARP: multimem.ld_reduce RS+update, multicast-store AG
  push  zero-copy with the push reduce-scatter (DEAR_PUSH_RS=1): pack writes
        each chunk into its owner's slot over NVLink, the owner sums locally

    torchrun --nproc-per-node P tools/sweep_collectives.py [--backends nccl,zc,slot,nvls]
        [--min-kb 64] [--max-mb 256]

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
    ap.add_argument("--backends", default="nccl,zc,slot,nvls,push")
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
    maxn = a.max_mb * 1024 * 1024 // 4
    heap = None
    for backend in a.backends.split(","):
        if backend == "nvls":
            if not dear.nvls_supported():
                if rank == 0:
                    print(json.dumps({"backend": "nvls", "unavailable": "no multicast support"}))
                continue
            if heap is None:
                heap = dear.SymmetricHeap(2 * 4 * maxn + (1 << 20))
                hp, hg = heap.tensor(maxn), heap.tensor(maxn)
            pbuf, gbuf = hp, hg
        else:
            pbuf = torch.zeros(maxn, device="cuda")
            gbuf = torch.zeros(maxn, device="cuda")
        os.environ["DEAR_ZERO_COPY"] = "0" if backend == "slot" else "1"
        os.environ["DEAR_PUSH_RS"] = "1" if backend == "push" else "0"
        rt_backend = {"zc": "peer", "slot": "peer", "push": "peer"}.get(backend, backend)
        size = a.min_kb * 1024
        points = []
        while size <= a.max_mb * 1024 * 1024:
            n = size // 4
            p, g = pbuf[:n], gbuf[:n]
            p.zero_()
            g.fill_(1.0)
            rt = dear.Runtime(comm, rank, P, policy="DEAR", lr=0.0, stream=s, backend=rt_backend,
                              heap=heap if backend == "nvls" else None)
            rt.register(1, p, g)
            rt.finalize()
            if backend in ("zc", "slot", "push"):
                assert rt.zero_copy == (backend != "slot"), backend
                assert rt.push_rs == (backend == "push"), backend
            rt.set_timing(True)
            st = {k: [] for k in ("pack", "rs", "update", "ag", "unpack")}
            for it in range(a.warmup + a.reps):
                with torch.cuda.stream(s):
                    rt.param_wait(1, s)
                    rt.grad_ready(1, s)
                    rt.step(s)
                rt.synchronize()
                if it >= a.warmup:
                    t = rt.timings()[0]
                    for k in st:
                        if t[k] is not None:
                            st[k].append(t[k])
            stride = rt.buckets()[0]["slot_stride"]
            rt.close()
            med = torch.tensor([statistics.median(st[k]) if st[k] else 0.0 for k in st],
                               device="cuda")
            dist.all_reduce(med, op=dist.ReduceOp.MAX)
            m = dict(zip(st, med.tolist()))
            if backend == "push":  # the pack moves the data over NVLink
                m["rs"] += m["pack"]
            bus = (P - 1) * stride * 4
            pt = {"backend": backend, "bytes": size, "P": P, "rs_ms": m["rs"], "ag_ms": m["ag"],
                  "pack_ms": m["pack"], "update_ms": m["update"], "unpack_ms": m["unpack"],
                  "rs_busbw_gbs": bus / (m["rs"] / 1e3) / 1e9 if m["rs"] else None,
                  "ag_busbw_gbs": bus / (m["ag"] / 1e3) / 1e9 if m["ag"] else None,
                  "note": {"nccl": "rs/ag: the NCCL calls alone",
                           "zc": "rs: fused RS+update kernel; ag: pull all-gather kernel",
                           "slot": "rs: fused RS+update after pack; ag: fused AG+unpack",
                           "nvls": "rs: multimem.ld_reduce RS+update; ag: multicast-store "
                                   "broadcast + arrival wait",
                           "push": "rs: pack (posted stores into the owners' slots) + local "
                                   "ring-order sum + update; ag: pull all-gather"}[backend]}
            points.append(pt)
            if rank == 0:
                print(json.dumps(pt), flush=True)
            size *= 2
        if rank == 0:
            cal = calibrate_alpha_beta([(q["bytes"], (q["rs_ms"] + q["ag_ms"]) / 1e3)
                                        for q in points], P)
            print(json.dumps({"backend": backend, "calibration": cal, "P": P,
                              "link_GBps_from_beta": (1 / cal["beta"] / 1e9) if cal["beta"]
                              else None}), flush=True)
        del pbuf, gbuf
        torch.cuda.empty_cache()
    if heap is not None:
        heap.close()
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
