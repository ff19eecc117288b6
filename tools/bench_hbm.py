#!/usr/bin/env python
"""Isolated timing of the DeAR bucket kernels (pack / update / unpack) on one
GPU: the runtime drives backprop-without-compute iterations (all gradients
reported back to back), so the comm stream runs the HBM-bound kernels alone.

    python tools/bench_hbm.py [--workload resnet50] [--iters 20] [--momentum 0.9]

Prints one JSON line: per stage total ms per iteration, algorithmic bytes
(pack 8 B/elem, update 12 B/shard-elem or 20 with momentum, unpack 8 B/elem
+ 2 B/elem for the bf16 copy) and GB/s vs MEASURED_PEAKS.json hbm_gbs.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--buffer", type=int, default=25_000_000)
    ap.add_argument("--momentum", type=float, default=0.0)
    ap.add_argument("--no-shadow", action="store_true")
    a = ap.parse_args()
    import torch

    # keep the separate pack / update / unpack kernels at P = 1 (not the fused
    # direct update), which is what every P > 1 bucket runs
    os.environ.setdefault("DEAR_DIRECT", "0")
    import paper_2302_12445_b200 as dear
    from paper_2302_12445_b200.presets import preset_param_counts

    counts = preset_param_counts(a.workload)
    dev = torch.device("cuda")
    off, offs = 0, []
    for n in counts:
        offs.append(off)
        off += (n + 63) // 64 * 64
    params = torch.randn(off, device=dev) * 0.01
    grads = torch.randn(off, device=dev) * 0.01
    shadow = torch.zeros(off, device=dev, dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    rt = dear.Runtime(None, 0, 1, policy="DEAR_FUSED", fusion_buffer_bytes=a.buffer, lr=1e-3,
                      momentum=a.momentum, stream=s)
    for l, (o, n) in enumerate(zip(offs, counts), start=1):
        rt.register(l, params[o:o + n], grads[o:o + n],
                    None if a.no_shadow else shadow[o:o + n])
    rt.finalize()
    buckets = rt.buckets()
    rt.set_timing(True)
    tot = {"pack": 0.0, "update": 0.0, "unpack": 0.0}
    for it in range(a.iters + 2):
        with torch.cuda.stream(s):
            for l in range(1, len(counts) + 1):
                rt.param_wait(l, s)
            for l in range(len(counts), 0, -1):
                rt.grad_ready(l, s)
            rt.step(s)
        rt.synchronize()
        if it >= 2:
            for st in rt.timings():
                for k in tot:
                    if st[k] is not None:
                        tot[k] += st[k]
    D = sum(counts)
    shard = sum(b["slot_stride"] for b in buckets)
    nbytes = {"pack": 8 * D, "update": (20 if a.momentum else 12) * shard,
              "unpack": (8 if a.no_shadow else 10) * D}
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    out = {"workload": a.workload, "buckets": len(buckets), "elems": D}
    for k in tot:
        ms = tot[k] / a.iters
        gbs = nbytes[k] / (ms / 1e3) / 1e9
        out[k] = {"ms_per_iter": ms, "bytes": nbytes[k], "gbs": gbs, "frac_of_measured_hbm": gbs / peak}
    print(json.dumps(out), flush=True)
    rt.close()


if __name__ == "__main__":
    main()
