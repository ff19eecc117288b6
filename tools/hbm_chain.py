#!/usr/bin/env python
"""Graph-chained timing of the bucket kernels (pack / update / unpack /
direct) at P = 1 — bench.py's hbm_kernels measurement on its own, for kernel
A/B builds (DEAR_LIB=libdear_<variant>.so).

    python tools/hbm_chain.py [--workload resnet50|bert_large] [--reps 20]
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
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch

    import bench
    import paper_2302_12445_b200 as dear
    from paper_2302_12445_b200.presets import preset_param_counts

    counts = preset_param_counts(a.workload)
    off, offs = 0, []
    for n in counts:
        offs.append(off)
        off += (n + 63) // 64 * 64

    class M:  # the bits of SyntheticModel _isolated_stage_times touches
        params_flat = torch.rand(off, device="cuda") * 0.02 - 0.01
        grads_flat = torch.rand(off, device="cuda") * 0.02 - 0.01
    shadow = torch.zeros(off, device="cuda", dtype=torch.bfloat16)
    stream = torch.cuda.Stream()

    def runtime(policy):
        rt = dear.Runtime(None, 0, 1, policy=policy, fusion_buffer_bytes=25_000_000, lr=1e-3,
                          stream=stream)
        for l, (o, n) in enumerate(zip(offs, counts), start=1):
            rt.register(l, M.params_flat[o:o + n], M.grads_flat[o:o + n], shadow[o:o + n])
        rt.finalize()
        return rt

    iso = bench._isolated_stage_times(M, runtime, stream, "DEAR_FUSED", reps=a.reps)
    hbm = bench.peaks()[0]
    D = sum(counts)
    rt = runtime("DEAR_FUSED")
    shard = sum(b["slot_stride"] for b in rt.buckets())
    rt.close()
    nbytes = {"pack": 8 * D, "update": 12 * shard, "unpack": 10 * D, "direct": 14 * D}
    out = {"workload": a.workload, "lib": os.environ.get("DEAR_LIB", "libdear.so")}
    for k, (ms, nl) in iso.items():
        out[k] = {"us_per_launch": round(1e3 * ms / nl, 2),
                  "frac": round(nbytes[k] / (ms / 1e3) / 1e9 / hbm, 3)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
