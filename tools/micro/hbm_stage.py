#!/usr/bin/env python
"""Bucket-kernel HBM fractions (pack / update / unpack / direct) on one GPU,
as bench.py's `hbm_kernels` block measures them, for A/B of build variants:

    DEAR_LIB=libdear_x.so python tools/micro/hbm_stage.py [--workload resnet50]

Best of 3 rounds of `reps` graph-replayed launches per stage.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--align4", action="store_true",
                    help="round every tensor to a multiple of 4 elements (every layer "
                         "starts 16 B aligned in its bucket: no realignment)")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2302_12445_b200.presets import preset_param_counts
    from paper_2302_12445_b200.synthetic import SyntheticModel

    torch.cuda.set_device(0)
    wl = bench.WORKLOADS[a.workload]
    counts = preset_param_counts(wl["preset"])
    if a.align4:
        counts = [(c + 3) // 4 * 4 for c in counts]
    model = SyntheticModel(counts, wl["hidden"], wl["batch"] * wl["tokens_per_sample"], seed=1)
    stream = torch.cuda.Stream()
    ns = argparse.Namespace(group_dependency=0, buffer=25_000_000, lr=0.05, momentum=0.0,
                            backend="auto", contention=1.0, order_search=0)
    runtime = lambda pol: bench.make_runtime(ns, model, None, 0, 1, stream, pol, True)  # noqa: E731
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    D = sum(counts)
    elem_bytes = {"pack": 8 * D, "update": 12 * D, "unpack": 10 * D, "direct": 14 * D}
    res = {}
    for rep in range(3):
        iso = bench._isolated_stage_times(model, runtime, stream, "DEAR_FUSED", reps=a.reps)
        for k, (t, nl) in iso.items():
            res.setdefault(k, []).append(elem_bytes[k] / (t / 1e3) / 1e9)
    # Calibration: torch's own device copy (dst.copy_(src), 8 B per element)
    # over the same five bucket-sized buffers, graph-replayed the same way.
    nb = 5
    n = D // nb
    src = [torch.randn(n, device="cuda") for _ in range(nb)]
    dst = [torch.empty_like(x) for x in src]
    for name, op in (("torch_copy", lambda x, y: y.copy_(x)),
                     ("torch_mul", lambda x, y: torch.mul(x, 0.5, out=y))):
        res[name] = [_chain_gbs(torch, stream, src, dst, op, a.reps)]
        elem_bytes[name] = 8 * n * nb
    out = {k: {"gbs_best": max(v), "frac_best": max(v) / hbm, "us_per_launch":
               elem_bytes[k] / max(v) / 1e3 / 5} for k, v in res.items()}
    print(json.dumps({"lib": os.environ.get("DEAR_LIB", "libdear.so"), "align4": a.align4,
                      "peak": hbm, **out}))


def _chain_gbs(torch, stream, src, dst, op, reps):
    """8 B per element over the buffers, `reps` rounds in one CUDA graph."""
    def chain(reps):
        for _ in range(reps):
            for x, y in zip(src, dst):
                op(x, y)
    with torch.cuda.stream(stream):
        chain(2)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            chain(reps)
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g.replay()
            e0.record(stream)
            g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / reps
            best = max(best, 8 * sum(x.numel() for x in src) / (t / 1e3) / 1e9)
    return best


if __name__ == "__main__":
    main()
