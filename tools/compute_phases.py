#!/usr/bin/env python
"""Compute-only step (no runtime) split into its phases, graph-replayed:
set_input, forward chain, zero_grad, backward chain — against the tile
tuner's chain estimates (profiling aid).

    python tools/compute_phases.py [--workload resnet50]
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
    ap.add_argument("--wgrad-split", type=int, default=0)
    a = ap.parse_args()
    import torch

    import bench
    from paper_2302_12445_b200.presets import preset_param_counts
    from paper_2302_12445_b200.synthetic import SyntheticModel

    wl = bench.WORKLOADS[a.workload]
    import time
    t0 = time.time()
    m = SyntheticModel(preset_param_counts(wl["preset"]), wl["hidden"],
                       wl["batch"] * wl["tokens_per_sample"], seed=1234,
                       wgrad_split=a.wgrad_split)
    t_build = time.time() - t0
    s = torch.cuda.Stream()
    names = ("base", "input", "ff", "zero", "bp")
    ev = {k: torch.cuda.Event(enable_timing=True, external=True) for k in names}

    def step():
        with torch.cuda.stream(s):
            ev["base"].record(s)
            m.set_input(None, s)
            ev["input"].record(s)
            for l in range(1, m.L + 1):
                m.forward_layer(l, s)
            ev["ff"].record(s)
            m.zero_grad()
            ev["zero"].record(s)
            for l in range(m.L, 0, -1):
                m.backward_layer(l, s)
            ev["bp"].record(s)

    run = bench.make_runner(step, True, s)
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    res = {k: [] for k in names[1:]}
    for _ in range(5):
        run()
        torch.cuda.synchronize()
        prev = "base"
        for k in names[1:]:
            res[k].append(ev[prev].elapsed_time(ev[k]))
            prev = k
    ms = {k: sorted(v)[len(v) // 2] for k, v in res.items()}
    t = m.tiles or {}
    print(json.dumps({"workload": a.workload, "L": m.L, "wgrad_split": a.wgrad_split,
                      "build_and_tune_s": round(t_build, 1),
                      "splits_used": m.wgrad[0].info()["splits"], "phases_ms": ms,
                      "ff_us_per_layer": ms["ff"] * 1e3 / m.L,
                      "bp_us_per_layer": ms["bp"] * 1e3 / m.L,
                      "tuner_chain_us": {"ff": t.get("ff", {}).get("us"),
                                         "bp_group": t.get("bp_group_us")},
                      "tiles": t}), flush=True)


if __name__ == "__main__":
    main()
