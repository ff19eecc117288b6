#!/usr/bin/env python
"""Backprop (grouped wgrad + dgrad) of the synthetic layer vs the weight
gradient's split-K and tile: graph-chained launch time, and from one traced
launch the end of the weight-gradient CTAs vs the data-gradient CTAs.

    python tools/gemm_bp_splits.py [--workload resnet50]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    a = ap.parse_args()
    import torch

    from bench_gemm import SHAPES
    from paper_2302_12445_b200.gemm import GemmPlan, set_trace, time_chain

    T, H, n = SHAPES[a.workload]
    R = math.ceil(n / H)
    rpad = (R + 63) // 64 * 64
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    xt = x.t().contiguous()
    dy = (torch.randn(T, rpad, device="cuda") * 1e-3).to(torch.bfloat16)
    dyt = dy.t().contiguous()
    W = torch.randn(R * H, device="cuda").to(torch.bfloat16)
    L = 16
    Gs = [torch.zeros(n + 64, device="cuda") for _ in range(L)]
    dx = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    dg = GemmPlan(dy, W, dx, T, H, R, b_mn_major=True, lda=rpad, ldb=H, ldd=H, early_operands=True)
    wgs = [GemmPlan(dyt, xt, G, R, H, T, lda=T, ldb=T, ldd=H, d_limit=n, accumulate=True,
                    early_operands=True) for G in Gs]
    s = torch.cuda.Stream()
    out = []
    for wbn, wpair in ((128, 0), (256, 0)):
        for sp in (1, 2, 4, 8, 16, 24):
            try:
                for w in wgs:
                    w.set_tile(wbn, wpair)
                    w.set_splits(sp)
            except Exception as e:
                continue
            us = time_chain(lambda i: GemmPlan.run_group([wgs[i % L], dg], s), L, s, reps=5)
            items = wgs[0].info()
            n_w = items["m_tiles"] * items["n_tiles"] * items["splits"]
            buf = torch.zeros(8 * 320, dtype=torch.int64, device="cuda")
            set_trace(buf)
            with torch.cuda.stream(s):
                GemmPlan.run_group([wgs[0], dg], s)
            torch.cuda.synchronize()
            set_trace(None)
            t = buf.view(-1, 8).cpu().numpy().astype("float64")
            ok = t[:, 0] > 0
            t0 = t[ok, 0].min()
            end = (t[:, 6] - t0) / 1e3
            idx = range(len(t))
            wend = max((end[i] for i in idx if ok[i] and i < n_w), default=0.0)
            dend = max((end[i] for i in idx if ok[i] and i >= n_w), default=0.0)
            import numpy as np
            wi = [i for i in idx if ok[i] and i < n_w]
            rel = (t - t0) / 1e3
            first = np.median([rel[i, 3] for i in wi]) if wi else 0.0
            mma = np.median([rel[i, 4] - rel[i, 3] for i in wi]) if wi else 0.0
            epi = np.median([rel[i, 5] - rel[i, 4] for i in wi]) if wi else 0.0
            epi_max = max([rel[i, 5] - rel[i, 4] for i in wi], default=0.0)
            rec = {"wgrad_bn": wbn, "pair": wpair, "splits": items["splits"], "wgrad_items": n_w,
                   "chain_us": us, "traced_wgrad_end_us": wend, "traced_dgrad_end_us": dend,
                   "wgrad_first_stage_us": float(first), "wgrad_mainloop_us": float(mma),
                   "wgrad_epilogue_us_median": float(epi), "wgrad_epilogue_us_max": float(epi_max),
                   "ctas": int(ok.sum())}
            out.append(rec)
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
