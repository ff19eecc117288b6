#!/usr/bin/env python
"""Per-CTA phase timeline of back-to-back GEMM launches (profiling aid).

    python tools/trace_gemm.py [--workload bert_large] [--kind ff|bp] [--launches 6]

Prints, per launch (µs relative to the first CTA start of that launch):
CTA-start spread, prologue, dependency release, first stage landed, last MMA
issued, epilogue done, CTA end; and the gap to the previous launch's last CTA.
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
    ap.add_argument("--workload", default="bert_large")
    ap.add_argument("--kind", default="ff", choices=["ff", "bp", "dgrad", "wgrad"])
    ap.add_argument("--launches", type=int, default=6)
    ap.add_argument("--transposed", action="store_true", help="FF as Y^T = W X^T")
    ap.add_argument("--early", action="store_true", help="early-operand plans")
    ap.add_argument("--bn", type=int, default=0)
    ap.add_argument("--pair", type=int, default=0)
    a = ap.parse_args()
    import torch

    from bench_gemm import SHAPES
    from paper_2302_12445_b200.gemm import GemmPlan, set_trace

    T, H, n = SHAPES[a.workload]
    R = math.ceil(n / H)
    rpad = (R + 63) // 64 * 64
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    xt = x.t().contiguous()
    dy = torch.randn(T, rpad, device="cuda").to(torch.bfloat16)
    dyt = dy.t().contiguous()
    W = torch.randn(R * H, device="cuda").to(torch.bfloat16)
    G = torch.zeros(n, device="cuda")
    y = torch.empty(T, rpad, device="cuda", dtype=torch.bfloat16)
    dx = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    e = a.early
    if a.transposed:
        yt = torch.empty(rpad, T, device="cuda", dtype=torch.bfloat16)
        ff = GemmPlan(W, x, yt, R, T, H, lda=H, ldb=H, ldd=T, early_operands=e)
    else:
        ff = GemmPlan(x, W, y, T, R, H, lda=H, ldb=H, ldd=rpad, early_operands=e)
    dg = GemmPlan(dy, W, dx, T, H, R, b_mn_major=True, lda=rpad, ldb=H, ldd=H, early_operands=e)
    wg = GemmPlan(dyt, xt, G, R, H, T, lda=T, ldb=T, ldd=H, d_limit=n, accumulate=True,
                  early_operands=e)
    if a.bn:
        {"ff": ff, "dgrad": dg, "wgrad": wg, "bp": wg}[a.kind].set_tile(a.bn, a.pair)
    run = {"ff": lambda: ff.run(), "dgrad": lambda: dg.run(), "wgrad": lambda: wg.run(),
           "bp": lambda: GemmPlan.run_group([wg, dg])}[a.kind]
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    bufs = [torch.zeros(8 * 320, dtype=torch.int64, device="cuda") for _ in range(a.launches)]
    for b in bufs:
        set_trace(b)
        run()
    set_trace(None)
    torch.cuda.synchronize()
    prev_end = None
    out = []
    for i, b in enumerate(bufs):
        t = b.view(-1, 8).cpu().numpy()
        t = t[t[:, 0] > 0].astype("float64")
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        rec = {"launch": i, "ctas": int(len(t)),
               "start_spread_us": float(rel[:, 0].max()),
               "prologue_us": float((rel[:, 1] - rel[:, 0]).mean()),
               "dep_release_us": float(rel[:, 2].mean()),
               "first_stage_us": float(rel[:, 3].mean()),
               "last_mma_us": float(rel[:, 4].max()),
               "epilogue_done_us": float(rel[:, 5].max()),
               "end_us": float(rel[:, 6].max()),
               "gap_from_prev_us": None if prev_end is None else float((t0 - prev_end) / 1e3)}
        prev_end = t[:, 6].max()
        out.append(rec)
    print(json.dumps({"workload": a.workload, "kind": a.kind,
                      "plans": {"ff": ff.info(), "dgrad": dg.info(), "wgrad": wg.info()},
                      "launches": out}), flush=True)


if __name__ == "__main__":
    main()
