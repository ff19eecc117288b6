#!/usr/bin/env python
"""Throughput of the tcgen05 GEMM on the synthetic-layer shapes (FF, grouped
wgrad+dgrad), back-to-back launches, CUDA events; cuBLAS (torch.matmul) on
the same FF/dgrad shapes as a yardstick only.

    python tools/bench_gemm.py [--workload resnet50|bert_large|bert_base] [--iters 50]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SHAPES = {  # (tokens, hidden, params per tensor)
    "resnet50": (64 * 160, 512, 159006),
    "bert_base": (64 * 64, 768, 534466),
    "bert_large": (32 * 64, 1024, 844723),
    "mlp4x1024": (64, 1024, 1049600),
}


def timeit(fn, iters):
    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="resnet50")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--layers", type=int, default=8, help="distinct layers cycled (L2 realism)")
    a = ap.parse_args()
    import torch

    from paper_2302_12445_b200.gemm import GemmPlan

    T, H, n = SHAPES[a.workload]
    R = math.ceil(n / H)
    rpad = (R + 63) // 64 * 64
    dev = "cuda"
    x = torch.randn(T, H, device=dev).to(torch.bfloat16)
    xt = x.t().contiguous()
    dy = torch.randn(T, rpad, device=dev).to(torch.bfloat16)
    dyt = dy.t().contiguous()
    Ws = [torch.randn(R * H, device=dev).to(torch.bfloat16) for _ in range(a.layers)]
    Gs = [torch.zeros(n, device=dev) for _ in range(a.layers)]
    y = torch.empty(T, rpad, device=dev, dtype=torch.bfloat16)
    dx = torch.empty(T, H, device=dev, dtype=torch.bfloat16)
    ff = [GemmPlan(x, W, y, T, R, H, lda=H, ldb=H, ldd=rpad) for W in Ws]
    dg = [GemmPlan(dy, W, dx, T, H, R, b_mn_major=True, lda=rpad, ldb=H, ldd=H) for W in Ws]
    wg = [GemmPlan(dyt, xt, G, R, H, T, lda=T, ldb=T, ldd=H, d_limit=n, accumulate=True)
          for G in Gs]
    flop = 2 * T * R * H
    out = {"workload": a.workload, "T": T, "H": H, "R": R,
           "ff_plan": ff[0].info(), "dgrad_plan": dg[0].info(), "wgrad_plan": wg[0].info()}
    k = [0]

    def nxt():
        k[0] = (k[0] + 1) % a.layers
        return k[0]

    t = timeit(lambda: ff[nxt()].run(), a.iters)
    out["ff"] = {"us": t * 1e3, "tflops": flop / (t / 1e3) / 1e12}
    t = timeit(lambda: dg[nxt()].run(), a.iters)
    out["dgrad"] = {"us": t * 1e3, "tflops": flop / (t / 1e3) / 1e12}
    t = timeit(lambda: wg[nxt()].run(), a.iters)
    out["wgrad"] = {"us": t * 1e3, "tflops": flop / (t / 1e3) / 1e12}

    def bp():
        i = nxt()
        GemmPlan.run_group([wg[i], dg[i]])
    t = timeit(bp, a.iters)
    out["bp_group"] = {"us": t * 1e3, "tflops": 2 * flop / (t / 1e3) / 1e12}
    # cuBLAS yardstick (not used by the product)
    Wm = [W.view(R, H) for W in Ws]
    t = timeit(lambda: torch.matmul(x, Wm[nxt()].t()), a.iters)
    out["cublas_ff"] = {"us": t * 1e3, "tflops": flop / (t / 1e3) / 1e12}
    t = timeit(lambda: torch.matmul(dy[:, :R], Wm[nxt()]), a.iters)
    out["cublas_dgrad"] = {"us": t * 1e3, "tflops": flop / (t / 1e3) / 1e12}
    t = timeit(lambda: torch.matmul(dyt[:R], xt.t()), a.iters)
    out["cublas_wgrad"] = {"us": t * 1e3, "tflops": flop / (t / 1e3) / 1e12}
    big = torch.randn(8192, 8192, device=dev).to(torch.bfloat16)
    dbig = torch.empty(8192, 8192, device=dev, dtype=torch.bfloat16)
    pb = GemmPlan(big, big, dbig, 8192, 8192, 8192, ldd=8192)
    t = timeit(lambda: pb.run(), 10)
    out["ours_8192"] = {"us": t * 1e3, "tflops": 2 * 8192**3 / (t / 1e3) / 1e12}
    t = timeit(lambda: torch.matmul(big, big.t()), 10)
    out["cublas_8192"] = {"us": t * 1e3, "tflops": 2 * 8192**3 / (t / 1e3) / 1e12}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
