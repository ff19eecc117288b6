#!/usr/bin/env python
"""Sweep the GEMM tile configuration (single-CTA vs 2-CTA pair, BN) on the
synthetic-layer shapes; event-timed back-to-back launches cycling 8 layers.

    python tools/sweep_gemm_tiles.py [--workloads resnet50,bert_base,bert_large]

Prints one JSON line per (workload, kind) with every config's µs and the
best one, and the cost model's own choice (the default plan) for comparison.
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
    ap.add_argument("--workloads", default="resnet50,bert_base,bert_large")
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--early", type=int, default=1, help="plans with early_operands")
    ap.add_argument("--kinds", default="ff,dgrad,wgrad")
    a = ap.parse_args()
    import torch

    from bench_gemm import SHAPES
    from paper_2302_12445_b200.gemm import GemmPlan

    def timeit(fn, iters):
        """µs per call, the calls captured in one CUDA graph (no host launch cost)."""
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(iters):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(3):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / (3 * iters)

    for wl in a.workloads.split(","):
        T, H, n = SHAPES[wl]
        R = math.ceil(n / H)
        rpad = (R + 63) // 64 * 64
        x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
        xt = x.t().contiguous()
        dy = torch.randn(T, rpad, device="cuda").to(torch.bfloat16)
        dyt = dy.t().contiguous()
        Ws = [torch.randn(R * H, device="cuda").to(torch.bfloat16) for _ in range(8)]
        Gs = [torch.zeros(n, device="cuda") for _ in range(8)]
        y = torch.empty(T, rpad, device="cuda", dtype=torch.bfloat16)
        dx = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
        e = bool(a.early)
        makers = {
            "ff": (lambda i: GemmPlan(x, Ws[i], y, T, R, H, lda=H, ldb=H, ldd=rpad,
                                      early_operands=e), T, R, False),
            "dgrad": (lambda i: GemmPlan(dy, Ws[i], dx, T, H, R, b_mn_major=True, lda=rpad,
                                         ldb=H, ldd=H, early_operands=e), T, H, True),
            "wgrad": (lambda i: GemmPlan(dyt, xt, Gs[i], R, H, T, lda=T, ldb=T, ldd=H,
                                         d_limit=n, accumulate=True, early_operands=e),
                      R, H, False),
        }
        for kind, (mk, M, N, mn) in makers.items():
            if kind not in a.kinds.split(","):
                continue
            res = {}
            configs = [("auto", None, None)]
            for pair in ("0", "2"):
                for bn in range(48, 257, 16):
                    if pair == "2" and mn and bn not in (128, 256):
                        continue
                    ntl = (N + bn - 1) // bn
                    if ntl > 1 and (ntl - 1) * bn >= N:
                        continue
                    configs.append((f"{'pair' if pair == '2' else 'single'}_bn{bn}", pair, bn))
            for name, pair, bn in configs:
                for k in ("DEAR_GEMM_PAIR", "DEAR_GEMM_BN"):
                    os.environ.pop(k, None)
                if pair is not None:
                    os.environ["DEAR_GEMM_PAIR"] = pair
                    os.environ["DEAR_GEMM_BN"] = str(bn)
                plans = [mk(i) for i in range(8)]
                info = plans[0].info()
                k = [0]

                def run():
                    k[0] = (k[0] + 1) % 8
                    plans[k[0]].run()
                res[name] = round(timeit(run, a.iters), 2)
                if name == "auto":
                    res["auto_cfg"] = f"{'pair' if info['pair'] else 'single'}_bn{info['bn']}"
                for p in plans:
                    p.close()
            best = min((v, k) for k, v in res.items() if k not in ("auto", "auto_cfg"))
            print(json.dumps({"workload": wl, "kind": kind, "M": M, "N": N, "early": e,
                              "auto": res["auto"], "auto_cfg": res["auto_cfg"],
                              "best": best[1], "best_us": best[0], "all": res}), flush=True)
        for k in ("DEAR_GEMM_PAIR", "DEAR_GEMM_BN"):
            os.environ.pop(k, None)


if __name__ == "__main__":
    main()
