"""Backprop grouped launch with BOTH problems in CTA-pair mode (one launch)
vs the tuned single-CTA tiles: graph-chained µs per grouped launch."""
import json, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))), "tools"))
import torch
from bench_gemm import SHAPES
from paper_2302_12445_b200.gemm import GemmPlan, time_chain

for wl in ("resnet50", "bert_large"):
    T, H, n = SHAPES[wl]
    R = math.ceil(n / H); rpad = (R + 63) // 64 * 64
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16); xt = x.t().contiguous()
    dy = (torch.randn(T, rpad, device="cuda") * 1e-3).to(torch.bfloat16); dyt = dy.t().contiguous()
    W = torch.randn(R * H, device="cuda").to(torch.bfloat16)
    L = 16
    Gs = [torch.zeros(n + 64, device="cuda") for _ in range(L)]
    dx = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.Stream()
    dg = GemmPlan(dy, W, dx, T, H, R, b_mn_major=True, lda=rpad, ldb=H, ldd=H, early_operands=True)
    wgs = [GemmPlan(dyt, xt, G, R, H, T, lda=T, ldb=T, ldd=H, d_limit=n, accumulate=True,
                    early_operands=True) for G in Gs]
    cfgs = [((128, 0), (256, 0)), ((256, 1), (256, 1)), ((128, 1), (256, 1)), ((256, 1), (128, 1)),
            ((128, 1), (128, 1))]
    for (wb, wp), (db, dp) in cfgs:
        for sp in (2, 4, 6, 8, 12):
            try:
                dg.set_tile(db, dp)
                for w in wgs:
                    w.set_tile(wb, wp)
                    w.set_splits(sp)
                for red in (False, True):
                    for w in wgs:
                        w.set_red_add(red)
                    us = time_chain(lambda i: GemmPlan.run_group([wgs[i % L], dg], s), L, s, reps=5)
                    print(json.dumps({"wl": wl, "wgrad": [wb, wp], "dgrad": [db, dp], "splits": wgs[0].info()["splits"],
                                      "red_add": red, "chain_us": round(us, 2)}), flush=True)
            except Exception as e:
                print(json.dumps({"wl": wl, "wgrad": [wb, wp], "dgrad": [db, dp], "splits": sp, "error": str(e)[:100]}))
    for w in wgs: w.close()
    dg.close()
