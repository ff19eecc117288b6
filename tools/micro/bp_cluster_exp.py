import math, os, sys, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch
from bench_gemm import SHAPES
from paper_2302_12445_b200.gemm import GemmPlan, time_chain
T, H, n = SHAPES[os.environ.get("WL", "resnet50")]
R = math.ceil(n / H); rpad = (R + 63) // 64 * 64
x = torch.randn(T, H, device="cuda").to(torch.bfloat16); xt = x.t().contiguous()
dy = (torch.randn(T, rpad, device="cuda") * 1e-3).to(torch.bfloat16); dyt = dy.t().contiguous()
W = torch.randn(R * H, device="cuda").to(torch.bfloat16)
L = 16
Gs = [torch.zeros(n + 64, device="cuda") for _ in range(L)]
dx = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
s = torch.cuda.Stream()
for cl in ("0", "1"):
    os.environ["DEAR_GEMM_CLUSTER"] = cl
    dg = GemmPlan(dy, W, dx, T, H, R, b_mn_major=True, lda=rpad, ldb=H, ldd=H, early_operands=True)
    for sp in (0, 2, 4, 8, 16):
        wgs = [GemmPlan(dyt, xt, G, R, H, T, lda=T, ldb=T, ldd=H, d_limit=n, accumulate=True,
                        early_operands=True, split_k=sp) for G in Gs]
        us = time_chain(lambda i: GemmPlan.run_group([wgs[i % L], dg], s), L, s, reps=5)
        usw = time_chain(lambda i: wgs[i % L].run(s), L, s, reps=5)
        print(json.dumps({"cluster": cl, "split_req": sp, "wgrad": wgs[0].info(), "dgrad": {k: dg.info()[k] for k in ("bn", "cm", "cn", "pair")}, "bp_chain_us": us, "wgrad_only_chain_us": usw}), flush=True)
        for w in wgs: w.close()
    dg.close()
