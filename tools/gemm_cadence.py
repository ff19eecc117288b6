#!/usr/bin/env python
"""Mainloop k-block cadence of the tcgen05 GEMM on chosen shapes (profiling aid).

    python tools/gemm_cadence.py            # the built-in shape set

For each shape: event-timed µs per launch (20 back-to-back launches), TFLOP/s,
and from the per-CTA %globaltimer trace the mean time per k-block between the
first landed stage and the last MMA issue of each CTA.
Separates per-SM operand-fetch limits from shared-tile hot spots: shape 'shareB'
has every CTA reading the same B tile, 'shareA' the same A tile.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2302_12445_b200.gemm import GemmPlan, set_trace

    shapes = [
        ("shareB_bn128", 148 * 128, 128, 8192, 128),
        ("shareB_bn256", 148 * 128, 256, 8192, 256),
        ("shareA_bn128", 128, 148 * 128, 8192, 128),
        ("shareA_bn256", 128, 148 * 256, 8192, 256),
        ("distinct_bn128", 1024, 18 * 128, 8192, 128),
        ("sq8192", 8192, 8192, 8192, 0),
        ("resnet_ff", 10240, 311, 512, 0),
        ("bertl_ff", 2048, 825, 1024, 0),
    ]
    only = sys.argv[1:]
    for name, M, N, K, bn in shapes:
        if only and name not in only:
            continue
        if bn:
            os.environ["DEAR_GEMM_BN"] = str(bn)
        else:
            os.environ.pop("DEAR_GEMM_BN", None)
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        ldd = (N + 63) // 64 * 64  # padded rows, as the synthetic layers use
        d = torch.empty(M, ldd, device="cuda", dtype=torch.bfloat16)
        p = GemmPlan(a, b, d, M, N, K, ldd=ldd)
        info = p.info()
        for _ in range(5):
            p.run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            p.run()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        buf = torch.zeros(8 * 160, dtype=torch.int64, device="cuda")
        set_trace(buf)
        p.run()
        set_trace(None)
        torch.cuda.synchronize()
        t = buf.view(-1, 8).cpu().numpy().astype("float64")
        t = t[t[:, 0] > 0]
        if os.environ.get("DEAR_LIB", "").startswith("libdear_wp"):
            lead = t[t[:, 7] > 0]  # CTAs that issued MMAs
            print(json.dumps({"shape": name, "info": info, "us": round(us, 2),
                              "tflops": round(2 * M * N * K / us / 1e6, 1),
                              "mma_loop_kcyc": round(float(lead[:, 7].mean()) / 1e3, 1),
                              "mma_wait_full_kcyc": round(float(lead[:, 3].mean()) / 1e3, 1),
                              "mma_wait_tmem_kcyc": round(float(lead[:, 5].mean()) / 1e3, 1),
                              "prod_wait_empty_kcyc": round(float(t[:, 4].mean()) / 1e3, 1)}),
                  flush=True)
            p.close()
            continue
        tiles = info["m_tiles"] * info["n_tiles"] * max(1, info["splits"])
        kb = (K + 63) // 64 // max(1, info["splits"])
        per_cta_tiles = tiles / len(t)
        main_us = (t[:, 4] - t[:, 3]) / 1e3
        cad = float(main_us.mean() / max(1.0, per_cta_tiles * kb - 1))
        print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "info": info,
                          "us": round(us, 2), "tflops": round(2 * M * N * K / us / 1e6, 1),
                          "ctas": int(len(t)), "kblock_us": round(cad, 3),
                          "first_stage_us": round(float(((t[:, 3] - t[:, 0]) / 1e3).mean()), 2)}),
              flush=True)
        p.close()


if __name__ == "__main__":
    main()
