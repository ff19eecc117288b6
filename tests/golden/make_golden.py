"""Generate the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Every number written here comes from oracle/_ref/libdearsim_ref.so — the
reference's own C++ sources (/root/reference/proj/src) compiled unmodified
(oracle/Makefile) — called through oracle/ref_capi.cpp. The fixtures pin the
plain-C restatement (oracle/dear_oracle.c) and, through it, the GPU path.

Run in the build container (needs /root/reference):
    python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.lib import Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
MLP_LAYER = 1024 * 1024 + 1024  # W[1024,1024] + b[1024] (BASELINE config 1)
BUFFERS = [0, 500_000, 1_000_000, 2_000_000, 4_000_000, 4_198_400, 8_396_800,
           16_000_000, 25_000_000, 64_000_000, 100_000_000]
PRESETS = ["resnet50", "densenet201", "inceptionv4", "bert_base", "bert_large"]


def plans(ref: Reference) -> dict:
    out = {"buffers": BUFFERS, "models": {}}
    models = {f"{n}/{'imbalanced' if p else 'uniform'}": ref.preset_params(n, p)
              for n in PRESETS for p in (0, 1)}
    models["mlp4x1024"] = np.full(4, MLP_LAYER, np.int64)
    rng = np.random.default_rng(23)
    for t in range(8):  # random models, like test_model_fusion.cpp:150-179
        L = int(rng.integers(1, 80))
        models[f"random{t}"] = (rng.uniform(0.01, 8.0, L) * 1e6 / 4).astype(np.int64)
    for name, counts in models.items():
        out["models"][name] = {
            "param_counts": counts.tolist(),
            "plans": {str(b): ref.build_plan(counts, b) for b in BUFFERS},
        }
    return out


def chunks(ref: Reference) -> dict:
    cases = []
    for P in (1, 2, 3, 4, 5, 7, 8, 16):
        for d in sorted({0, 1, max(1, P - 1), P, P + 1, 1000, 4097, 1049600, 4198400,
                         5913061, 6_291_456}):
            b, e = ref.chunk_ranges(d, P)
            cases.append({"d": d, "P": P, "begin": b.tolist(), "end": e.tolist()})
    return {"cases": cases}


def collective(ref: Reference):
    arrays = {}
    meta = []
    seed = 1000
    for P in (1, 2, 3, 4, 5, 8, 16):
        for d in sorted({1, max(1, P - 1), P, P + 1, 1000, 4097}):
            seed += 1
            v = ref.random_vectors(P, d, seed)
            rs, rounds = ref.ring_reduce_scatter(v)
            avg = ref.all_reduce(v, average=True)
            assert all(np.array_equal(avg[0], avg[k]) for k in range(P))
            w0 = ref.random_vectors(1, d, seed + 50_000)[0]
            sgd = ref.sgd_step(w0, v, 0.05)
            key = f"P{P}_d{d}"
            arrays[key + "_rs"] = rs
            arrays[key + "_avg"] = avg[0]
            arrays[key + "_sgd"] = sgd[0]
            meta.append({"key": key, "P": P, "d": d, "seed": seed, "w_seed": seed + 50_000,
                         "lr": 0.05, "rounds": rounds})
    # acceptance.cpp:157-181 style: P=8, d=4097, lr=0.05, 3 chained steps.
    P, d = 8, 4097
    w = ref.random_vectors(1, d, 202)[0]
    ws = [w]
    for step in range(3):
        g = ref.random_vectors(P, d, 203 + step)
        out = ref.sgd_step(ws[-1], g, 0.05)
        assert all(np.array_equal(out[0], out[k]) for k in range(P))
        ws.append(out[0])
    arrays["sgd3_P8_d4097"] = ws[-1]
    meta.append({"key": "sgd3_P8_d4097", "P": P, "d": d, "w_seed": 202,
                 "grad_seeds": [203, 204, 205], "lr": 0.05})
    # First values of the tests' generator (test_collective.cpp:27-37).
    arrays["rng_seed1_P2_d5"] = ref.random_vectors(2, 5, 1).reshape(-1)
    return arrays, {"cases": meta}


def schedules(ref: Reference) -> dict:
    scen = []
    # The reference's golden traces (test_simulate.cpp:52-110): latency-only
    # clusters with alpha = per-collective time.
    scen.append(dict(name="two_layer_wfbp", counts=[1, 1], t_ff=[1, 1], t_bp=[2, 2],
                     policy="WFBP", buffer=0, P=2, alpha=1.0, beta=0.0))
    scen.append(dict(name="two_layer_dear", counts=[1, 1], t_ff=[1, 1], t_bp=[2, 2],
                     policy="DEAR", buffer=0, P=2, alpha=1.0, beta=0.0))
    for pol in ("WFBP", "DEAR"):
        scen.append(dict(name=f"comm_heavy_{pol.lower()}", counts=[1, 1, 1], t_ff=[1] * 3,
                         t_bp=[1] * 3, policy=pol, buffer=0, P=2, alpha=1.5, beta=0.0))
    rng = np.random.default_rng(7)
    for t in range(12):
        L = int(rng.integers(2, 40))
        counts = np.exp(rng.uniform(np.log(1e3), np.log(4e6), L)).astype(np.int64)
        tff = np.exp(rng.uniform(np.log(1e-4), np.log(2e-3), L))
        tbp = tff * rng.uniform(1.2, 2.0, L)
        P = int(rng.choice([2, 4, 8]))
        pol = ["WFBP", "WFBP_FUSED", "DEAR", "DEAR_FUSED"][t % 4]
        buf = int(rng.choice([1_000_000, 4_000_000, 25_000_000])) if "FUSED" in pol else 0
        scen.append(dict(name=f"random{t}_{pol.lower()}", counts=counts.tolist(),
                         t_ff=tff.tolist(), t_bp=tbp.tolist(), policy=pol, buffer=buf, P=P,
                         alpha=float(np.exp(rng.uniform(np.log(1e-6), np.log(1e-4)))),
                         beta=float(np.exp(rng.uniform(np.log(1e-11), np.log(2e-9))))))
    # BERT-Large preset at 25 MB, the headline config.
    bl = ref.preset_params("bert_large")
    for pol in ("WFBP_FUSED", "DEAR_FUSED"):
        scen.append(dict(name=f"bert_large_{pol.lower()}", counts=bl.tolist(),
                         t_ff=[1e-3 / len(bl)] * len(bl), t_bp=[2e-3 / len(bl)] * len(bl),
                         policy=pol, buffer=25_000_000, P=8, alpha=3e-6, beta=1 / 700e9))
    for s in scen:
        s["result"] = ref.simulate(s["counts"], s["t_ff"], s["t_bp"], s["policy"], s["buffer"],
                                   False, s["P"], s["alpha"], s["beta"])
    return {"scenarios": scen}


def main() -> None:
    ref = Reference()
    with open(os.path.join(OUT, "plans.json"), "w") as f:
        json.dump(plans(ref), f, separators=(",", ":"))
    with open(os.path.join(OUT, "chunks.json"), "w") as f:
        json.dump(chunks(ref), f, separators=(",", ":"))
    arrays, meta = collective(ref)
    np.savez_compressed(os.path.join(OUT, "collective.npz"), **arrays)
    with open(os.path.join(OUT, "collective.json"), "w") as f:
        json.dump(meta, f, indent=1)
    with open(os.path.join(OUT, "schedules.json"), "w") as f:
        json.dump(schedules(ref), f, separators=(",", ":"))
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
