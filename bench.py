#!/usr/bin/env python
"""DeAR on B200 — training-step throughput on synthetic preset-shaped layers.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload resnet50]
    torchrun --nproc-per-node N bench.py --gpus N ...     (driver launch, N > 1)
    python bench.py --impl reference ...                  (the reference's CPU path)

One step = one DeAR iteration: feed-forward of every layer (each gated on its
own bucket's all-gather + unpack), backprop (wgrad + dgrad tcgen05 GEMMs per
layer) with pack -> reduce-scatter -> shard SGD update per fusion bucket on
the comm stream, and the all-gathers of the updated shards that the next
forward waits on. The whole iteration is captured once as a CUDA graph
(`--no-graph` runs it eagerly). Per-GPU work is fixed as N grows (weak
scaling). Printed: ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# BASELINE.json configs 1-4. tokens_per_sample turns a layer's parameters into
# dense-layer flops: 2 * params * tokens for FF. ResNet-50: 4.1 GMAC / 25.6M
# params ~= 160 MACs per parameter per image; BERT: 64-token sentences
# (PAPER.md:195); batch sizes per GPU from PAPER.md Table I.
WORKLOADS = {
    "mlp4x1024": dict(preset="mlp4x1024", hidden=1024, tokens_per_sample=1, batch=64,
                      config="BASELINE config 1: synthetic 4-layer fp32 MLP (1024-wide)"),
    "resnet50": dict(preset="resnet50", hidden=512, tokens_per_sample=160, batch=64,
                     config="BASELINE config 2: ResNet-50-shaped gradient set "
                            "(25.6M params, 161 tensors)"),
    "bert_base": dict(preset="bert_base", hidden=768, tokens_per_sample=64, batch=64,
                      config="BASELINE config 3: BERT-Base-shaped (110.1M params, 206 tensors)"),
    "bert_large": dict(preset="bert_large", hidden=1024, tokens_per_sample=64, batch=32,
                       config="BASELINE config 4: BERT-Large-shaped (336.2M params, 398 tensors)"),
}
METRIC = "samples/s at 1/2/4/8 B200 (DeAR vs WFBP)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="resnet50", choices=list(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="samples per GPU (0 = workload default)")
    ap.add_argument("--policy", default="DEAR_FUSED")
    ap.add_argument("--baseline-policy", default="WFBP_FUSED")
    ap.add_argument("--buffer", type=int, default=25_000_000, help="fusion buffer bytes")
    ap.add_argument("--lr", type=float, default=0.05)
    ap.add_argument("--momentum", type=float, default=0.0)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--backend", default="auto", choices=["auto", "nccl", "peer", "nvls"],
                    help="bucket collectives: fused NVLink peer kernels (auto when N > 1), "
                         "NVLS multicast kernels on a symmetric heap, or NCCL RS/AG")
    ap.add_argument("--group-dependency", type=int, default=1,
                    help="DEAR with dear_group_dependency (AG_g <- RS_g) and the comm "
                         "dispatch order simulated on measured times (0: global barrier)")
    ap.add_argument("--order-search", type=int, default=1,
                    help="time the simulated dispatch orders of several contention "
                         "factors and keep the fastest (0: use --contention only)")
    ap.add_argument("--contention", type=float, default=1.0,
                    help="comm-stage slow-down next to the GEMMs assumed when planning the "
                         "group-dependency dispatch order")
    ap.add_argument("--no-ablation", action="store_true", help="skip WFBP / compute-only runs")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-calibrate", action="store_true",
                    help="north star: skip the t_ag = 1.25 t_ff batch comparison (N > 1)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--buffer-sweep-bytes",
                    default="1000000,5000000,10000000,25000000,50000000,100000000",
                    help="N > 1: BASELINE config 3 (BERT-Base) DeAR vs WFBP at these fusion "
                         "buffers ('' to skip)")
    ap.add_argument("--extra-workload", default="bert_large",
                    help="also measure DeAR vs WFBP on this workload (north-star "
                         "comparison); 'none' to skip")
    ap.add_argument("--partition-bytes", type=int, default=4_000_000,
                    help="PRIORITY_PARTITION ablation (north star, N > 1): part size")
    ap.add_argument("--no-priority-partition", action="store_true")
    ap.add_argument("--north-star-batches", default="64",
                    help="N > 1: also compare DeAR / WFBP at these per-GPU batches")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the post-timing oracle parity check of one bucket")
    ap.add_argument("--parity-steps", type=int, default=3)
    ap.add_argument("--no-timeline", action="store_true",
                    help="skip the post-timing measured-timeline validation")
    ap.add_argument("--timeline-out", default="", help="write the measured Chrome trace here")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="only run this many graph replays (for ncu launch lists)")
    return ap.parse_args()


# --------------------------------------------------------------- helpers ----
class ClockSampler:
    """SM clocks and throttle reasons sampled during the timed region: NVML
    polled from a thread every `period_ms` (nvidia-smi's own sampling is too
    coarse for a region of a few tens of ms; it remains the fallback). Samples
    carry their time; the summary keeps the ones inside [start, end] of the
    timed region (time_loop marks them)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int, period_ms: float = 2.0):
        self.index, self.proc, self.rows = index, None, []
        self.period_ms = period_ms
        self.start = self.end = None
        self.source = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            bits = [N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                    N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap]
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)

            def poll():
                while not self._stop.is_set():
                    try:
                        sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                        rs = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                    except Exception:
                        break
                    flags = ["Active" if rs & b else "Not Active" for b in bits]
                    self.rows.append((time.monotonic(), [str(sm), str(mx), "0", *flags]))
                    time.sleep(self.period_ms / 1e3)
            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
            self.source = "nvml"
        except Exception:
            self._start_smi()
        t0 = time.monotonic()
        while not self.rows and time.monotonic() - t0 < 3.0:
            time.sleep(0.005)
        return self

    def _start_smi(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            self.source = "nvidia-smi"
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [x.strip() for x in line.split(",")]))

    def mark(self, which: str) -> None:
        setattr(self, which, time.monotonic())

    def __exit__(self, *a):
        self._stop.set()
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        rows = [r for t, r in self.rows if self.start is not None and self.end is not None
                and self.start <= t <= self.end]
        in_region = len(rows)
        if not rows:
            rows = [r for _, r in self.rows]
        sm = [float(r[0]) for r in rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in rows if len(r) >= 7
                          for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows), "samples_in_timed_region": in_region,
                "source": self.source}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d["bf16_tflops_sustained"], "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


# ------------------------------------------------------------ reference arm --
def reference_arm(a, wl, world: int, rank: int, emit: bool = True, threads: int = 0):
    """The reference's own CPU path (oracle/_ref: proj/src/collective.cpp
    sgd_step per fusion bucket, fp64, P = N virtual workers), all host cores
    (threads = 0) or `threads` threads (1 = the reference's own single-threaded
    execution)."""
    if rank != 0:
        return None
    import numpy as np

    from oracle.lib import Reference
    from paper_2302_12445_b200.presets import preset_param_counts
    from oracle.schedule import fusion_plan

    counts = preset_param_counts(wl["preset"])
    P = max(1, world)
    plan = fusion_plan([4 * c for c in counts], a.buffer if "FUSED" in a.policy else 0)
    buckets = [sum(counts[lo - 1:hi]) for lo, hi in plan]
    D = sum(buckets)
    cores = threads if threads > 0 else (os.cpu_count() or 1)
    # Bound memory (P replicas + P grads in fp64, ~3x transient) to ~12 GB and
    # the sample to the requested seconds: take whole buckets in plan order.
    cap = int(12e9 / (8 * P * 5))
    sample, tot = [], 0
    for b in buckets:
        if tot + b > cap and sample:
            break
        sample.append(b)
        tot += b
    ref = Reference()
    t1 = ref.time_sgd_steps(sample, P, cores, 1, seed=7)[0]  # warm-up
    if emit:  # the reference arm proper: exactly K timed steps after W warm-ups
        for _ in range(max(0, a.warmup - 1)):
            ref.time_sgd_steps(sample, P, cores, 1, seed=7)
        steps = a.steps
    else:     # cpu_baseline leg of our line: bounded to ~cpu_seconds
        steps = max(1, min(50, int(a.cpu_seconds / max(t1, 1e-6))))
    ts = ref.time_sgd_steps(sample, P, cores, steps, seed=8)
    t_sample = float(np.median(ts))
    t_full = t_sample * D / tot
    batch = a.batch or wl["batch"]
    value = batch * P / t_full
    cpu = {"value": value, "unit": "samples/s", "cores": cores, "kind": "reference",
           "sample": f"oracle/_ref sgd_step (reference collective.cpp, fp64) over "
                     f"{len(sample)}/{len(buckets)} fusion buckets ({tot}/{D} elements) x P={P} "
                     f"virtual workers, {steps} steps, {cores} threads; per-step time scaled "
                     f"to the full model; samples/s = batch {batch} x P / step time",
           "step_seconds_full_model": t_full}
    if emit:
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
                "steps": steps, "warmup": a.warmup, "ms_per_step": t_full * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": {"workload": wl["config"], "policy": a.policy,
                           "fusion_buffer_bytes": a.buffer, "global_batch": batch * P},
                "impl": "reference", "cpu_baseline": cpu,
                "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
    return cpu


# ----------------------------------------------------------------- GPU arm --
class Step:
    """One DeAR iteration over the synthetic model through the public API."""

    def __init__(self, model, rt, stream, x_host=None, out_host=None, prefetch=True):
        import torch

        self.m, self.rt, self.s = model, rt, stream
        self.x_host, self.out_host = x_host, out_host
        # e2e input pipeline (what a pinned-memory data loader does): every step
        # copies one batch host -> device, the NEXT step's, on a copy stream
        # overlapped with this step's compute; this step's batch (landed during
        # the previous step) moves staging -> model input with a D2D copy.
        self.prefetch = prefetch and x_host is not None
        if self.prefetch:
            self.x_stage = torch.empty_like(model.x)
            self.x_stage.copy_(x_host)  # primes the first step (outside timing)
            self.copy_stream = torch.cuda.Stream()

    def __call__(self):
        import torch

        m, rt, s = self.m, self.rt, self.s
        with torch.cuda.stream(s):
            if self.prefetch:
                m.x.copy_(self.x_stage)
                m.set_input(None)
                self.copy_stream.wait_stream(s)  # staging buffer consumed
                with torch.cuda.stream(self.copy_stream):
                    self.x_stage.copy_(self.x_host, non_blocking=True)
            else:
                m.set_input(self.x_host)
            for l in range(1, m.L + 1):
                if rt is not None:
                    rt.param_wait(l, s)
                m.forward_layer(l, s)
            m.zero_grad()
            for l in range(m.L, 0, -1):
                m.backward_layer(l, s)
                if rt is not None:
                    rt.grad_ready(l, s)
            if rt is not None:
                rt.step(s)
                rt.join(s)
            if self.prefetch:
                s.wait_stream(self.copy_stream)  # next batch landed (joins the graph)
            if self.out_host is not None:
                self.out_host.copy_(m.result_scalar(), non_blocking=True)


def _mark(name):
    """DEAR_BENCH_TRACE=1: device-synchronise and log a section marker to
    stderr (localises an asynchronous CUDA error to the section before it)."""
    if os.environ.get("DEAR_BENCH_TRACE") != "1":
        return
    import time

    import torch

    try:
        torch.cuda.synchronize()
        status = "ok"
    except Exception as e:  # noqa: BLE001
        status = f"{type(e).__name__}: {e}"[:200]
    print(f"[bench-trace {time.strftime('%H:%M:%S')} rank {os.environ.get('RANK', '0')}] "
          f"{name}: {status}", file=sys.stderr, flush=True)


def time_loop(fn, steps, warmup, stream, dist_on, clock=None):
    import torch

    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if dist_on:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clock is not None:
        clock.mark("start")
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    if clock is not None:
        clock.mark("end")
    ms = e0.elapsed_time(e1)
    if dist_on:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = t.item()
        torch.distributed.barrier()
    return ms / steps


def make_runner(step, use_graph, stream):
    """Eager step, or a CUDA graph of it (captured after one eager step)."""
    import torch

    if not use_graph:
        return step
    step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
        step()
    torch.cuda.synchronize()

    def replay():
        with torch.cuda.stream(stream):  # replay on the timed stream
            g.replay()
    return replay


def make_runtime(a, model, comm, rank, world, stream, policy, defer):
    """Runtime over the model's tensors. For DEAR policies with
    --group-dependency (the reference's dear_group_dependency, policy.hpp:44),
    the comm stream's dispatch order is planned by the reference's scheduler
    (costmodel.predict_iteration = simulate.cpp:65-159) on this run's own
    measurements: per-layer GEMM chain times from the tile tuner and per-bucket
    RS-side (pack+RS+update) / AG-side (AG+unpack) stage times of comm-only
    iterations, scaled by an assumed contention factor; the candidate orders of
    several factors are timed and the fastest kept. Rank 0's orders are
    broadcast (collectives must be issued in the same order on every rank)."""
    import torch

    import paper_2302_12445_b200 as dear
    from paper_2302_12445_b200 import costmodel

    gd = bool(a.group_dependency) and policy.startswith("DEAR")
    rt = dear.Runtime(comm, rank, world, policy=policy, fusion_buffer_bytes=a.buffer,
                      lr=a.lr, momentum=a.momentum, defer_allgather=defer,
                      backend=a.backend, stream=stream, dear_group_dependency=gd,
                      heap=model.heap if a.backend == "nvls" else None)
    for l in range(1, model.L + 1):
        rt.register(l, model.params[l - 1], model.grads[l - 1], model.shadows[l - 1])
    rt.finalize()
    rt.comm_order_info = None
    if not gd:
        return rt
    # Stage times of comm-only iterations (gradients reported back to back, no
    # GEMMs): the pure comm-stream cost per bucket, scaled by --contention for
    # the slow-down next to the layer GEMMs.
    rt.set_timing(True)
    for _ in range(3):
        with torch.cuda.stream(stream):
            for l in range(1, model.L + 1):
                rt.param_wait(l, stream)
            for l in range(model.L, 0, -1):
                rt.grad_ready(l, stream)
            rt.step(stream)
        rt.synchronize()
    torch.cuda.synchronize()
    st = rt.timings()
    rt.set_timing(False)
    tiles = model.tiles or {}
    t_ff = (tiles.get("ff", {}).get("us") or 10.0) * 1e-6
    t_bp = (tiles.get("bp_group_us") or 20.0) * 1e-6
    lb = [4 * n for n in model.numels]

    def simulate(ct):
        k = ct / 1e3
        rs = [k * sum(v for v in (x["pack"], x["rs"], x["update"]) if v) for x in st]
        ag = [k * sum(v for v in (x["ag"], x["unpack"]) if v) for x in st]
        sim = costmodel.predict_iteration(lb, [t_ff] * model.L, [t_bp] * model.L, policy,
                                          a.buffer, world, 0.0, 0.0, group_dependency=True,
                                          rs_times=rs, ag_times=ag)
        order = torch.tensor(sim["comm_order"], dtype=torch.int32, device="cuda")
        if world > 1:  # every rank issues the same sequence
            torch.distributed.broadcast(order, 0)
        return order.cpu().tolist(), sim["iteration_seconds"]

    def backfilled(order):
        last_rs = max(i for i, v in enumerate(order) if v > 0)
        return sum(1 for v in order[:last_rs] if v < 0)

    # Candidate orders: the scheduler simulated over a range of assumed
    # comm slow-downs (different numbers of all-gathers back-filled into
    # backprop); each is timed as the real graph-replayed step (max over
    # ranks, so all ranks pick the same) and the fastest is kept.
    cands = {}
    for ct in (a.contention,) if not a.order_search else (0.6, 0.8, 1.0, 1.2, 1.5):
        order, pred = simulate(ct)
        cands.setdefault(backfilled(order), (ct, order, pred))
    trials = []
    for nb, (ct, order, pred) in sorted(cands.items()):
        rt.set_comm_order(order)
        ms = float("nan")
        if len(cands) > 1:
            run = make_runner(Step(model, rt, stream), True, stream)
            ms = time_loop(run, 6, 3, stream, world > 1)
            del run
            rt.synchronize()
        trials.append({"contention": ct, "ags_during_backprop": nb,
                       "ms": ms if ms == ms else None,
                       "predicted_ms": pred * 1e3, "order": order})
    best = min(trials, key=lambda t: (t["ms"] if t["ms"] is not None else 0.0))
    rt.set_comm_order(best["order"])
    rt.comm_order_info = {"source": "reference scheduler simulated on measured stage times; "
                                    "fastest of the candidate orders",
                          "contention": best["contention"],
                          "ags_during_backprop": best["ags_during_backprop"],
                          "candidates": [{k: v for k, v in t.items() if k != "order"}
                                         for t in trials],
                          "stage_us_mean": {k: sum(x[k] or 0.0 for x in st) * 1e3 / len(st)
                                            for k in ("pack", "rs", "update", "ag", "unpack")},
                          # per bucket (plan order): RS side (pack + RS + update) and
                          # AG side (AG + unpack) of a comm-only iteration, ms
                          "stage_ms": [[sum(v for v in (x["pack"], x["rs"], x["update"]) if v),
                                        sum(v for v in (x["ag"], x["unpack"]) if v)] for x in st],
                          "t_ff_us": t_ff * 1e6, "t_bp_us": t_bp * 1e6, "buckets": len(st)}
    return rt


def gpu_arm(a, wl, world, rank, local_rank):
    import torch

    import paper_2302_12445_b200 as dear
    from paper_2302_12445_b200.presets import preset_param_counts
    from paper_2302_12445_b200.synthetic import SyntheticModel

    dist_on = world > 1
    torch.cuda.set_device(local_rank)
    comm = None
    if dist_on:
        import torch.distributed as dist

        import datetime

        # A healthy run never waits minutes in one collective: fail instead of
        # hanging the job if a rank dies.
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"),
                                timeout=datetime.timedelta(minutes=5))
        comm = dear.init()
    batch = a.batch or wl["batch"]
    tokens = batch * wl["tokens_per_sample"]
    counts = preset_param_counts(wl["preset"])
    model = SyntheticModel(counts, wl["hidden"], tokens, seed=1234,
                           symmetric=a.backend == "nvls" and world > 1)
    stream = torch.cuda.Stream()
    use_graph = not a.no_graph
    hbm, tf_burst, tf_sus, peak_kind = peaks()

    def runtime(policy):
        return make_runtime(a, model, comm, rank, world, stream, policy, use_graph)

    res = {}
    # --- headline: DeAR, inputs resident ---------------------------------
    rt = runtime(a.policy)
    backend_used = rt.backend
    zero_copy = bool(getattr(rt, "zero_copy", False))
    nb = len(rt.buckets())
    bucket_launches = (nb if world == 1 and a.momentum == 0 else
                       2 * nb + 1 if zero_copy else 3 * nb)
    rt_order_info = rt.comm_order_info
    buckets = rt.buckets()
    run = make_runner(Step(model, rt, stream), use_graph, stream)
    if a.profile_steps:
        run()  # warm
        torch.cuda.synchronize()
        # ncu --nvtx --nvtx-include "dear_profile/" selects exactly these steps
        torch.cuda.nvtx.range_push("dear_profile")
        for _ in range(a.profile_steps):
            run()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
        rt.synchronize()
        if rank == 0:
            print(json.dumps({"profile_steps": a.profile_steps}), flush=True)
        return None
    with ClockSampler(local_rank) as clk:
        ms = time_loop(run, a.steps, a.warmup, stream, dist_on, clock=clk)
    res["dear_ms"] = ms
    clocks = clk.summary()

    # --- e2e through the public API: pinned host input in, scalar out -------
    x_host = torch.empty(model.x.shape, dtype=model.x.dtype, pin_memory=True)
    x_host.copy_(model.x.cpu())
    out_host = torch.empty((), dtype=model.y.dtype, pin_memory=True)
    rt.synchronize()
    run_e2e = make_runner(Step(model, rt, stream, x_host, out_host), use_graph, stream)
    res["e2e_ms"] = time_loop(run_e2e, a.steps, a.warmup, stream, dist_on)
    h2d = x_host.numel() * x_host.element_size()  # one batch per step (prefetched, Step)
    d2h = out_host.element_size()

    # --- per-stage timings (one instrumented eager step) ---------------------
    rt.synchronize()
    rt.set_timing(True)
    Step(model, rt, stream)()
    rt.synchronize()
    torch.cuda.synchronize()
    stage = rt.timings()
    rt.set_timing(False)
    # GEMM launch durations inside one eager step (compute stream events).
    gemm_ms, gemm_flops = _time_gemms(model, rt, stream)
    rt.synchronize()
    ok_replicas = rt.check_replicas()
    rt.close()

    # --- HBM kernels in isolation: comm-only iterations (no GEMMs) -----------
    _mark("main DeAR step measured")
    iso = _isolated_stage_times(model, runtime, stream, a.policy)
    _mark("isolated stage times")

    # --- ablation: same kernels, WFBP schedule; compute-only ------------------
    if not a.no_ablation:
        rtw = runtime(a.baseline_policy)
        runw = make_runner(Step(model, rtw, stream), use_graph, stream)
        res["wfbp_ms"] = time_loop(runw, a.steps, a.warmup, stream, dist_on)
        rtw.synchronize()
        rtw.close()
    # Compute-only step (the layer GEMM chain, no runtime): also the GEMM
    # roofline's timed region.
    _mark("ablation done")
    runc = make_runner(Step(model, None, stream), use_graph, stream)
    res["compute_ms"] = time_loop(runc, a.steps, a.warmup, stream, dist_on)

    # Everything below runs after the headline measurement. A failure in one
    # of these sections is recorded in the line instead of losing it; after a
    # CUDA error the context is unusable, so the remaining GPU sections are
    # skipped and the process exits right after printing (main()).
    broken = []

    def guarded(name, fn):
        if broken:
            return {"skipped": f"after the error in {broken[0]}"}
        try:
            return fn()
        except Exception as e:  # noqa: BLE001 - reported in the JSON line
            broken.append(name)
            print(f"[bench] {name} failed: {type(e).__name__}: {e}", file=sys.stderr, flush=True)
            return {"error": f"{type(e).__name__}: {e}"[:400]}

    _mark("headline measured")
    extra = None
    if a.extra_workload != "none" and a.extra_workload != a.workload:
        extra = guarded("north_star", lambda: compare_policies(a, a.extra_workload, comm, world,
                                                               rank, stream))
    config3 = None
    if world > 1 and a.buffer_sweep_bytes:
        config3 = guarded("config3", lambda: buffer_sweep(a, "bert_base", comm, world, rank,
                                                          stream))
    # Post-timing checks (nothing below is timed): one measured iteration in the
    # reference's trace schema, validated; oracle parity of one full bucket at
    # the bench configuration.
    timeline = None if a.no_timeline else guarded(
        "timeline", lambda: _measured_timeline(a, model, comm, rank, world, stream))
    parity = None if a.no_parity else guarded(
        "parity", lambda: _bench_parity(a, model, comm, rank, world, stream))
    gpu_arm.broken = broken
    if rank != 0:
        return None
    samples = batch * world
    value = samples / (res["dear_ms"] / 1e3)
    e2e = samples / (res["e2e_ms"] / 1e3)
    # Bucket-stage rooflines (isolated): algorithmic bytes per element.
    D = sum(counts)
    shard = sum(b["slot_stride"] for b in buckets)
    # isolated stages run at P = 1 when N = 1 (update over whole buckets)
    elem_bytes = {"pack": 8 * D, "update": (20 if a.momentum else 12) * shard,
                  "unpack": 10 * D, "direct": 14 * D}
    roof = {}
    for k, nbytes in elem_bytes.items():
        if k not in iso:
            continue
        t, launches = iso[k]
        roof[k] = {"bound": "hbm", "achieved": nbytes / (t / 1e3) / 1e9, "peak": hbm,
                   "unit": "GB/s", "frac": nbytes / (t / 1e3) / 1e9 / hbm,
                   "bytes_per_step": nbytes, "ms_per_step": t,
                   "launches_per_step": launches, "us_per_launch": 1e3 * t / launches,
                   "timing": "graph-replayed chain of launches (dear_bench_stage), "
                             "CUDA events, no GEMMs"}
    busbw = {}
    if world > 1:
        for k in ("rs", "ag"):
            ts = [(b["slot_stride"], st[k]) for b, st in zip(buckets, stage) if st[k]]
            tot_t = sum(t for _, t in ts)
            tot_b = sum((world - 1) * s * 4 for s, _ in ts)
            busbw[k] = tot_b / (tot_t / 1e3) / 1e9 if tot_t else None
    # GEMM roofline over the timed region: the step's GEMM flops / the
    # compute-only step (graph-replayed chain of the 3L layer GEMMs, which
    # overlap under programmatic dependent launch; CUDA events on `stream`).
    # Per-launch isolated timing (events between launches, no overlap) is
    # reported beside it.
    gemm_achieved = gemm_flops / (res["compute_ms"] / 1e3) / 1e12
    gemm_isolated = gemm_flops / (gemm_ms / 1e3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": res["dear_ms"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        # the DeAR path (params, grads, reduction, update) is fp32 as the north
        # star requires; the synthetic layer GEMMs compute in bf16
        "dtype": "fp32", "compute_dtype": "bf16",
        "data": "synthetic (seeded inputs; random-init params; no dataset)",
        "config": {"workload": wl["config"], "policy": a.policy, "collectives": backend_used,
                   "zero_copy": zero_copy,
                   "dear_group_dependency": bool(a.group_dependency),
                   "comm_order": rt_order_info,
                   "fusion_buffer_bytes": a.buffer, "buckets": len(buckets),
                   "batch_per_gpu": batch, "global_batch": samples, "tokens_per_gpu": tokens,
                   "hidden": wl["hidden"], "params": D, "cuda_graph": use_graph,
                   "l2": "working set (params+grads+buckets) > 126 MB L2; no flush"},
        "e2e": {"value": e2e, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "input_pipeline": "each step: D2D of its batch from staging, H2D of the next "
                                  "batch (pinned) on a copy stream overlapped with compute, "
                                  "D2H of the loss scalar",
                "d2h_bytes_per_step": d2h},
        "clocks": clocks,
        # our kernels per step: FF + grouped BP GEMMs (two launches when the
        # tuned wgrad / dgrad tiles differ in pair mode) and the bucket kernels:
        # P = 1 one direct update per bucket; zero-copy peer RS-update + AG per
        # bucket + the one-warp "gradients consumed" wait at dear_step; slot
        # peer pack + RS-update + AG-unpack; NCCL pack + update + unpack (the
        # NCCL collectives themselves are not counted)
        "gpu_launches": a.steps * (model.gemm_launches_per_step() + bucket_launches),
        "roofline": {"bound": "tensor", "kernel": "tcgen05 GEMM chain (FF + grouped wgrad/dgrad)",
                     "achieved": gemm_achieved, "peak": tf_sus, "unit": "TFLOP/s",
                     "frac": gemm_achieved / tf_sus, "traffic": _ncu_traffic(a.workload),
                     "peak_kind": f"{peak_kind} sustained",
                     "flops_per_step": gemm_flops, "gemm_ms_per_step": res["compute_ms"],
                     "isolated_launch_tflops": gemm_isolated},
        "hbm_kernels": roof,
        "gemm_tiles": model.tiles,
        "replicas_identical": ok_replicas,
    }
    line["compute_only_ms"] = res["compute_ms"]
    line["exposed_comm_pct"] = max(0.0, 100 * (res["dear_ms"] - res["compute_ms"]) /
                                   res["dear_ms"])
    if "wfbp_ms" in res:
        line["wfbp"] = {"policy": a.baseline_policy, "value": samples / (res["wfbp_ms"] / 1e3),
                        "ms_per_step": res["wfbp_ms"]}
        line["dear_over_wfbp"] = res["wfbp_ms"] / res["dear_ms"]
        line["wfbp_exposed_comm_pct"] = max(0.0, 100 * (res["wfbp_ms"] - res["compute_ms"]) /
                                            res["wfbp_ms"])
    if busbw:
        line["busbw_gbs"] = busbw
    if extra is not None:
        line["north_star"] = extra
    if config3 is not None:
        line["config3_buffer_sweep"] = config3
    if parity is not None:
        line["parity"] = parity
    if timeline is not None:
        line["timeline"] = timeline
    if world == 1 and not a.no_cpu:
        # BASELINE.md §2's plan: the reference's single-threaded execution;
        # the all-cores figure (each bucket's sgd_step on its own thread) beside it.
        line["cpu_baseline"] = reference_arm(a, wl, world, rank, emit=False, threads=1)
        line["cpu_baseline_all_cores"] = reference_arm(a, wl, world, rank, emit=False)
    return line


def _measured_timeline(a, model, comm, rank, world, stream):
    """One iteration in the reference's framing — BP_L..BP_1 then FF_1..FF_L of
    the next iteration (task_graph.cpp:127-146), with the bucket collectives in
    between — measured from two consecutive graph replays of the bench step
    (per-layer compute-stream events + the runtime's comm-stream stamps, all
    from one base event) and checked with timeline.validate: RS_g after the BP
    of g's lowest layer (:148-154), FF_l after the all-gather + unpack of
    g(l) (:207), no overlap on the compute stream (simulate.cpp:161-210)."""
    import torch

    from paper_2302_12445_b200 import timeline as T

    rt = make_runtime(a, model, comm, rank, world, stream, a.policy, True)
    L = model.L

    def ev():
        return torch.cuda.Event(enable_timing=True, external=True)
    ff = [(ev(), ev()) for _ in range(L)]
    bp = [(ev(), ev()) for _ in range(L)]

    class Marked(Step):
        def __call__(self):
            m, s = self.m, self.s
            with torch.cuda.stream(s):
                for l in range(1, L + 1):
                    rt.param_wait(l, s)
                    ff[l - 1][0].record(s)
                    m.forward_layer(l, s)
                    ff[l - 1][1].record(s)
                m.zero_grad()
                for l in range(L, 0, -1):
                    bp[l - 1][0].record(s)
                    m.backward_layer(l, s)
                    bp[l - 1][1].record(s)
                    rt.grad_ready(l, s)
                rt.step(s)
                rt.join(s)

    rt.set_timing(True)
    run = make_runner(Marked(model, rt, stream), True, stream)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    run()
    torch.cuda.synchronize()
    st_i = rt.timeline(t0)
    bp_i = [(f"BP l{l}", t0.elapsed_time(bp[l - 1][0]), t0.elapsed_time(bp[l - 1][1]))
            for l in range(L, 0, -1)]
    run()
    torch.cuda.synchronize()
    st_n = rt.timeline(t0)
    ff_n = [(f"FF l{l}", t0.elapsed_time(ff[l - 1][0]), t0.elapsed_time(ff[l - 1][1]))
            for l in range(1, L + 1)]
    # Reduction side from replay i; an all-gather from replay i when it ran in
    # that replay's backprop window (WFBP, back-filled DeAR), else from replay
    # i+1 (deferred into the next forward).
    bp0 = bp_i[0][1]
    stamps, ends_i, starts_n = [], [], []
    for si, sn in zip(st_i, st_n):
        s = dict(si)
        if not (si["ag0"] is not None and si["ag0"] >= bp0):
            for k in ("ag0", "ag1", "unpack1"):
                s[k] = sn[k]
            if sn["ag0"] is not None:
                starts_n.append(sn["ag0"])
        stamps.append(s)
        ends_i += [v for k, v in s.items() if v is not None and k in ("pack1", "rs1", "update1")]
        if si["ag0"] is not None and si["ag0"] >= bp0:
            ends_i += [v for v in (si["ag1"], si["unpack1"]) if v is not None]
    buckets = rt.buckets()
    rt.set_timing(False)
    rt.synchronize()
    rt.close()
    tl = T.build(bp_i + ff_n, buckets, stamps, a.policy)
    if rank != 0:
        return None
    if a.timeline_out:
        with open(a.timeline_out, "w") as f:
            f.write(T.dumps(tl))
    comm_ev = [e for e in tl["events"] if e["resource"] == "Comm"]
    # The two replays are separated by a host sync: the iteration is the BP
    # window of replay i (to its last comm event) plus the FF window of replay
    # i+1 (from its first comm event), without the gap in between.
    bp_win = max([bp_i[-1][2]] + ends_i) - bp0
    ff_win = ff_n[-1][2] - min([ff_n[0][1]] + starts_n)
    it = bp_win + ff_win
    return {"framing": "BP of replay i + FF of replay i+1 (the reference's iteration)",
            "iteration_ms": it, "bp_window_ms": bp_win, "ff_window_ms": ff_win,
            "ff_ms": tl["ff_ms"], "bp_ms": tl["bp_ms"],
            "exposed_comm_ms": max(0.0, it - tl["ff_ms"] - tl["bp_ms"]), "compute_events": 2 * L,
            "comm_events": len(comm_ev), "violations": tl["violations"]}


def _bench_parity(a, model, comm, rank, world, stream):
    """Oracle parity at the bench configuration (a checker, run after all
    timing): the bench's own runtime (same policy, buffer, backend, kernels)
    driven for --parity-steps S-SGD steps on seeded inputs (the reference
    tests' generator: w0 seed 77, rank r's gradients row r of seed 1000+step),
    then the largest bucket is compared with the oracle's fp32 ring-order
    restatement (bit-exact expected) and its fp64 sgd_step (collective.cpp:
    166-194; max relative deviation, tolerance 1e-5)."""
    import numpy as np
    import torch

    import paper_2302_12445_b200 as dear
    from oracle.lib import Restated

    o = Restated()
    rt = dear.Runtime(comm, rank, world, policy=a.policy, fusion_buffer_bytes=a.buffer,
                      lr=a.lr, momentum=a.momentum, backend=a.backend, stream=stream,
                      heap=model.heap if a.backend == "nvls" else None)
    for l in range(1, model.L + 1):
        rt.register(l, model.params[l - 1], model.grads[l - 1], model.shadows[l - 1])
    rt.finalize()
    buckets = rt.buckets()
    gi = max(range(len(buckets)), key=lambda i: buckets[i]["elems"])
    lo, hi, d = buckets[gi]["low"], buckets[gi]["high"], buckets[gi]["elems"]
    layers = list(range(lo, hi + 1))
    offs = np.cumsum([0] + [model.numels[l - 1] for l in layers])
    w0 = o.random_vectors_f32(1, d, 77)[0]
    with torch.cuda.stream(stream):
        model.params_flat.zero_()
        for j, l in enumerate(layers):
            model.params[l - 1].copy_(torch.from_numpy(w0[offs[j]:offs[j + 1]]))
    torch.cuda.synchronize()
    P, S = world, a.parity_steps
    for s in range(S):
        g = o.random_vectors_f32(P, d, 1000 + s)
        with torch.cuda.stream(stream):
            for l in range(1, model.L + 1):
                rt.param_wait(l, stream)
            model.grads_flat.zero_()
            for j, l in enumerate(layers):
                model.grads[l - 1].copy_(torch.from_numpy(g[rank, offs[j]:offs[j + 1]]))
            for l in range(model.L, 0, -1):
                rt.grad_ready(l, stream)
            rt.step(stream)
    rt.synchronize()
    torch.cuda.synchronize()
    got = torch.cat([model.params[l - 1].detach().float() for l in layers]).cpu().numpy()
    same = rt.check_replicas()
    backend, zc = rt.backend, rt.zero_copy
    rt.close()
    if rank != 0:
        return None
    w32, buf, has = w0.copy(), np.zeros(d, np.float32), False
    w64 = w0.astype(np.float64)
    for s in range(S):
        g = o.random_vectors_f32(P, d, 1000 + s)
        w32, buf, has = o.sgd_step_f32(w32, buf, has, g, a.lr, a.momentum, 0.0, 0.0, False,
                                       (P & (P - 1)) == 0)
        if a.momentum:
            w64 = None
        else:
            w64 = o.sgd_step(w64, g.astype(np.float64), a.lr)
    rel = None
    if w64 is not None:
        rel = float(np.max(np.abs(got - w64) / np.maximum(1.0, np.abs(w64))))
    return {"bucket": gi + 1, "layers": [lo, hi], "elems": d, "steps": S, "ranks": P,
            "collectives": backend, "zero_copy": zc,
            "bit_exact_fp32_ring": bool(np.array_equal(got, w32)),
            "max_rel_vs_fp64": rel, "tolerance": 1e-5,
            "within_tolerance": rel is not None and rel <= 1e-5,
            "replicas_identical": bool(same),
            "oracle": "oracle/dear_oracle.c sgd_step_f32 (ring order) and sgd_step (fp64)"}


def _ncu_traffic(workload):
    """DRAM bytes per GEMM launch from the committed ncu --set full capture
    (profiles/r02z_ncu_traffic.json, the final tree's), or None when none was
    taken for this workload."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        "r02z_ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)[workload]["gemm_traffic_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def _time_gemms(model, rt, stream):
    """Average GEMM launch time inside one eager DeAR step (events between the
    layer GEMMs on the compute stream)."""
    import torch

    evs = []
    with torch.cuda.stream(stream):
        for l in range(1, model.L + 1):
            rt.param_wait(l, stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            model.forward_layer(l, stream)
            e1.record(stream)
            evs.append((e0, e1, model.ff[l - 1].flops))
        model.zero_grad()
        for l in range(model.L, 0, -1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            model.backward_layer(l, stream)
            e1.record(stream)
            evs.append((e0, e1, model.wgrad[l - 1].flops + model.dgrad[l - 1].flops))
            rt.grad_ready(l, stream)
        rt.step(stream)
    torch.cuda.synchronize()
    ms = sum(e0.elapsed_time(e1) for e0, e1, _ in evs)
    return ms, sum(f for _, _, f in evs)


def _isolated_stage_times(model, runtime, stream, policy, reps=20):
    """pack / update / unpack (and the P = 1 direct update) per step with no
    GEMMs running: each stage's kernel over every bucket, `reps` rounds
    captured as one CUDA graph (dear_bench_stage) and timed with CUDA events
    on `stream`, so a launch's average duration carries no host launch gap.
    Returns {stage: (ms per step, launches per step)}."""
    import torch

    import paper_2302_12445_b200 as dear

    # DEAR_DIRECT=0: at P = 1 keep the separate pack / update / unpack kernels
    # (what every P > 1 NCCL bucket runs) next to the fused direct update.
    os.environ["DEAR_DIRECT"] = "0"
    try:
        rt = runtime(policy)
    finally:
        os.environ.pop("DEAR_DIRECT", None)
    rt_dir = runtime(policy) if rt.world_size == 1 else None
    nb = len(rt.buckets())
    out = {}
    for k, r in (("pack", rt), ("update", rt), ("unpack", rt), ("direct", rt_dir)):
        if r is None:
            continue
        try:
            with torch.cuda.stream(stream):
                r.bench_stage(k, 2, stream)
        except dear.InvalidArgument:  # no direct-update tables (momentum)
            continue
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            r.bench_stage(k, reps, stream)
        with torch.cuda.stream(stream):
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
        torch.cuda.synchronize()
        out[k] = (e0.elapsed_time(e1) / reps, nb)
        del g
    rt.close()
    if rt_dir is not None:
        rt_dir.close()
    # the stages rewrote parameters with synthetic values: restore sane ones
    model.params_flat.uniform_(-0.02, 0.02)
    model.grads_flat.zero_()
    return out


def _policy_pair(a, model, comm, world, rank, stream, batch, steps, warm, backend=None,
                 buffer=None):
    """DeAR vs WFBP on `model` (same kernels, same fusion buffer), graph-replayed
    steps, max over ranks. Also the measured per-step comm-stream times of the
    DeAR runtime's comm-only iterations (t_rs = pack + RS + update side,
    t_ag = AG + unpack side; make_runtime measures them for its dispatch order)."""
    import argparse

    ab = argparse.Namespace(**vars(a))
    if backend is not None:
        ab.backend = backend
    if buffer is not None:
        ab.buffer = buffer
    res = {}
    stage_ms = None
    for policy in (a.policy, a.baseline_policy):
        rt = make_runtime(ab, model, comm, rank, world, stream, policy, True)
        res["collectives"] = rt.backend
        res["zero_copy"] = bool(getattr(rt, "zero_copy", False))
        if rt.comm_order_info:
            info = rt.comm_order_info
            stage_ms = info["stage_ms"]
            res["comm_order"] = {k: v for k, v in info.items()
                                 if k in ("ags_during_backprop", "contention")}
            st, nb = info["stage_us_mean"], info["buckets"]
            res["t_rs_ms"] = nb * (st["pack"] + st["rs"] + st["update"]) / 1e3
            res["t_ag_ms"] = nb * (st["ag"] + st["unpack"]) / 1e3
        run = make_runner(Step(model, rt, stream), True, stream)
        ms = time_loop(run, steps, warm, stream, world > 1)
        rt.synchronize()
        rt.close()
        res[policy] = {"ms_per_step": ms, "samples_per_s": batch * world / (ms / 1e3)}
    if stage_ms is not None and model.tiles:
        # the reference's scheduler (simulate.cpp:65-159 via
        # costmodel.predict_iteration) fed with this run's measured per-layer
        # GEMM chain times and per-bucket comm-only stage times, against the
        # measured graph-replayed steps. Same buckets for both policies (same
        # fusion buffer); WFBP's all-reduce = RS + AG.
        from paper_2302_12445_b200 import costmodel

        L = model.L
        t_ff = [model.tiles["ff"]["us"] * 1e-6] * L
        t_bp = [model.tiles["bp_group_us"] * 1e-6] * L
        lb = [4 * n for n in model.numels]
        rs = [x[0] * 1e-3 for x in stage_ms]
        ag = [x[1] * 1e-3 for x in stage_ms]
        pred = {}
        for policy in (a.policy, a.baseline_policy):
            gd = bool(a.group_dependency) and policy.startswith("DEAR")
            sim = costmodel.predict_iteration(lb, t_ff, t_bp, policy, ab.buffer, world, 0.0, 0.0,
                                              group_dependency=gd, rs_times=rs, ag_times=ag)
            meas = res[policy]["ms_per_step"]
            pred[policy] = {"predicted_ms": sim["iteration_seconds"] * 1e3, "measured_ms": meas,
                            "measured_over_predicted": meas / (sim["iteration_seconds"] * 1e3)}
        pred["predicted_dear_over_wfbp"] = (pred[a.baseline_policy]["predicted_ms"] /
                                            pred[a.policy]["predicted_ms"])
        res["simulated"] = pred
    return res


def _priority_partition(a, model, comm, world, rank, stream, batch, steps, warm):
    """The ByteScheduler baseline of the reference (PRIORITY_PARTITION,
    task_graph.cpp:215-258) on the same kernels: every layer's all-reduce in
    parts of --partition-bytes, dispatched in the order the reference scheduler
    gives on this run's measured per-layer GEMM times and per-part comm-only
    stage times (the negotiation has no runtime counterpart)."""
    import torch

    import paper_2302_12445_b200 as dear
    from paper_2302_12445_b200 import costmodel

    rt = dear.Runtime(comm, rank, world, policy="PRIORITY_PARTITION", lr=a.lr,
                      momentum=a.momentum, backend=a.backend, stream=stream,
                      partition_bytes=a.partition_bytes,
                      heap=model.heap if a.backend == "nvls" else None)
    for l in range(1, model.L + 1):
        rt.register(l, model.params[l - 1], model.grads[l - 1], model.shadows[l - 1])
    rt.finalize()
    rt.set_timing(True)
    for _ in range(3):
        with torch.cuda.stream(stream):
            for l in range(1, model.L + 1):
                rt.param_wait(l, stream)
            for l in range(model.L, 0, -1):
                rt.grad_ready(l, stream)
            rt.step(stream)
        rt.synchronize()
    st = rt.timings()
    rt.set_timing(False)
    ar = [sum(v for v in (x["pack"], x["rs"], x["update"], x["ag"], x["unpack"]) if v) * 1e-3
          for x in st]
    L = model.L
    t_ff = [model.tiles["ff"]["us"] * 1e-6] * L
    t_bp = [model.tiles["bp_group_us"] * 1e-6] * L
    sim = costmodel.predict_iteration([4 * n for n in model.numels], t_ff, t_bp,
                                      "PRIORITY_PARTITION", 0, world, 0.0, 0.0,
                                      partition_bytes=a.partition_bytes,
                                      negotiation_rounds=0, ar_times=ar)
    order = torch.tensor(sim["comm_order"], dtype=torch.int32, device="cuda")
    if world > 1:
        torch.distributed.broadcast(order, 0)
    rt.set_comm_order(order.cpu().tolist())
    run = make_runner(Step(model, rt, stream), True, stream)
    ms = time_loop(run, steps, warm, stream, world > 1)
    rt.synchronize()
    rt.close()
    return {"partition_bytes": a.partition_bytes, "parts": len(st), "ms_per_step": ms,
            "samples_per_s": batch * world / (ms / 1e3),
            "predicted_ms": sim["iteration_seconds"] * 1e3}


def buffer_sweep(a, wl_name, comm, world, rank, stream):
    """BASELINE config 3: DeAR vs WFBP on the BERT-Base-shaped layers over a
    fusion-buffer sweep (same kernels, default transport), each measured step
    beside the reference scheduler's prediction on this run's measured stage
    times (simulate.cpp:65-159)."""
    import torch

    from paper_2302_12445_b200.presets import preset_param_counts
    from paper_2302_12445_b200.synthetic import SyntheticModel

    wl = WORKLOADS[wl_name]
    steps, warm = max(5, a.steps // 2), max(3, a.warmup)
    batch = wl["batch"]
    model = SyntheticModel(preset_param_counts(wl["preset"]), wl["hidden"],
                           batch * wl["tokens_per_sample"], seed=4321)
    run = make_runner(Step(model, None, stream), True, stream)
    comp = time_loop(run, steps, warm, stream, True)
    out = {"workload": wl["config"], "batch_per_gpu": batch, "compute_only_ms": comp,
           "steps": steps, "warmup": warm, "buffers": {}}
    for buf in (int(x) for x in a.buffer_sweep_bytes.split(",") if x.strip()):
        r = _policy_pair(a, model, comm, world, rank, stream, batch, steps, warm, buffer=buf)
        d, w = r[a.policy]["ms_per_step"], r[a.baseline_policy]["ms_per_step"]
        row = {"DEAR_ms": d, "WFBP_ms": w, "dear_over_wfbp": w / d,
               "exposed_comm_pct": max(0.0, 100 * (d - comp) / d),
               "wfbp_exposed_comm_pct": max(0.0, 100 * (w - comp) / w),
               "collectives": r.get("collectives")}
        if "simulated" in r:
            row["predicted_DEAR_ms"] = r["simulated"][a.policy]["predicted_ms"]
            row["predicted_WFBP_ms"] = r["simulated"][a.baseline_policy]["predicted_ms"]
        out["buffers"][str(buf)] = row
    model.close()
    del model
    torch.cuda.empty_cache()
    return out


def compare_policies(a, wl_name, comm, world, rank, stream):
    """DeAR vs WFBP (same kernels, same fusion buffer) and compute-only on a
    second workload: the north-star comparison (BERT-Large-shaped layers).

    Next to the measured step times: the measured t_ff / t_bp (tile tuner's
    per-layer chain times x L) and t_rs / t_ag (comm-only iterations) with the
    reference's Eq. 7 (DeAR) / Eq. 8 (all-reduce) predictions
    (analysis.cpp:50-60). DeAR's edge over WFBP exists only where t_rs + t_ag
    exceeds t_bp (SURVEY §7 "hard parts"); with N > 1 the comparison is
    repeated at the batch that puts the measured t_ag at 1.25 t_ff, the band
    SURVEY §7 names (t_ag = 1.2-1.33 t_ff), when that batch differs from the
    paper's."""
    import torch

    from paper_2302_12445_b200 import costmodel
    from paper_2302_12445_b200.presets import preset_param_counts
    from paper_2302_12445_b200.synthetic import SyntheticModel

    wl = WORKLOADS[wl_name]
    dist_on = world > 1
    steps, warm = max(5, a.steps // 2), max(3, a.warmup)

    import paper_2302_12445_b200 as dear

    nvls_ok = world > 1 and dear.nvls_supported()

    def one(batch, with_nccl):
        _mark(f"north_star batch {batch}: start")
        model = SyntheticModel(preset_param_counts(wl["preset"]), wl["hidden"],
                               batch * wl["tokens_per_sample"], seed=4321,
                               symmetric=a.backend == "nvls" and world > 1)
        _mark("north_star: model built (tiles tuned)")
        out = {"batch_per_gpu": batch}
        run = make_runner(Step(model, None, stream), True, stream)
        comp = time_loop(run, steps, warm, stream, dist_on)
        _mark("north_star: compute-only timed")
        out["compute_only_ms"] = comp
        tiles = model.tiles or {}
        t_ff = tiles.get("ff", {}).get("us", 0.0) * model.L / 1e3
        t_bp = tiles.get("bp_group_us", 0.0) * model.L / 1e3
        # The resolved default backend first; with N > 1 also NCCL, the north
        # star's named transport (DeAR's edge over WFBP grows with comm cost),
        # and the NVLS transport (on its own symmetric-heap copy of the model).
        extra = []
        if with_nccl and world > 1 and a.backend != "nccl":
            extra.append("nccl")
        if with_nccl and nvls_ok and a.backend != "nvls":
            extra.append("nvls")
        for be in [None] + extra:
            m = model
            try:
                if be == "nvls":
                    m = SyntheticModel(preset_param_counts(wl["preset"]), wl["hidden"],
                                       batch * wl["tokens_per_sample"], seed=4321,
                                       symmetric=True)
                _mark(f"north_star: policy pair on {be or 'default'}")
                res = _policy_pair(a, m, comm, world, rank, stream, batch, steps, warm, be)
            except Exception as e:  # an optional transport must not sink the line
                if be is None:
                    raise
                out[be] = {"error": f"{type(e).__name__}: {e}"[:300]}
                continue
            finally:
                if m is not model:
                    m.close()
            d, w = res[a.policy]["ms_per_step"], res[a.baseline_policy]["ms_per_step"]
            res.update({"dear_over_wfbp": w / d,
                        "exposed_comm_pct": max(0.0, 100 * (d - comp) / d),
                        "wfbp_exposed_comm_pct": max(0.0, 100 * (w - comp) / w)})
            if "t_rs_ms" in res:
                t_rs, t_ag = res["t_rs_ms"], res["t_ag_ms"]
                eq = costmodel.theoretical_times(t_ff, t_bp, t_rs, t_ag)
                res["eq78"] = {"t_ff_ms": t_ff, "t_bp_ms": t_bp, "t_rs_ms": t_rs,
                               "t_ag_ms": t_ag, "eq7_dear_ms": eq["dear"],
                               "eq8_allreduce_ms": eq["baseline"],
                               "eq_ratio": eq["baseline"] / eq["dear"] if eq["dear"] else None,
                               "t_ag_over_t_ff": t_ag / t_ff if t_ff else None}
            if be is None:
                if with_nccl and world > 1 and not a.no_priority_partition:
                    try:
                        pp = _priority_partition(a, m, comm, world, rank, stream, batch, steps,
                                                 warm)
                        pp["dear_over_pp"] = pp["ms_per_step"] / res[a.policy]["ms_per_step"]
                    except Exception as e:
                        pp = {"error": f"{type(e).__name__}: {e}"[:300]}
                    res["priority_partition"] = pp
                out.update(res)
            else:
                out[be] = res
        if with_nccl and world > 1:
            # BASELINE configs 3/4 "fusion buffer sweep": the same comparison
            # with 10 MB buckets on the default transport, where per-bucket
            # costs make the step comm-bound and DeAR's reordering can matter.
            sw = {}
            for buf in (10_000_000,):
                r = _policy_pair(a, model, comm, world, rank, stream, batch, steps, warm,
                                 buffer=buf)
                d, w = r[a.policy]["ms_per_step"], r[a.baseline_policy]["ms_per_step"]
                sw[str(buf)] = {"DEAR_ms": d, "WFBP_ms": w, "dear_over_wfbp": w / d,
                                "exposed_comm_pct": max(0.0, 100 * (d - comp) / d)}
            out["buffer_sweep"] = sw
        model.close()
        del model
        torch.cuda.empty_cache()
        return out

    base = wl["batch"]
    out = {"workload": wl["config"], "fusion_buffer_bytes": a.buffer, "steps": steps,
           "warmup": warm}
    out.update(one(base, True))
    eq = out.get("eq78")
    if world > 1 and eq and eq["t_ag_ms"] > 0 and eq["t_ff_ms"] > 0 and not a.no_calibrate:
        # t_ff scales with the batch, t_ag does not: the batch with t_ag = 1.25 t_ff.
        # Rank 0 decides (the measurements are rank-local): every rank must run
        # the same collectives.
        b = int(round(base * eq["t_ag_ms"] / (1.25 * eq["t_ff_ms"])))
        b = max(4, min(b, 4 * base))
        bt = torch.tensor([b], dtype=torch.int64, device="cuda")
        torch.distributed.broadcast(bt, 0)
        b = int(bt.item())
        if abs(b - base) >= max(2, base // 8):
            cal = one(b, False)
            cal["rule"] = "batch with measured t_ag = 1.25 t_ff (SURVEY §7: 1.2-1.33)"
            out["calibrated_batch"] = cal
    if world > 1 and a.north_star_batches:
        # DeAR vs WFBP as the compute / comm ratio grows (same kernels, default
        # transport): per-layer compute scales with the batch, the buckets do not.
        sweep = {}
        for b in (int(x) for x in a.north_star_batches.split(",") if x.strip()):
            if b == base:
                continue
            r = one(b, False)
            d, w = r[a.policy]["ms_per_step"], r[a.baseline_policy]["ms_per_step"]
            sweep[str(b)] = {"compute_only_ms": r["compute_only_ms"], "DEAR_ms": d, "WFBP_ms": w,
                             "dear_over_wfbp": w / d, "exposed_comm_pct": r["exposed_comm_pct"],
                             "wfbp_exposed_comm_pct": r["wfbp_exposed_comm_pct"],
                             "samples_per_s": r[a.policy]["samples_per_s"]}
        out["batch_sweep"] = sweep
    return out


def main():
    a = parse()
    wl = WORKLOADS[a.workload]
    world = int(os.environ.get("WORLD_SIZE", a.gpus))
    rank = int(os.environ.get("RANK", 0))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if a.impl == "reference":
        reference_arm(a, wl, world, rank)
        return 0
    line = gpu_arm(a, wl, world, rank, local_rank)
    if line is not None:
        print(json.dumps(line), flush=True)
    if getattr(gpu_arm, "broken", None):
        # A post-headline section hit an error (recorded in the line); the
        # CUDA context / communicators may be unusable: leave without teardown.
        sys.stdout.flush()
        sys.stderr.flush()
        os._exit(0)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
