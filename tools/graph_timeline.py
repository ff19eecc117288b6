#!/usr/bin/env python
"""Comm/compute timeline of one CUDA-graph-replayed step (the bench's timed
form), per bucket, on every rank; rank 0 prints a JSON summary.

    torchrun --nproc-per-node P tools/graph_timeline.py [--workload bert_large]
        [--policy DEAR_FUSED] [--group-dependency 1]

Compute-stream markers: step start (base), forward end, backward end, step
end. Comm stream: the runtime's per-bucket stamps (pack0, pack1, rs1,
update1, ag0, ag1, unpack1), all as ms from the step start.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="bert_large")
    ap.add_argument("--policy", default="DEAR_FUSED")
    ap.add_argument("--group-dependency", type=int, default=1)
    ap.add_argument("--contention", type=float, default=1.0)
    ap.add_argument("--buffer", type=int, default=25_000_000)
    ap.add_argument("--backend", default="auto")
    ap.add_argument("--out", default="")
    ap.add_argument("--clock-steps", type=int, default=0,
                    help="also replay this many steps under the nvidia-smi clock sampler")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import bench
    import paper_2302_12445_b200 as dear
    from paper_2302_12445_b200.presets import preset_param_counts
    from paper_2302_12445_b200.synthetic import SyntheticModel

    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    lr_ = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(lr_)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{lr_}"))
        comm = dear.init()
    wl = bench.WORKLOADS[a.workload]
    model = SyntheticModel(preset_param_counts(wl["preset"]), wl["hidden"],
                           wl["batch"] * wl["tokens_per_sample"], seed=1234)
    stream = torch.cuda.Stream()
    ns = argparse.Namespace(group_dependency=a.group_dependency, buffer=a.buffer, lr=0.05,
                            momentum=0.0, backend=a.backend, contention=a.contention,
                            order_search=1)
    if a.policy == "NONE":  # compute only: the same marks without the runtime
        class _NoRt:
            comm_order_info = None

            def __getattr__(self, name):
                return lambda *args, **kw: None

            def timeline(self, base):
                return []
        rt = _NoRt()
    else:
        rt = bench.make_runtime(ns, model, comm, rank, world, stream, a.policy, True)
    # external: recorded inside the graph capture, timed after a replay
    ev = {k: torch.cuda.Event(enable_timing=True, external=True)
          for k in ("base", "ff", "bp", "end")}

    class Marked(bench.Step):
        def __call__(self):
            m, s = self.m, self.s
            with torch.cuda.stream(s):
                ev["base"].record(s)
                for l in range(1, m.L + 1):
                    rt.param_wait(l, s)
                    m.forward_layer(l, s)
                ev["ff"].record(s)
                m.zero_grad()
                for l in range(m.L, 0, -1):
                    m.backward_layer(l, s)
                    rt.grad_ready(l, s)
                ev["bp"].record(s)
                rt.step(s)
                rt.join(s)
                ev["end"].record(s)

    rt.set_timing(True)
    run = bench.make_runner(Marked(model, rt, stream), True, stream)
    for _ in range(5):
        run()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    run()
    torch.cuda.synchronize()
    tl = rt.timeline(ev["base"])
    clocks = None
    if a.clock_steps:
        import time as _t
        with bench.ClockSampler(lr_) as clk:
            t0 = _t.time()
            for _ in range(a.clock_steps):
                run()
            torch.cuda.synchronize()
            wall = _t.time() - t0
        clocks = dict(clk.summary(), wall_ms_per_step=1e3 * wall / a.clock_steps)
        pw = [float(r[2]) for _, r in clk.rows if len(r) >= 7 and r[2].replace(".", "").isdigit() and float(r[2]) > 0]
        clocks["power_w_median"] = sorted(pw)[len(pw) // 2] if pw else None
    marks = {k: ev["base"].elapsed_time(ev[k]) for k in ("ff", "bp", "end")}
    out = {"rank": rank, "policy": a.policy, "gd": a.group_dependency, "marks_ms": marks,
           "clocks": clocks,
           "comm_order": rt.comm_order_info, "buckets": tl}
    # comm-stream busy time split by phase
    rs_spans = [(b["pack0"], b["update1"] if b["update1"] is not None else b["rs1"]) for b in tl
                if b["pack0"] is not None]
    ag_spans = [(b["ag0"], b["unpack1"] if b["unpack1"] is not None else b["ag1"]) for b in tl
                if b["ag0"] is not None]
    out["rs_busy_ms"] = sum(e - s for s, e in rs_spans if e is not None)
    out["ag_busy_ms"] = sum(e - s for s, e in ag_spans if e is not None)
    out["last_rs_end_ms"] = max((e for _, e in rs_spans if e is not None), default=None)
    out["ag_in_ff_phase"] = sum(1 for s, _ in ag_spans if s < marks["ff"])
    out["ag_in_bp_phase"] = sum(1 for s, _ in ag_spans if marks["ff"] <= s < marks["bp"])
    out["ag_after_bp"] = sum(1 for s, _ in ag_spans if s >= marks["bp"])
    if rank == 0:
        print(json.dumps({k: v for k, v in out.items() if k != "buckets"}), flush=True)
        if a.out:
            with open(a.out, "w") as f:
                json.dump(out, f)
    rt.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
