#!/usr/bin/env python
"""Copy-engine peer bandwidth on one node (single process, P GPUs): D2D peer
copies (cudaMemcpyPeerAsync via torch) of one size, 1 copy and P-1 concurrent
pushes from GPU 0 (one stream per destination), optionally while GPU 0 runs a
GEMM chain (SM contention check)."""
import json
import sys

import torch


def main():
    P = torch.cuda.device_count()
    for i in range(P):
        for j in range(P):
            if i != j:
                assert torch.cuda.can_device_access_peer(i, j)
    sizes = [int(x * 2**20) for x in (1, 4, 6.25, 16, 25, 64)]
    out = []
    for nbytes in sizes:
        n = nbytes // 4
        src = torch.randn(n, device="cuda:0")
        dsts = [torch.empty(n, device=f"cuda:{j}") for j in range(1, P)]
        streams = [torch.cuda.Stream(device="cuda:0") for _ in range(P - 1)]
        res = {"bytes": nbytes}
        for conc in (1, P - 1):
            for _ in range(3):
                for k in range(conc):
                    with torch.cuda.stream(streams[k]):
                        dsts[k].copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            reps = 20
            cur = torch.cuda.current_stream()
            e0.record(cur)
            for k in range(conc):
                streams[k].wait_event(e0)
            for _ in range(reps):
                for k in range(conc):
                    with torch.cuda.stream(streams[k]):
                        dsts[k].copy_(src, non_blocking=True)
            for k in range(conc):
                cur.wait_stream(streams[k])
            e1.record(cur)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / reps
            res[f"conc{conc}_us"] = round(us, 2)
            res[f"conc{conc}_gbs_total"] = round(conc * nbytes / us / 1e3, 1)
        # pull: GPU 0 reads from P-1 peers concurrently (copies issued on GPU 0 streams)
        srcs = [torch.randn(n, device=f"cuda:{j}") for j in range(1, P)]
        dst0 = [torch.empty(n, device="cuda:0") for _ in range(P - 1)]
        torch.cuda.synchronize()
        cur = torch.cuda.current_stream()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        for k in range(P - 1):
            streams[k].wait_event(e0)
        for _ in range(20):
            for k in range(P - 1):
                with torch.cuda.stream(streams[k]):
                    dst0[k].copy_(srcs[k], non_blocking=True)
        for k in range(P - 1):
            cur.wait_stream(streams[k])
        e1.record(cur)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        res["pull_us"] = round(us, 2)
        res["pull_gbs_total"] = round((P - 1) * nbytes / us / 1e3, 1)
        out.append(res)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
