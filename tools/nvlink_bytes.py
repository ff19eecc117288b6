#!/usr/bin/env python
"""NVLink bytes moved by the bucket collectives, per transport, from the
GPUs' own NVLink data counters (NVML NVLink throughput fields, the counters
behind `nvidia-smi nvlink -gt d`) read before and after K comm-only DeAR
iterations of one bucket. ncu cannot replay a kernel that waits on another
GPU, so this is the NVLink-byte evidence for the peer / NVLS kernels; the
algorithmic bytes per iteration are printed beside it.

    torchrun --nproc-per-node P tools/nvlink_bytes.py [--mb 64] [--iters 50]
        [--backends nccl,zc,nvls]

Rank 0 prints one JSON line per transport: TX / RX bytes per iteration of
every GPU (max over GPUs), the per-GPU algorithmic bytes of RS + AG, and the
elapsed comm time.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def nvlink_kib(index: int) -> tuple[int, int]:
    """Cumulative NVLink TX / RX bytes over all links of GPU `index`: the per-link
    NVLINK_COUNT_XMIT/RCV_BYTES fields (Blackwell), else the device-wide
    THROUGHPUT_DATA / THROUGHPUT_RAW counters (KiB)."""
    import pynvml as N

    h = N.nvmlDeviceGetHandleByIndex(index)
    links = int(getattr(N, "NVML_NVLINK_MAX_LINKS", 18))
    tx = rx = 0
    ok = False
    for link in range(links):
        try:
            vals = N.nvmlDeviceGetFieldValues(h, [(N.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES, link),
                                                  (N.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES, link)])
        except Exception:
            break
        if any(v.nvmlReturn != 0 for v in vals):
            continue
        ok = True
        tx += int(vals[0].value.ullVal)
        rx += int(vals[1].value.ullVal)
    if ok:
        nvlink_kib.source = "NVML NVLINK_COUNT_XMIT/RCV_BYTES, summed over links"
        return tx, rx
    for ftx, frx in ((N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX),
                     (N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX, N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX)):
        vals = N.nvmlDeviceGetFieldValues(h, [ftx, frx])
        if all(v.nvmlReturn == 0 for v in vals):
            nvlink_kib.source = f"NVML field {ftx}/{frx} (KiB)"
            return int(vals[0].value.ullVal) * 1024, int(vals[1].value.ullVal) * 1024
    raise RuntimeError("no NVLink byte counter is readable through NVML on this GPU")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=int, default=64)
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--backends", default="nccl,zc,nvls")
    a = ap.parse_args()
    import pynvml
    import torch
    import torch.distributed as dist

    import paper_2302_12445_b200 as dear

    pynvml.nvmlInit()
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    lr = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lr)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    comm = dear.init()
    s = torch.cuda.Stream()
    n = a.mb * (1 << 20) // 4
    for backend in a.backends.split(","):
        heap = None
        if backend == "nvls":
            if not dear.nvls_supported():
                continue
            heap = dear.SymmetricHeap(8 * n + (1 << 20))
            p, g = heap.tensor(n).zero_(), heap.tensor(n).fill_(1.0)
        else:
            p, g = torch.zeros(n, device="cuda"), torch.ones(n, device="cuda")
        rt = dear.Runtime(comm, rank, P, policy="DEAR", lr=0.0, stream=s,
                          backend={"zc": "peer"}.get(backend, backend), heap=heap)
        rt.register(1, p, g)
        rt.finalize()

        def it():
            with torch.cuda.stream(s):
                rt.param_wait(1, s)
                rt.grad_ready(1, s)
                rt.step(s)

        for _ in range(5):
            it()
        rt.synchronize()
        torch.cuda.synchronize()
        dist.barrier()
        tx0, rx0 = nvlink_kib(lr)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(a.iters):
            it()
        rt.join(s)
        e1.record(s)
        rt.synchronize()
        torch.cuda.synchronize()
        tx1, rx1 = nvlink_kib(lr)
        dist.barrier()
        t = torch.tensor([(tx1 - tx0) * 1.0 / a.iters, (rx1 - rx0) * 1.0 / a.iters,
                          e0.elapsed_time(e1) / a.iters], device="cuda", dtype=torch.float64)
        allv = [torch.zeros_like(t) for _ in range(P)]
        dist.all_gather(allv, t)
        stride = rt.buckets()[0]["slot_stride"]
        rt.close()
        if heap is not None:
            heap.close()
        if rank == 0:
            # per GPU and iteration: RS moves (P-1)/P of the bucket out and in,
            # AG the same (ring / pull convention); NVLS moves the whole bucket
            # out (ld_reduce) and in (multicast store) per GPU.
            alg = 2 * (P - 1) * stride * 4
            print(json.dumps({
                "backend": backend, "P": P, "bucket_bytes": 4 * n, "iters": a.iters,
                "tx_bytes_per_iter": [v[0].item() for v in allv],
                "rx_bytes_per_iter": [v[1].item() for v in allv],
                "comm_ms_per_iter": max(v[2].item() for v in allv),
                "alg_bytes_per_gpu_ring_convention": alg,
                "source": nvlink_kib.source}),
                flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
