"""torchrun worker for the multi-GPU (NCCL over NVLink) parity tests.

    torchrun --nproc-per-node N tests/dist_worker.py <case>

case "runtime": the C-ABI runtime through NCCL on seeded gradients (the
reference tests' generator), every policy, 3 steps; parameters must be
bit-identical across ranks and within 1e-5 of the oracle's fp64 sgd_step
(per fusion bucket), momentum variant against the fp64 momentum restatement.
case "distoptim": DistOptim on a torch MLP, each rank its own micro-batch;
parameters must match single-process torch.optim.SGD on the averaged
gradient within 1e-5.
Exit code 0 = pass.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_2302_12445_b200 as dear  # noqa: E402
from dear_harness import initial_weights, oracle_run, seeded_grads  # noqa: E402
from oracle.lib import Restated  # noqa: E402

RAGGED = [1000, 4097, 3, 0, 2049, 1, 70001, 513, 12345, 7, 262144, 100003]


def close(a, b, tol=1e-5):
    return bool(np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.abs(b))))


def run_runtime(comm, rank, P, policy, buf, steps, lr, backend="nccl", comm_order=None,
                flat=False, shadow=False, **kw):  # explicit backend
    """flat=True: every layer's parameters (and gradients) are views of ONE flat
    tensor at 64-element aligned offsets, which lets the peer backend map them
    directly (zero-copy); the runtime must then report zero_copy."""
    o = Restated()
    numels = RAGGED
    offs = np.concatenate([[0], np.cumsum(numels)]).astype(np.int64)
    w0 = initial_weights(o, numels)
    s = torch.cuda.Stream()
    heap = None
    if backend == "nvls":
        flat = True
        heap = dear.SymmetricHeap(4 * 3 * (sum((n + 63) // 64 * 64 for n in numels) + 64)
                                  + (1 << 16))
    rt = dear.Runtime(comm, rank, P, policy=policy, fusion_buffer_bytes=buf, lr=lr, stream=s,
                      backend=backend, dear_group_dependency=comm_order is not None, heap=heap,
                      **kw)
    params, grads, shadows = [], [], []
    if flat:
        aoffs = [0]
        for n in numels:
            aoffs.append(aoffs[-1] + (n + 63) // 64 * 64)
        if heap is not None:
            pflat = heap.tensor(aoffs[-1] + 64).zero_()
            gflat = heap.tensor(aoffs[-1] + 64).zero_()
            shflat = heap.tensor(aoffs[-1] + 64, torch.bfloat16).zero_() if shadow else None
        else:
            pflat = torch.zeros(aoffs[-1] + 64, device="cuda")
            gflat = torch.zeros_like(pflat)
            shflat = torch.zeros(aoffs[-1] + 64, device="cuda", dtype=torch.bfloat16) \
                if shadow else None
    for l in range(1, len(numels) + 1):
        src = torch.from_numpy(w0[offs[l - 1]:offs[l]].copy()).cuda()
        if flat:
            p = pflat[aoffs[l - 1]:aoffs[l - 1] + numels[l - 1]]
            p.copy_(src)
            g = gflat[aoffs[l - 1]:aoffs[l - 1] + numels[l - 1]]
            sh = shflat[aoffs[l - 1]:aoffs[l - 1] + max(1, numels[l - 1])] if shadow else None
        else:
            p, g = src, torch.zeros_like(src)
            sh = None
        rt.register(l, p, g, sh)
        params.append(p)
        grads.append(g)
        shadows.append(sh)
    rt.finalize()
    if flat and backend == "peer" and os.environ.get("DEAR_ZERO_COPY", "1") != "0":
        assert rt.zero_copy, "flat parameters/gradients must enable the zero-copy peer path"
        if os.environ.get("DEAR_PUSH_RS") == "1":
            assert rt.push_rs, "DEAR_PUSH_RS=1 must take the push reduce-scatter"
    if comm_order is not None:
        rt.set_comm_order(comm_order)
    with torch.cuda.stream(s):
        for step in range(steps):
            G = seeded_grads(o, P, numels, step)
            for l in range(1, len(numels) + 1):
                rt.param_wait(l, s)
            for l in range(len(numels), 0, -1):
                grads[l - 1].copy_(torch.from_numpy(G[rank, offs[l - 1]:offs[l]].copy()))
                rt.grad_ready(l, s)
            rt.step(s)
    rt.synchronize()
    torch.cuda.synchronize()
    same = rt.check_replicas()
    trace = rt.trace()
    w = torch.cat([p for p in params]).cpu().numpy()
    if shadow:
        sh = torch.cat([x[:n] for x, n in zip(shadows, numels)]).float().cpu().numpy()
        run_runtime.shadow_ok = bool(np.array_equal(
            sh, torch.from_numpy(w).to(torch.bfloat16).float().numpy()))
    rt.close()
    if heap is not None:
        heap.close()
    return w, same, trace


def case_runtime(rank, P):
    comm = dear.init()
    o = Restated()
    ok = True
    for policy, buf in (("DEAR_FUSED", 100_000), ("DEAR", 0), ("WFBP_FUSED", 400_000),
                        ("WFBP", 0), ("DEAR_FUSED", 25_000_000), ("PRIORITY_PARTITION", 0)):
        pb = 40_000 if policy == "PRIORITY_PARTITION" else 0
        w, same, trace = run_runtime(comm, rank, P, policy, buf, 3, 0.05, partition_bytes=pb)
        exp = oracle_run(o, RAGGED, P, 3, policy, buf, 0.05, f32=False, partition_bytes=pb)
        allw = [torch.zeros_like(torch.from_numpy(w)).cuda() for _ in range(P)]
        dist.all_gather(allw, torch.from_numpy(w).cuda())
        bit_same = all(torch.equal(allw[0], x) for x in allw)
        good = same and bit_same and close(w.astype(np.float64), exp)
        if rank == 0:
            print(f"[runtime P={P}] {policy:11s} buf={buf:>9} replicas={same and bit_same} "
                  f"oracle_1e-5={close(w.astype(np.float64), exp)} trace0={trace[:2]}", flush=True)
        ok &= good
    kw = dict(momentum=0.9, weight_decay=1e-3, nesterov=True)
    w, same, _ = run_runtime(comm, rank, P, "DEAR_FUSED", 200_000, 4, 0.02, **kw)
    exp = oracle_run(o, RAGGED, P, 4, "DEAR_FUSED", 200_000, 0.02, f32=False, **kw)
    good = same and close(w.astype(np.float64), exp)
    if rank == 0:
        print(f"[runtime P={P}] momentum/wd/nesterov replicas={same} oracle_1e-5={good}",
              flush=True)
    ok &= good
    # dear_group_dependency: all-gathers back-filled between reduce-scatters
    from paper_2302_12445_b200 import costmodel as cm
    L = len(RAGGED)
    G = cm.predict_iteration([4 * n for n in RAGGED], [1.0] * L, [1.0] * L, "DEAR_FUSED",
                             100_000, P, 0.0, 0.0)["buckets"]
    order = cm.predict_iteration([4 * n for n in RAGGED], [0.5] * L, [1.0] * L, "DEAR_FUSED",
                                 100_000, P, 0.0, 0.0, group_dependency=True,
                                 rs_times=[1.5] * G, ag_times=[1.0] * G)["comm_order"]
    w, same, trace = run_runtime(comm, rank, P, "DEAR_FUSED", 100_000, 3, 0.05, "nccl",
                                 comm_order=order)
    exp32 = oracle_run(o, RAGGED, P, 3, "DEAR_FUSED", 100_000, 0.05, f32=True)
    exp64 = oracle_run(o, RAGGED, P, 3, "DEAR_FUSED", 100_000, 0.05, f32=False)
    want = [("RS g%d" % v) if v > 0 else ("AG g%d" % -v) for v in order]
    good = same and close(w.astype(np.float64), exp64) and trace == want and \
        True
    if rank == 0:
        print(f"[runtime P={P}] group_dependency order={order[:8]}.. replicas={same} "
              f"trace_is_order={trace == want} oracle_1e-5={close(w.astype(np.float64), exp64)}",
              flush=True)
    ok &= good
    comm.close()
    return ok



def case_peer(rank, P):
    """NVLink peer backend: fused RS+update / AG+unpack kernels sum in the
    reference's ring order, so parameters are BIT-EXACT with the fp32
    ring-order restatement (and within 1e-5 of the fp64 oracle)."""
    comm = dear.init()
    o = Restated()
    ok = True
    for flat in (False, True):
        for policy, buf in (("DEAR_FUSED", 100_000), ("DEAR", 0), ("WFBP_FUSED", 400_000),
                            ("WFBP", 0), ("DEAR_FUSED", 25_000_000), ("PRIORITY_PARTITION", 0)):
            pb = 40_000 if policy == "PRIORITY_PARTITION" else 0
            w, same, _ = run_runtime(comm, rank, P, policy, buf, 3, 0.05, backend="peer",
                                     flat=flat, partition_bytes=pb)
            exp32 = oracle_run(o, RAGGED, P, 3, policy, buf, 0.05, f32=True, partition_bytes=pb)
            exp64 = oracle_run(o, RAGGED, P, 3, policy, buf, 0.05, f32=False, partition_bytes=pb)
            good = same and np.array_equal(w, exp32) and close(w.astype(np.float64), exp64)
            if rank == 0:
                print(f"[peer P={P} {'zero-copy' if flat else 'slots'}] {policy:11s} "
                      f"buf={buf:>9} replicas={same} "
                      f"bit_exact_fp32_ring={np.array_equal(w, exp32)} "
                      f"oracle_1e-5={close(w.astype(np.float64), exp64)}", flush=True)
            ok &= good
        kw = dict(momentum=0.9, weight_decay=1e-3, nesterov=True)
        w, same, _ = run_runtime(comm, rank, P, "DEAR_FUSED", 200_000, 4, 0.02, backend="peer",
                                 flat=flat, **kw)
        exp32 = oracle_run(o, RAGGED, P, 4, "DEAR_FUSED", 200_000, 0.02, f32=True, **kw)
        good = same and np.array_equal(w, exp32)
        if rank == 0:
            print(f"[peer P={P} {'zero-copy' if flat else 'slots'}] momentum/wd/nesterov "
                  f"bit_exact={good}", flush=True)
        ok &= good
    # dear_group_dependency: all-gathers back-filled between reduce-scatters
    from paper_2302_12445_b200 import costmodel as cm
    L = len(RAGGED)
    G = cm.predict_iteration([4 * n for n in RAGGED], [1.0] * L, [1.0] * L, "DEAR_FUSED",
                             100_000, P, 0.0, 0.0)["buckets"]
    order = cm.predict_iteration([4 * n for n in RAGGED], [0.5] * L, [1.0] * L, "DEAR_FUSED",
                                 100_000, P, 0.0, 0.0, group_dependency=True,
                                 rs_times=[1.5] * G, ag_times=[1.0] * G)["comm_order"]
    w, same, trace = run_runtime(comm, rank, P, "DEAR_FUSED", 100_000, 3, 0.05, "peer",
                                 comm_order=order, flat=True)
    exp32 = oracle_run(o, RAGGED, P, 3, "DEAR_FUSED", 100_000, 0.05, f32=True)
    exp64 = oracle_run(o, RAGGED, P, 3, "DEAR_FUSED", 100_000, 0.05, f32=False)
    want = [("RS g%d" % v) if v > 0 else ("AG g%d" % -v) for v in order]
    good = same and close(w.astype(np.float64), exp64) and trace == want and \
        ("peer" == "nccl" or np.array_equal(w, exp32))
    if rank == 0:
        print(f"[peer P={P}] group_dependency order={order[:8]}.. replicas={same} "
              f"trace_is_order={trace == want} oracle_1e-5={close(w.astype(np.float64), exp64)}",
              flush=True)
    ok &= good
    comm.close()
    return ok



def case_push(rank, P):
    """Push reduce-scatter (DEAR_PUSH_RS=1): every rank writes each chunk of
    its gradients into its owner's push buffer over NVLink and the owner sums
    its slots in ring order — the peer case's checks, bit-exact, plus the bf16
    copy written by the push RS."""
    os.environ["DEAR_PUSH_RS"] = "1"
    ok = case_peer(rank, P)
    comm = dear.init()
    o = Restated()
    w, same, _ = run_runtime(comm, rank, P, "DEAR_FUSED", 100_000, 3, 0.05, backend="peer",
                             flat=True, shadow=True)
    exp32 = oracle_run(o, RAGGED, P, 3, "DEAR_FUSED", 100_000, 0.05, f32=True)
    good = same and np.array_equal(w, exp32) and run_runtime.shadow_ok
    if rank == 0:
        print(f"[push P={P}] bf16 copy + bit_exact={good}", flush=True)
    comm.close()
    return ok and good


def case_push_mismatch(rank, P):
    """DEAR_PUSH_RS set on rank 0 only: every rank's connect must fail with a
    clear error instead of running mismatched protocols."""
    os.environ["DEAR_PUSH_RS"] = "1" if rank == 0 else "0"
    comm = dear.init()
    try:
        run_runtime(comm, rank, P, "DEAR_FUSED", 100_000, 1, 0.05, backend="peer", flat=True)
        ok = False
    except dear.InvalidArgument as e:
        ok = "disagree on DEAR_PUSH_RS" in str(e)
        if rank == 0:
            print(f"[push mismatch] rejected: {e}", flush=True)
    comm.close()
    return ok


def case_nvls(rank, P):
    """NVLS backend: the switch sums each owned chunk (multimem.ld_reduce) and
    the owners broadcast with multicast stores. P = 2: a + b is order-free, so
    BIT-EXACT with the fp32 ring restatement; otherwise within 1e-5 of the
    fp64 oracle; replicas bit-identical (every rank stores the same bits)."""
    comm = dear.init()
    o = Restated()
    ok = True
    for policy, buf in (("DEAR_FUSED", 100_000), ("DEAR", 0), ("WFBP_FUSED", 400_000),
                        ("WFBP", 0), ("DEAR_FUSED", 25_000_000), ("PRIORITY_PARTITION", 0)):
        pb = 40_000 if policy == "PRIORITY_PARTITION" else 0
        w, same, trace = run_runtime(comm, rank, P, policy, buf, 3, 0.05, backend="nvls",
                                     shadow=True, partition_bytes=pb)
        exp32 = oracle_run(o, RAGGED, P, 3, policy, buf, 0.05, f32=True, partition_bytes=pb)
        exp64 = oracle_run(o, RAGGED, P, 3, policy, buf, 0.05, f32=False, partition_bytes=pb)
        bit = bool(np.array_equal(w, exp32))
        good = same and close(w.astype(np.float64), exp64) and run_runtime.shadow_ok and \
            (bit or P != 2)
        if rank == 0:
            print(f"[nvls P={P}] {policy:11s} buf={buf:>9} replicas={same} bit_exact_fp32_ring={bit}"
                  f" oracle_1e-5={close(w.astype(np.float64), exp64)} "
                  f"bf16_copy={run_runtime.shadow_ok}", flush=True)
        ok &= good
    kw = dict(momentum=0.9, weight_decay=1e-3, nesterov=True)
    w, same, _ = run_runtime(comm, rank, P, "DEAR_FUSED", 200_000, 4, 0.02, backend="nvls", **kw)
    exp64 = oracle_run(o, RAGGED, P, 4, "DEAR_FUSED", 200_000, 0.02, f32=False, **kw)
    good = same and close(w.astype(np.float64), exp64)
    if rank == 0:
        print(f"[nvls P={P}] momentum/wd/nesterov replicas={same} oracle_1e-5={good}", flush=True)
    ok &= good
    # group dependency: back-filled all-gathers
    from paper_2302_12445_b200 import costmodel as cm
    L = len(RAGGED)
    G = cm.predict_iteration([4 * n for n in RAGGED], [1.0] * L, [1.0] * L, "DEAR_FUSED",
                             100_000, P, 0.0, 0.0)["buckets"]
    order = cm.predict_iteration([4 * n for n in RAGGED], [0.5] * L, [1.0] * L, "DEAR_FUSED",
                                 100_000, P, 0.0, 0.0, group_dependency=True,
                                 rs_times=[1.5] * G, ag_times=[1.0] * G)["comm_order"]
    w, same, trace = run_runtime(comm, rank, P, "DEAR_FUSED", 100_000, 3, 0.05, "nvls",
                                 comm_order=order)
    exp64 = oracle_run(o, RAGGED, P, 3, "DEAR_FUSED", 100_000, 0.05, f32=False)
    want = [("RS g%d" % v) if v > 0 else ("AG g%d" % -v) for v in order]
    good = same and close(w.astype(np.float64), exp64) and trace == want
    if rank == 0:
        print(f"[nvls P={P}] group_dependency replicas={same} trace_is_order={trace == want} "
              f"oracle_1e-5={close(w.astype(np.float64), exp64)}", flush=True)
    ok &= good
    comm.close()
    return ok


def case_distoptim_nvls(rank, P):
    return case_distoptim(rank, P, backend="nvls")


def case_timeout(rank, P):
    """A peer that never arrives: rank 1 skips its gradients of one iteration.
    Rank 0's zero-copy reduce-scatter must give up after DEAR_PEER_TIMEOUT_S
    with a CUDA error (a trap), not hang the GPU."""
    import time

    comm = dear.init()
    s = torch.cuda.Stream()
    rt = dear.Runtime(comm, rank, P, policy="DEAR_FUSED", fusion_buffer_bytes=1 << 20, lr=0.1,
                      stream=s, backend="peer")
    p = torch.zeros(8192, device="cuda")
    g = torch.zeros(8192, device="cuda")
    rt.register(1, p[:4096], g[:4096])
    rt.register(2, p[4096:], g[4096:])
    rt.finalize()
    dist.barrier()
    ok = True
    if rank == 0:
        t0 = time.time()
        rt.grad_ready(2, s)
        rt.grad_ready(1, s)
        try:
            torch.cuda.synchronize()
            ok = False
            print("[timeout] rank 0: no error although rank 1 never arrived", flush=True)
        except Exception as e:  # the trap surfaces as a CUDA error
            dt = time.time() - t0
            ok = dt < 60
            print(f"[timeout] rank 0 trapped after {dt:.1f} s: {type(e).__name__}", flush=True)
        os._exit(0 if ok else 1)
    time.sleep(20)  # rank 1 never reports; exits after rank 0 gave up
    os._exit(0)


def case_distoptim(rank, P, backend="auto"):
    comm = dear.init()
    torch.manual_seed(0)
    layers = [torch.nn.Linear(64, 128), torch.nn.ReLU(), torch.nn.Linear(128, 96),
              torch.nn.ReLU(), torch.nn.Linear(96, 10)]
    model = torch.nn.Sequential(*layers).cuda()
    ref = torch.nn.Sequential(*[type(m)(*([m.in_features, m.out_features]
                                          if isinstance(m, torch.nn.Linear) else []))
                                for m in layers]).cuda()
    ref.load_state_dict(model.state_dict())
    kw = dict(lr=0.1, momentum=0.9, weight_decay=1e-4)
    opt = dear.DistOptim(torch.optim.SGD(model.parameters(), **kw), model, comm=comm,
                         policy="DEAR_FUSED", fusion_buffer_bytes=20_000, backend=backend)
    ropt = torch.optim.SGD(ref.parameters(), foreach=False, **kw)
    g = torch.Generator(device="cpu").manual_seed(42)
    for step in range(5):
        xs = [torch.randn(16, 64, generator=g) for _ in range(P)]
        ys = [torch.randint(0, 10, (16,), generator=g) for _ in range(P)]
        loss = torch.nn.functional.cross_entropy(model(xs[rank].cuda()), ys[rank].cuda())
        loss.backward()
        opt.step()
        opt.zero_grad()
        # reference: mean of the P micro-batch gradients, one process
        ropt.zero_grad()
        for r in range(P):
            torch.nn.functional.cross_entropy(ref(xs[r].cuda()), ys[r].cuda()).div(P).backward()
        ropt.step()
    opt.synchronize()
    ok = opt.check_replicas()
    for p, q in zip(model.parameters(), ref.parameters()):
        ok &= close(p.detach().double().cpu().numpy(), q.detach().double().cpu().numpy(), 1e-5)
    zc = opt.runtime.zero_copy
    if opt.runtime.backend == "peer":
        ok &= zc  # flat parameter / gradient buffers: the zero-copy path must engage
    if rank == 0:
        print(f"[distoptim P={P}] backend={opt.runtime.backend} zero_copy={zc} "
              f"match single-process SGD on averaged grads: {ok}", flush=True)
    opt.close()
    comm.close()
    return ok


def main():
    case = sys.argv[1]
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    ok = {"runtime": case_runtime, "distoptim": case_distoptim, "peer": case_peer,
          "nvls": case_nvls, "distoptim_nvls": case_distoptim_nvls, "push": case_push,
          "push_mismatch": case_push_mismatch,
          "timeout": case_timeout}[case](rank, P)
    t = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(t)
    dist.destroy_process_group()
    sys.exit(int(t.item() != 0))


if __name__ == "__main__":
    main()
