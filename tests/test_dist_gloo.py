"""Multi-process (world_size 2 and 3, gloo on CPU) checks of the N > 1 host
logic: NCCL-id bootstrap over torch.distributed, and the decoupled data path
run across real processes with the product's shard layout — rank r owns chunk
(r+1) mod P (collective.cpp:94), reduce-scatter = sum of slot r, shard-local
update, all-gather, unpack — ending bit-identical on every rank and equal to
the oracle's sgd_step."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import paper_2302_12445_b200 as dear
        from oracle.lib import Restated

        # 1) the NCCL unique id reaches every rank intact
        obj = [dear.Communicator.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert all(i == ids[0] and len(i) == 128 for i in ids)

        # 2) decoupled S-SGD over the product's bucket/shard layout
        o = Restated()
        numels = [1000, 4097, 3, 2049, 1, 513]
        L = len(numels)
        plan = dear.build_fusion_plan([4 * n for n in numels], 24_000)
        offs = np.concatenate([[0], np.cumsum(numels)])
        w = o.random_vectors(1, int(offs[-1]), 77)[0].astype(np.float32)
        lr = np.float32(0.05)
        prescale = (world & (world - 1)) == 0
        inv_p = np.float32(1.0 / world)
        for step in range(3):
            G = o.random_vectors(world, int(offs[-1]), 1000 + step).astype(np.float32)
            g = G[rank]
            for lo, hi in plan:
                a, b = int(offs[lo - 1]), int(offs[hi])
                d = b - a
                ranges = dear.chunk_ranges(d, world)
                S = dear.slot_stride(d, world)
                buf = np.zeros(world * S, np.float32)
                for c, (cb, ce) in enumerate(ranges):  # pack: chunk c -> slot owner(c)
                    slot = dear.chunk_owner(c, world)
                    v = g[a + cb:a + ce]
                    buf[slot * S: slot * S + (ce - cb)] = v * inv_p if prescale else v
                t = torch.from_numpy(buf)
                dist.all_reduce(t)  # sum; rank r keeps slot r (= reduce-scatter)
                own_c = dear.slot_chunk(rank, world)
                cb, ce = ranges[own_c]
                mean = t.numpy()[rank * S: rank * S + (ce - cb)]
                if not prescale:
                    mean = mean * inv_p
                shard = (w[a + cb:a + ce] - lr * mean).astype(np.float32)
                gathered = [torch.zeros(S) for _ in range(world)]
                sh = torch.zeros(S)
                sh[: ce - cb] = torch.from_numpy(shard)
                dist.all_gather(gathered, sh)
                for r in range(world):  # unpack: slot r carries chunk (r+1) mod P
                    c = dear.slot_chunk(r, world)
                    cb2, ce2 = ranges[c]
                    w[a + cb2:a + ce2] = gathered[r].numpy()[: ce2 - cb2]
        allw = [None] * world
        dist.all_gather_object(allw, w.tobytes())
        assert all(x == allw[0] for x in allw), "replicas diverged"
        # oracle (fp64 sgd_step per bucket) within 1e-5
        exp = o.random_vectors(1, int(offs[-1]), 77)[0]
        for step in range(3):
            G = o.random_vectors(world, int(offs[-1]), 1000 + step).astype(np.float32)
            for lo, hi in plan:
                a, b = int(offs[lo - 1]), int(offs[hi])
                exp[a:b] = o.sgd_step(exp[a:b], G[:, a:b].astype(np.float64), 0.05)
        ok = np.all(np.abs(w - exp) <= 1e-5 * np.maximum(1, np.abs(exp)))
        q.put((rank, bool(ok), L))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_decoupled_path_across_processes(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    res = [q.get(timeout=5) for _ in range(world)]
    assert all(ok for _, ok, _ in res)
