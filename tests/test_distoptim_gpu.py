"""DistOptim (the PyTorch integration) on one GPU.

P = 1: the direct-update path (no collectives). P = 2: two replicas in this
process on LocalGroup(2, "peer"), i.e. the multi-GPU zero-copy peer kernels
driven by the real autograd hooks (post-accumulate-grad -> dear_grad_ready,
forward pre-hook -> dear_param_wait). Both must match single-process
torch.optim.SGD on the averaged gradient within 1e-5 (the north star's
tolerance), including under an LR scheduler: the rate set by
``scheduler.step()`` between iterations applies to the next iteration's
updates, which the gradient hooks enqueue during backward.
"""
import numpy as np
import pytest
import torch

import paper_2302_12445_b200 as dear

pytestmark = pytest.mark.gpu


def _mlp(seed=0):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.ReLU(),
                               torch.nn.Linear(128, 96), torch.nn.ReLU(),
                               torch.nn.Linear(96, 10)).cuda()


def _close(model, ref, tol=1e-5):
    for p, q in zip(model.parameters(), ref.parameters()):
        a, b = p.detach().double().cpu().numpy(), q.detach().double().cpu().numpy()
        if not np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.abs(b))):
            return False
    return True


def _batches(P, steps, seed=42):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return [([torch.randn(16, 64, generator=g) for _ in range(P)],
             [torch.randint(0, 10, (16,), generator=g) for _ in range(P)]) for _ in range(steps)]


def _sched(opt):
    # warm-up from 0 then decay: the first update must use lr 0
    return torch.optim.lr_scheduler.LambdaLR(opt, lambda s: [0.0, 0.5, 1.0, 0.7, 0.3, 0.1, 0.05][s])


def _reference(P, data, kw, sched):
    ref = _mlp()
    ropt = torch.optim.SGD(ref.parameters(), foreach=False, **kw)
    rs = _sched(ropt) if sched else None
    for xs, ys in data:
        ropt.zero_grad()
        for r in range(P):
            torch.nn.functional.cross_entropy(ref(xs[r].cuda()), ys[r].cuda()).div(P).backward()
        ropt.step()
        if rs:
            rs.step()
    return ref


@pytest.mark.parametrize("kw", [dict(lr=0.1), dict(lr=0.1, momentum=0.9, weight_decay=1e-4)])
@pytest.mark.parametrize("sched", [False, True])
def test_distoptim_one_rank(kw, sched):
    data = _batches(1, 6)
    model = _mlp()
    base = torch.optim.SGD(model.parameters(), **kw)
    opt = dear.DistOptim(base, model, policy="DEAR_FUSED", fusion_buffer_bytes=20_000)
    s = _sched(base) if sched else None
    for xs, ys in data:
        torch.nn.functional.cross_entropy(model(xs[0].cuda()), ys[0].cuda()).backward()
        opt.step()
        opt.zero_grad()
        if s:
            s.step()
    opt.synchronize()
    ok = _close(model, _reference(1, data, kw, sched))
    opt.close()
    assert ok


@pytest.mark.parametrize("kw", [dict(lr=0.1), dict(lr=0.1, momentum=0.9, weight_decay=1e-4)])
@pytest.mark.parametrize("sched", [False, True])
@pytest.mark.parametrize("policy,buf", [("DEAR_FUSED", 20_000), ("WFBP", 0)])
def test_distoptim_two_ranks_peer_kernels(kw, sched, policy, buf):
    P = 2
    data = _batches(P, 6)
    group = dear.LocalGroup(P, "peer")
    streams = [torch.cuda.Stream() for _ in range(P)]
    models, opts, scheds = [], [], []
    for r in range(P):
        m = _mlp()
        base = torch.optim.SGD(m.parameters(), **kw)
        opts.append(dear.DistOptim(base, m, comm=group, rank=r, policy=policy,
                                   fusion_buffer_bytes=buf, stream=streams[r]))
        models.append(m)
        scheds.append(_sched(base) if sched else None)
    torch.cuda.synchronize()
    group.connect()
    assert all(o.runtime.zero_copy for o in opts), "flat buffers must take the zero-copy path"
    for xs, ys in data:
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                loss = torch.nn.functional.cross_entropy(models[r](xs[r].cuda()), ys[r].cuda())
                loss.backward()
        for r in range(P):
            with torch.cuda.stream(streams[r]):
                opts[r].step()
                opts[r].zero_grad()
            if scheds[r]:
                scheds[r].step()
    for o in opts:
        o.synchronize()
    torch.cuda.synchronize()
    ref = _reference(P, data, kw, sched)
    ok = all(_close(m, ref) for m in models) and all(o.check_replicas() for o in opts)
    for o in opts:
        o.close()
    group.close()
    assert ok


def test_distoptim_without_model_joins_the_stream():
    """model=None: no forward pre-hooks, so step() itself makes the caller's
    stream wait for the all-gathers."""
    data = _batches(1, 3)
    model = _mlp()
    opt = dear.DistOptim(torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9), None,
                         policy="DEAR_FUSED", fusion_buffer_bytes=20_000)
    for xs, ys in data:
        torch.nn.functional.cross_entropy(model(xs[0].cuda()), ys[0].cuda()).backward()
        opt.step()
        opt.zero_grad()
    ok = _close(model, _reference(1, data, dict(lr=0.1, momentum=0.9), False))
    opt.close()
    assert ok
    with pytest.raises(ValueError):
        dear.DistOptim(torch.optim.SGD(_mlp().parameters(), lr=0.1), None, defer_allgather=True)
