"""NVLS backend on one GPU (P = 1 multicast team): the multimem.ld_reduce
reduce-scatter + update and the multicast-store all-gather run through the
symmetric heap; with one rank the switch's sum is the gradient itself, so the
result must be BIT-EXACT with the fp32 restatement (collective.cpp:166-194).
The P = 2 / 4 parity runs in tests/dist_worker.py ("nvls")."""
import numpy as np
import pytest
import torch

from dear_harness import initial_weights, oracle_run, seeded_grads

pytestmark = pytest.mark.gpu

RAGGED = [1000, 4097, 3, 0, 2049, 1, 70001, 513, 12345, 7, 262144, 100003]


@pytest.fixture(scope="module", autouse=True)
def _need_nvls():
    import paper_2302_12445_b200 as dear

    if not dear.nvls_supported():
        pytest.skip("no NVLS multicast support on this GPU")


def _run(restated, policy, buf, steps, lr, shadow=False, **kw):
    import paper_2302_12445_b200 as dear

    numels = RAGGED
    offs = np.concatenate([[0], np.cumsum(numels)]).astype(np.int64)
    w0 = initial_weights(restated, numels)
    aoffs = [0]
    for n in numels:
        aoffs.append(aoffs[-1] + (n + 63) // 64 * 64)
    heap = dear.SymmetricHeap(4 * 3 * (aoffs[-1] + 64) + (1 << 16))
    pflat = heap.tensor(aoffs[-1] + 64).zero_()
    gflat = heap.tensor(aoffs[-1] + 64).zero_()
    shflat = heap.tensor(aoffs[-1] + 64, torch.bfloat16).zero_() if shadow else None
    rt = dear.Runtime(None, 0, 1, policy=policy, fusion_buffer_bytes=buf, lr=lr, heap=heap, **kw)
    params, grads, shadows = [], [], []
    for l in range(1, len(numels) + 1):
        n = numels[l - 1]
        p = pflat[aoffs[l - 1]:aoffs[l - 1] + n]
        p.copy_(torch.from_numpy(w0[offs[l - 1]:offs[l]].copy()))
        g = gflat[aoffs[l - 1]:aoffs[l - 1] + n]
        sh = shflat[aoffs[l - 1]:aoffs[l - 1] + max(n, 1)] if shadow else None
        rt.register(l, p, g, sh)
        params.append(p)
        grads.append(g)
        shadows.append(sh)
    rt.finalize()
    assert rt.backend == "nvls"
    for step in range(steps):
        G = seeded_grads(restated, 1, numels, step)
        for l in range(1, len(numels) + 1):
            rt.param_wait(l)
        for l in range(len(numels), 0, -1):
            grads[l - 1].copy_(torch.from_numpy(G[0, offs[l - 1]:offs[l]].copy()))
            rt.grad_ready(l)
        rt.step()
    rt.synchronize()
    torch.cuda.synchronize()
    w = torch.cat(params).cpu().numpy()
    sh = torch.cat([s[:n] for s, n in zip(shadows, numels)]).float().cpu().numpy() if shadow else None
    rt.close()
    heap.close()
    return w, sh


@pytest.mark.parametrize("policy,buf", [("DEAR_FUSED", 100_000), ("DEAR", 0),
                                        ("WFBP_FUSED", 400_000), ("WFBP", 0)])
def test_nvls_single_rank_bit_exact(restated, policy, buf):
    w, _ = _run(restated, policy, buf, 3, 0.05)
    assert np.array_equal(w, oracle_run(restated, RAGGED, 1, 3, policy, buf, 0.05, f32=True))


def test_nvls_momentum_and_bf16_copy(restated):
    kw = dict(momentum=0.9, weight_decay=1e-3, nesterov=True)
    w, sh = _run(restated, "DEAR_FUSED", 200_000, 4, 0.02, shadow=True, **kw)
    assert np.array_equal(w, oracle_run(restated, RAGGED, 1, 4, "DEAR_FUSED", 200_000, 0.02,
                                        f32=True, **kw))
    assert np.array_equal(sh, torch.from_numpy(w).to(torch.bfloat16).float().numpy())


def test_distoptim_nvls_single_rank():
    import paper_2302_12445_b200 as dear

    torch.manual_seed(0)
    model = torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.ReLU(),
                                torch.nn.Linear(128, 10)).cuda()
    ref = torch.nn.Sequential(torch.nn.Linear(64, 128), torch.nn.ReLU(),
                              torch.nn.Linear(128, 10)).cuda()
    ref.load_state_dict(model.state_dict())
    opt = dear.DistOptim(torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9), model,
                         backend="nvls", fusion_buffer_bytes=20_000)
    ropt = torch.optim.SGD(ref.parameters(), lr=0.1, momentum=0.9, foreach=False)
    g = torch.Generator().manual_seed(1)
    for _ in range(4):
        x, y = torch.randn(16, 64, generator=g).cuda(), torch.randint(0, 10, (16,), generator=g).cuda()
        torch.nn.functional.cross_entropy(model(x), y).backward()
        opt.step()
        opt.zero_grad()
        ropt.zero_grad()
        torch.nn.functional.cross_entropy(ref(x), y).backward()
        ropt.step()
    opt.synchronize()
    for p, q in zip(model.parameters(), ref.parameters()):
        torch.testing.assert_close(p, q, rtol=1e-5, atol=1e-6)
    opt.close()
