"""Numerics of the hand-written tcgen05 GEMM against a plain PyTorch fp32
reference of the same op (bf16 inputs, fp32 accumulate)."""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["auto", "single", "pair", "cluster"], autouse=True)
def tile_mode(request, monkeypatch):
    """Every case runs with the default tile choice, forced single-CTA tiles,
    forced 2-CTA pairs (cta_group::2) and opt-in TMA-multicast clusters."""
    env = {"auto": ("0", "1"), "single": ("0", "0"), "pair": ("0", "2"),
           "cluster": ("1", "0")}[request.param]
    monkeypatch.setenv("DEAR_GEMM_CLUSTER", env[0])
    monkeypatch.setenv("DEAR_GEMM_PAIR", env[1])
    return request.param


def _ref(a, b, mn_major):
    bb = b.float().t() if mn_major else b.float()
    return a.float() @ bb.t()


def _check(out, ref, K):
    # fp32 accumulation of bf16 products; different summation order than the
    # reference matmul: tolerance scales with sqrt(K).
    err = (out.float() - ref).abs().max().item()
    scale = ref.abs().max().item() + 1e-6
    assert err <= 2e-3 * scale * max(1.0, (K / 256) ** 0.5), (err, scale)


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 256, 1024), (4096, 825, 1024),
                                   (300, 100, 70), (1000, 520, 513), (129, 17, 8)])
@pytest.mark.parametrize("mn_major", [False, True])
def test_gemm_fp32_out(M, N, K, mn_major):
    from paper_2302_12445_b200.gemm import GemmPlan

    torch.manual_seed(M * 7 + N)
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    if mn_major:
        ldb = (N + 7) // 8 * 8
        bstore = torch.randn(K, ldb, device="cuda").to(torch.bfloat16)
        b = bstore[:, :N]
    else:
        ldk = (K + 7) // 8 * 8
        bstore = torch.randn(N, ldk, device="cuda").to(torch.bfloat16)
        b = bstore[:, :K]
    lda = (K + 7) // 8 * 8
    astore = torch.zeros(M, lda, device="cuda", dtype=torch.bfloat16)
    astore[:, :K] = a
    d = torch.full((M, N), float("nan"), device="cuda")
    plan = GemmPlan(astore, bstore, d, M, N, K, b_mn_major=mn_major, lda=lda,
                    ldb=bstore.stride(0), ldd=N)
    plan.run()
    torch.cuda.synchronize()
    _check(d, _ref(astore[:, :K], b, mn_major), K)


@pytest.mark.parametrize("M,N,K", [(825, 1024, 4096), (311, 512, 10240), (96, 64, 256)])
def test_gemm_splitk_accumulate_flat_limit(M, N, K):
    """Weight-gradient shape: D (flat, partial last row) += A @ B^T, split-K."""
    from paper_2302_12445_b200.gemm import GemmPlan

    torch.manual_seed(1)
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    limit = M * N - N // 3
    flat = torch.zeros(limit + 64, device="cuda")
    flat[limit:] = 12345.0  # sentinel past the bound must survive
    base = torch.randn(limit, device="cuda")
    flat[:limit] = base
    plan = GemmPlan(a, b, flat, M, N, K, ldd=N, d_limit=limit, accumulate=True)
    assert plan.info()["splits"] >= 1
    plan.run()
    torch.cuda.synchronize()
    ref = (a.float() @ b.float().t()).reshape(-1)[:limit] + base
    _check(flat[:limit], ref, K)
    assert torch.all(flat[limit:] == 12345.0)
    # split-K override (plan-time tuner): accumulates once more, same result
    plan.set_splits(3)
    nkb = (K + 63) // 64
    per = -(-nkb // min(3, nkb))
    assert plan.info()["splits"] == -(-nkb // per)  # equal k-block ranges
    plan.run()
    torch.cuda.synchronize()
    _check(flat[:limit], ref + (a.float() @ b.float().t()).reshape(-1)[:limit], K)
    assert torch.all(flat[limit:] == 12345.0)


@pytest.mark.parametrize("M,N,K", [(4096, 825, 1024), (200, 72, 128)])
def test_gemm_bf16_out(M, N, K):
    from paper_2302_12445_b200.gemm import GemmPlan

    torch.manual_seed(2)
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    ldd = (N + 7) // 8 * 8
    d = torch.zeros(M, ldd, device="cuda", dtype=torch.bfloat16)
    plan = GemmPlan(a, b, d, M, N, K, ldd=ldd)
    plan.run()
    torch.cuda.synchronize()
    ref = a.float() @ b.float().t()
    # bf16 output: one bf16 rounding (2^-8 relative) on top of the fp32 tolerance
    err = (d[:, :N].float() - ref).abs()
    assert torch.all(err <= ref.abs() * 2.0**-8 + 2e-3 * ref.abs().max()), err.max()


@pytest.mark.parametrize("early", [False, True])
@pytest.mark.parametrize("M,N,K", [(8192, 1024, 512), (10240, 311, 512), (2048, 825, 1024)])
def test_gemm_persistent_many_tiles(M, N, K, tile_mode, early):
    """More tiles than SMs: exercises the persistent loop and both TMEM
    accumulators (epilogue of tile i overlapping the mainloop of tile i+1)."""
    from paper_2302_12445_b200.gemm import GemmPlan

    torch.manual_seed(3)
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    d = torch.full((M, N), float("nan"), device="cuda")
    plan = GemmPlan(a, b, d, M, N, K, ldd=N, early_operands=early)
    info = plan.info()
    assert info["m_tiles"] * info["n_tiles"] > 0
    if tile_mode == "pair":
        assert info["pair"] == 1 and info["cm"] == 2
    if tile_mode in ("single", "cluster"):
        assert info["pair"] == 0
    for _ in range(3):  # repeated launches (programmatic dependent launch chain)
        plan.run()
    torch.cuda.synchronize()
    _check(d, a.float() @ b.float().t(), K)
    if early:
        # D written by a chained GEMM while the next one streams its operands:
        # the later launch's stores must land after the earlier one's.
        d2 = torch.full((M, N), float("nan"), device="cuda")
        p2 = GemmPlan(a, b, d2, M, N, K, ldd=N, early_operands=True)
        b2 = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        p3 = GemmPlan(a, b2, d2, M, N, K, ldd=N, early_operands=True)
        for _ in range(4):
            p2.run()
            p3.run()
        torch.cuda.synchronize()
        _check(d2, a.float() @ b2.float().t(), K)


def test_gemm_group_wgrad_dgrad():
    """One launch computing a layer's weight gradient (split-K, fp32 reduce
    into a flat buffer) and data gradient (MN-major weights, bf16 out)."""
    from paper_2302_12445_b200.gemm import GemmPlan

    torch.manual_seed(4)
    T, H, R, n = 10240, 512, 311, 159006
    dy = torch.randn(T, 320, device="cuda").to(torch.bfloat16)
    dyt = dy.t().contiguous()
    x = torch.randn(T, H, device="cuda").to(torch.bfloat16)
    xt = x.t().contiguous()
    W = torch.zeros(R * H, device="cuda", dtype=torch.bfloat16)
    W[:n] = torch.randn(n, device="cuda").to(torch.bfloat16)
    G = torch.zeros(n + 64, device="cuda")
    G[n:] = 7.0
    dx = torch.zeros(T, H, device="cuda", dtype=torch.bfloat16)
    wg = GemmPlan(dyt, xt, G, R, H, T, lda=T, ldb=T, ldd=H, d_limit=n, accumulate=True)
    dg = GemmPlan(dy, W, dx, T, H, R, b_mn_major=True, lda=320, ldb=H, ldd=H)
    GemmPlan.run_group([wg, dg])
    torch.cuda.synchronize()
    ref_g = (dyt[:R].float() @ xt.float().t()).reshape(-1)[:n]
    _check(G[:n], ref_g, T)
    assert torch.all(G[n:] == 7.0)
    ref_dx = dy[:, :R].float() @ W.view(R, H).float()
    err = (dx.float() - ref_dx).abs()
    assert torch.all(err <= ref_dx.abs() * 2.0**-8 + 4e-3 * ref_dx.abs().max()), err.max()

