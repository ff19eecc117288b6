"""GPU parity of the full DeAR pipeline (pack -> RS -> update -> AG -> unpack)
against the oracle, on one device. P > 1 runs as a local group (P ranks in one
process, ring-order collective kernels), which makes the result bit-exact
with the fp32 restatement of the reference's ring order — and within the
north star's 1e-5 of the fp64 restatement of collective.cpp."""
import numpy as np
import pytest

from dear_harness import oracle_run, run_local

pytestmark = pytest.mark.gpu

# Ragged tensors: odd sizes put layer and chunk boundaries at every
# alignment; 0-size and 1-size tensors are legal (model.cpp:57).
RAGGED = [1000, 4097, 3, 0, 2049, 1, 70001, 513, 12345, 7]


def _close(a, b, tol):
    return np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.abs(b)))


@pytest.mark.parametrize("P", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("policy,buf", [("DEAR_FUSED", 40_000), ("DEAR", 0),
                                        ("WFBP_FUSED", 100_000), ("WFBP", 0)])
def test_local_group_matches_oracle(restated, P, policy, buf):
    steps, lr = 3, 0.05
    got, _, _, same = run_local(RAGGED, P, steps, policy, buf, lr)
    exp32 = oracle_run(restated, RAGGED, P, steps, policy, buf, lr, f32=True)
    exp64 = oracle_run(restated, RAGGED, P, steps, policy, buf, lr, f32=False)
    for r in range(P):
        assert np.array_equal(got[r], got[0]), "replicas must stay bit-identical"
        assert np.array_equal(got[r], exp32), "fp32 ring-order restatement is bit-exact"
        assert _close(got[r].astype(np.float64), exp64, 1e-5)
    assert all(same)


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_momentum_weight_decay_nesterov(restated, P):
    kw = dict(momentum=0.9, dampening=0.0, weight_decay=1e-3, nesterov=True)
    got, _, _, _ = run_local(RAGGED, P, 4, "DEAR_FUSED", 60_000, 0.02, **kw)
    exp32 = oracle_run(restated, RAGGED, P, 4, "DEAR_FUSED", 60_000, 0.02, f32=True, **kw)
    exp64 = oracle_run(restated, RAGGED, P, 4, "DEAR_FUSED", 60_000, 0.02, f32=False, **kw)
    assert np.array_equal(got[0], exp32)
    assert _close(got[0].astype(np.float64), exp64, 1e-5)


def test_dampening_momentum(restated):
    kw = dict(momentum=0.8, dampening=0.3, weight_decay=0.0, nesterov=False)
    got, _, _, _ = run_local(RAGGED, 2, 3, "DEAR", 0, 0.05, **kw)
    exp32 = oracle_run(restated, RAGGED, 2, 3, "DEAR", 0, 0.05, f32=True, **kw)
    assert np.array_equal(got[0], exp32)


def test_shadow_copy_is_bf16_of_params(restated):
    got, sh, _, _ = run_local(RAGGED, 2, 2, "DEAR_FUSED", 40_000, 0.05, shadow=True)
    import torch

    exp = torch.from_numpy(got[0]).to(torch.bfloat16).float().numpy()
    assert np.array_equal(sh[0], exp)


def test_deferred_allgather_same_result(restated):
    a, _, ta, _ = run_local(RAGGED, 4, 3, "DEAR_FUSED", 40_000, 0.05, defer_allgather=False)
    b, _, tb, _ = run_local(RAGGED, 4, 3, "DEAR_FUSED", 40_000, 0.05, defer_allgather=True)
    assert np.array_equal(a, b)


def test_trace_is_reference_dispatch_order():
    """The collectives a rank enqueues follow the reference simulator's Comm
    dispatch order (task_graph.cpp:181-210 + simulate.cpp:100-134)."""
    from oracle.schedule import build_graph, comm_dispatch_order, simulate

    numels = RAGGED
    for policy, buf in (("DEAR_FUSED", 40_000), ("DEAR", 0), ("WFBP_FUSED", 100_000),
                        ("WFBP", 0)):
        _, _, traces, _ = run_local(numels, 2, 2, policy, buf, 0.05)
        tasks, _ = build_graph([4 * n for n in numels], [1.0] * len(numels),
                               [2.0] * len(numels), policy, buf, P=2, alpha=1e-3, beta=0.0)
        span, _ = simulate(tasks)
        want = comm_dispatch_order(tasks, span)
        assert traces[-1][0] == want, policy
        assert traces[-1][1] == want


def _gd_order(numels, buf, P, t_bp, rs, ag):
    """Dispatch order of the reference scheduler with dear_group_dependency."""
    from paper_2302_12445_b200 import costmodel as cm

    L = len(numels)
    G = cm.predict_iteration([4 * n for n in numels], [1.0] * L, [1.0] * L, "DEAR_FUSED", buf,
                             P, 0.0, 0.0)["buckets"]
    return cm.predict_iteration([4 * n for n in numels], [t_bp / 2] * L, [t_bp] * L,
                                "DEAR_FUSED", buf, P, 0.0, 0.0, group_dependency=True,
                                rs_times=[rs] * G, ag_times=[ag] * G)["comm_order"]


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("defer", [False, True])
@pytest.mark.parametrize("regime", ["backfill", "all_in_backprop", "all_at_step"])
def test_group_dependency_comm_order(restated, P, defer, regime):
    """dear_group_dependency with a dispatch order from the reference
    scheduler: same parameters as the barrier schedule (bit-exact with the
    fp32 ring restatement), and the rank's comm-stream trace IS that order."""
    buf, steps, lr = 40_000, 3, 0.05
    rs, ag = {"backfill": (1.5, 1.0), "all_in_backprop": (0.01, 0.01),
              "all_at_step": (100.0, 100.0)}[regime]
    order = _gd_order(RAGGED, buf, P, 1.0, rs, ag)
    got, _, traces, same = run_local(RAGGED, P, steps, "DEAR_FUSED", buf, lr,
                                     defer_allgather=defer, comm_order=order)
    exp32 = oracle_run(restated, RAGGED, P, steps, "DEAR_FUSED", buf, lr, f32=True)
    for r in range(P):
        assert np.array_equal(got[r], exp32)
    assert all(same)
    want = [("RS g%d" % v) if v > 0 else ("AG g%d" % -v) for v in order]
    if defer:
        # the AGs after the last RS are deferred into the next forward (not yet
        # enqueued when the trace is read right after dear_step)
        last_rs = max(i for i, v in enumerate(order) if v > 0)
        want = want[:last_rs + 1]
    assert traces[-1][0] == want
    if regime == "backfill":
        last_rs = max(i for i, v in enumerate(order) if v > 0)
        assert any(v < 0 for v in order[:last_rs]) and any(v < 0 for v in order[last_rs:])


def test_comm_order_validation():
    import torch

    from paper_2302_12445_b200 import InvalidArgument, LocalGroup, Runtime

    g = LocalGroup(1)
    p = torch.zeros(3000, device="cuda")
    gr = torch.zeros(3000, device="cuda")
    rt = Runtime(g, 0, 1, policy="DEAR_FUSED", fusion_buffer_bytes=4000, lr=0.1,
                 dear_group_dependency=True)
    for l in range(3):
        rt.register(l + 1, p[1000 * l:1000 * (l + 1)], gr[1000 * l:1000 * (l + 1)])
    rt.finalize()
    G = len(rt.buckets())
    assert G == 3
    for bad in ([1, -1, 2, -2, 3], [1, 2, -3, 3, -1, -2], [2, 1, 3, -1, -2, -3],
                [1, -1, 2, -1, 3, -3], [1, -1, 2, -2, 3, 4]):
        with pytest.raises(InvalidArgument):
            rt.set_comm_order(bad)
    rt.set_comm_order([1, -1, 2, 3, -3, -2])
    rt.set_comm_order([])
    rt.close()
    rt2 = Runtime(g, 0, 1, policy="DEAR_FUSED", fusion_buffer_bytes=4000, lr=0.1)
    for l in range(3):
        rt2.register(l + 1, p[1000 * l:1000 * (l + 1)], gr[1000 * l:1000 * (l + 1)])
    rt2.finalize()
    with pytest.raises(InvalidArgument):  # needs dear_group_dependency
        rt2.set_comm_order([1, -1, 2, -2, 3, -3])
    rt2.close()
    g.close()


@pytest.mark.parametrize("policy,buf", [("DEAR_FUSED", 40_000), ("WFBP", 0)])
def test_direct_update_p1_matches_pipeline(restated, monkeypatch, policy, buf):
    """P = 1 without momentum runs one fused update straight from the
    gradients (14 B/elem); it must equal the pack/update/unpack pipeline
    (DEAR_DIRECT=0) bit for bit, parameters and bf16 copies, and the oracle."""
    kw = dict(weight_decay=1e-3)
    got, sh, _, _ = run_local(RAGGED, 1, 3, policy, buf, 0.05, shadow=True, **kw)
    monkeypatch.setenv("DEAR_DIRECT", "0")
    ref, sh_ref, _, _ = run_local(RAGGED, 1, 3, policy, buf, 0.05, shadow=True, **kw)
    assert np.array_equal(got, ref)
    assert np.array_equal(sh, sh_ref)
    exp32 = oracle_run(restated, RAGGED, 1, 3, policy, buf, 0.05, f32=True, **kw)
    assert np.array_equal(got[0], exp32)


def _pp_order(numels, P, pb):
    """The reference scheduler's PRIORITY_PARTITION dispatch sequence
    (task_graph.cpp:215-258 + simulate.cpp:65-159) on nominal times."""
    from paper_2302_12445_b200 import costmodel as cm

    L = len(numels)
    return cm.predict_iteration([4 * n for n in numels], [1.0] * L, [2.0] * L,
                                "PRIORITY_PARTITION", 0, P, 1e-3, 1e-9,
                                partition_bytes=pb)["comm_order"]


@pytest.mark.parametrize("P,transport", [(1, "ring"), (2, "ring"), (3, "ring"), (2, "peer"),
                                         (4, "peer")])
@pytest.mark.parametrize("ordered", [False, True])
def test_priority_partition(restated, P, transport, ordered):
    """PRIORITY_PARTITION: every layer's all-reduce in ceil(bytes / 40 KB)
    parts, each its own bucket. Parameters bit-exact with the fp32 ring
    restatement over the same parts; with the reference scheduler's dispatch
    sequence the rank's comm trace is exactly that sequence ("AR l<l> p<k>")."""
    from paper_2302_12445_b200 import costmodel as cm

    pb = 40_000
    order = _pp_order(RAGGED, P, pb) if ordered else None
    got, _, traces, same = run_local(RAGGED, P, 3, "PRIORITY_PARTITION", 0, 0.05,
                                     transport=transport, flat=transport == "peer",
                                     comm_order=order, partition_bytes=pb, shadow=True)
    exp32 = oracle_run(restated, RAGGED, P, 3, "PRIORITY_PARTITION", 0, 0.05, f32=True,
                       partition_bytes=pb)
    assert all(same)
    for r in range(P):
        assert np.array_equal(got[r], exp32)
    parts = [(l, k + 1) for l, n in cm.partition_plan([4 * n for n in RAGGED], pb)
             for k in range(n)]
    seq = order if ordered else list(range(1, len(parts) + 1))
    assert traces[-1][0] == ["AR l%d p%d" % parts[g - 1] for g in seq]
    assert len(parts) > len(RAGGED)  # some layers really are split
