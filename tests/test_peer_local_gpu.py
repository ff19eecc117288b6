"""The multi-GPU NVLink peer data path, on ONE device (LocalGroup(P,
transport="peer")): P contexts in this process run the same fused kernel code
as one process per GPU — the zero-copy reduce-scatter + update and all-gather
bodies, or the slot path's pack_kernel<true> + reduce-scatter + all-gather —
with in-process deltas instead of IPC mappings and the same in-kernel
cross-rank counters, each collective one cooperative launch over all ranks. Their sums follow the reference's ring
order (collective.cpp:70-90), so parameters must be BIT-EXACT with the fp32
ring restatement and within 1e-5 of the fp64 sgd_step (collective.cpp:166-194).
"""
import numpy as np
import pytest

from dear_harness import oracle_run, run_local

pytestmark = pytest.mark.gpu

RAGGED = [1000, 4097, 3, 0, 2049, 1, 70001, 513, 12345, 7, 262144, 100003]
POLICIES = [("DEAR_FUSED", 100_000), ("DEAR", 0), ("WFBP_FUSED", 400_000), ("WFBP", 0),
            ("DEAR_FUSED", 25_000_000)]


def _close(a, b, tol=1e-5):
    return np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.abs(b)))


# P = 8 runs the compile-time 8-rank kernel instances (the 8-GPU bench path).
@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("zero_copy", [True, False])
@pytest.mark.parametrize("policy,buf", POLICIES)
def test_peer_kernels_bit_exact(restated, P, zero_copy, policy, buf):
    got, _, _, same = run_local(RAGGED, P, 3, policy, buf, 0.05, transport="peer", flat=True,
                                zero_copy=zero_copy)
    assert run_local.zero_copy == [zero_copy] * P, "expected transport was not taken"
    exp32 = oracle_run(restated, RAGGED, P, 3, policy, buf, 0.05, f32=True)
    exp64 = oracle_run(restated, RAGGED, P, 3, policy, buf, 0.05, f32=False)
    assert all(same)
    for r in range(P):
        assert np.array_equal(got[r], exp32), f"rank {r}: not bit-exact with the ring order"
        assert _close(got[r].astype(np.float64), exp64)


def test_peer_slot_path_with_separate_tensors(restated):
    """Per-layer tensors (no common layout): the connect falls back to the
    slot path by itself."""
    got, _, _, same = run_local(RAGGED, 2, 3, "DEAR_FUSED", 100_000, 0.05, transport="peer")
    assert run_local.zero_copy == [False, False]
    exp32 = oracle_run(restated, RAGGED, 2, 3, "DEAR_FUSED", 100_000, 0.05, f32=True)
    assert all(same) and np.array_equal(got[0], exp32)


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("zero_copy", [True, False])
def test_peer_momentum_wd_nesterov_shadow(restated, P, zero_copy):
    kw = dict(momentum=0.9, dampening=0.0, weight_decay=1e-3, nesterov=True)
    got, sh, _, same = run_local(RAGGED, P, 4, "DEAR_FUSED", 200_000, 0.02, transport="peer",
                                 flat=True, zero_copy=zero_copy, shadow=True, **kw)
    exp32 = oracle_run(restated, RAGGED, P, 4, "DEAR_FUSED", 200_000, 0.02, f32=True, **kw)
    assert all(same)
    assert np.array_equal(got[0], exp32)
    import torch

    assert np.array_equal(sh[0], torch.from_numpy(got[0]).to(torch.bfloat16).float().numpy())


@pytest.mark.parametrize("defer", [False, True])
def test_peer_group_dependency_and_deferred(restated, defer):
    from paper_2302_12445_b200 import costmodel as cm

    L, P, buf = len(RAGGED), 2, 100_000
    G = cm.predict_iteration([4 * n for n in RAGGED], [1.0] * L, [1.0] * L, "DEAR_FUSED", buf,
                             P, 0.0, 0.0)["buckets"]
    order = cm.predict_iteration([4 * n for n in RAGGED], [0.5] * L, [1.0] * L, "DEAR_FUSED",
                                 buf, P, 0.0, 0.0, group_dependency=True, rs_times=[1.5] * G,
                                 ag_times=[1.0] * G)["comm_order"]
    got, _, traces, same = run_local(RAGGED, P, 3, "DEAR_FUSED", buf, 0.05, transport="peer",
                                     flat=True, comm_order=order, defer_allgather=defer)
    exp32 = oracle_run(restated, RAGGED, P, 3, "DEAR_FUSED", buf, 0.05, f32=True)
    assert all(same) and np.array_equal(got[0], exp32)
    want = [("RS g%d" % v) if v > 0 else ("AG g%d" % -v) for v in order]
    if defer:
        want = want[:max(i for i, v in enumerate(order) if v > 0) + 1]
    assert traces[-1][0] == want


def test_peer_lr_schedule(restated):
    """dear_set_lr is stream-ordered (a one-thread kernel, no host sync): each
    step's rate applies to exactly that step's updates."""
    sched = [0.1, 0.05, 0.0, 0.2]
    got, _, _, _ = run_local(RAGGED, 2, 4, "DEAR_FUSED", 100_000, 0.3, transport="peer",
                             flat=True, lr_schedule=sched)
    exp32 = oracle_run(restated, RAGGED, 2, 4, "DEAR_FUSED", 100_000, 0.3, f32=True,
                       lr_schedule=sched)
    assert np.array_equal(got[0], exp32)
