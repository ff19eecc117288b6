"""NVLS backend checks that need only one GPU. A multicast team needs at
least two GPUs (cuMulticastCreate rejects numDevices = 1), so the data-path
parity of the NVLS kernels runs in tests/dist_worker.py ("nvls",
"distoptim_nvls") under test_multigpu.py; here: the single-rank request
fails loudly instead of silently falling back to another transport."""
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_single_rank_heap_is_rejected():
    import paper_2302_12445_b200 as dear

    with pytest.raises(dear.InvalidArgument, match="at least 2 GPUs"):
        dear.SymmetricHeap(1 << 20)


def test_nvls_backend_needs_a_heap():
    import paper_2302_12445_b200 as dear

    with pytest.raises(ValueError):
        dear.Runtime(None, 0, 1, backend="nvls")
    with pytest.raises(dear.InvalidArgument):
        model = torch.nn.Linear(8, 8).cuda()
        dear.DistOptim(torch.optim.SGD(model.parameters(), lr=0.1), model, backend="nvls")
