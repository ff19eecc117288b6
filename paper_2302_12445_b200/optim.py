"""DistOptim — the user-facing DeAR wrapper.

    import paper_2302_12445_b200 as dear
    comm = dear.init()                                   # NCCL over torch.distributed
    opt = torch.optim.SGD(model.parameters(), lr=0.05, momentum=0.9)
    opt = dear.DistOptim(opt, model, comm=comm, policy="DEAR_FUSED",
                         fusion_buffer_bytes=25_000_000)
    for x, y in loader:
        loss = loss_fn(model(x), y)
        loss.backward()
        opt.step()
        opt.zero_grad()
    opt.synchronize()                                    # before eval / checkpoint

Every learnable tensor is one reference "layer" (LayerSpec is one learnable
tensor, model.hpp:24-34), numbered 1..L in ``model.parameters()`` order
(input side first). A post-accumulate-grad hook per tensor reports gradient
readiness (BackPipe), a forward pre-hook per module waits for that module's
buckets (FeedPipe). The wrapped optimizer supplies the hyper-parameters; the
update itself runs shard-locally on the GPU between reduce-scatter and
all-gather, so the wrapped optimizer's own ``step`` is never called.
The learning rate is read from ``param_groups[0]["lr"]`` when the first
gradient of an iteration is reported (the updates run during backward), so an
LR scheduler stepped between iterations takes effect on the next iteration's
update, exactly as with ``torch.optim.SGD``.

One-GPU multi-rank runs: pass ``comm=LocalGroup(P, transport="peer")`` and a
distinct ``rank`` (and compute ``stream``) per replica, then call
``group.connect()`` once every replica's DistOptim exists.

Only ``torch.optim.SGD`` is supported — the reference's update is SGD
(collective.cpp:166-194); momentum / weight decay / nesterov are an unpinned
extension following torch semantics.
"""
from __future__ import annotations

from typing import Optional

import torch

from .runtime import Communicator, LocalGroup, Runtime, SymmetricHeap


class DistOptim:
    def __init__(self, optimizer: torch.optim.Optimizer, model: Optional[torch.nn.Module] = None,
                 *, comm=None, rank: int = 0, policy: str = "DEAR_FUSED",
                 fusion_buffer_bytes: int = 25_000_000, defer_allgather: bool = False,
                 backend: str = "auto", stream: Optional[torch.cuda.Stream] = None,
                 flatten: bool = True, partition_bytes: int = 0):
        if not isinstance(optimizer, torch.optim.SGD):
            raise TypeError("DistOptim supports torch.optim.SGD (the reference's update rule)")
        if len(optimizer.param_groups) != 1:
            raise ValueError("DistOptim supports a single parameter group")
        g = optimizer.param_groups[0]
        if backend == "nvls" and not flatten:
            raise ValueError("the nvls backend needs flatten=True (the flat buffers live in the "
                             "symmetric heap)")
        if g.get("maximize", False):
            raise ValueError("maximize=True is not supported")
        if model is None and defer_allgather:
            raise ValueError("defer_allgather needs the model: its forward pre-hooks flush "
                             "the deferred all-gathers")
        self.optimizer = optimizer
        self.model = model
        self._stream = stream
        params = list(model.parameters()) if model is not None else list(g["params"])
        opt_ids = {id(p) for p in g["params"]}
        params = [p for p in params if p.requires_grad and id(p) in opt_ids]
        if not params:
            raise ValueError("build_fusion_plan: empty model")
        self.params = params
        self._lr = float(g["lr"])
        self._in_backward = False
        self._heap = None
        if backend == "nvls":
            # The flat parameter / gradient buffers live in a symmetric heap
            # mapped through one NVLS multicast object (collective).
            n = sum((p.numel() + 63) // 64 * 64 for p in params if p.requires_grad)
            self._heap = SymmetricHeap(2 * 4 * max(n, 64) + (1 << 16))
        if isinstance(comm, LocalGroup):
            world, rank_ = comm.P, rank
        elif isinstance(comm, Communicator):
            world, rank_ = comm.world_size, comm.rank
        else:
            world, rank_ = 1, 0
        self.runtime = Runtime(comm, rank_, world, policy=policy, heap=self._heap,
                               fusion_buffer_bytes=fusion_buffer_bytes, lr=self._lr,
                               momentum=float(g.get("momentum", 0.0)),
                               dampening=float(g.get("dampening", 0.0)),
                               weight_decay=float(g.get("weight_decay", 0.0)),
                               nesterov=bool(g.get("nesterov", False)),
                               defer_allgather=defer_allgather, backend=backend,
                               stream=stream, partition_bytes=partition_bytes)
        for p in params:
            if p.dtype != torch.float32 or not p.is_cuda or not p.is_contiguous():
                raise ValueError("DistOptim needs contiguous fp32 CUDA parameters")
        if flatten:
            # One flat parameter buffer and one flat gradient buffer (64-element
            # aligned views, layer order): the NVLink peer backend then maps
            # them directly (zero-copy: no pack, no bucket buffer).
            offs, n = [], 0
            for p in params:
                offs.append(n)
                n += (p.numel() + 63) // 64 * 64
            if self._heap is not None:
                pflat = self._heap.tensor(max(n, 64)).zero_()
                gflat = self._heap.tensor(max(n, 64)).zero_()
            else:
                pflat = torch.zeros(max(n, 64), dtype=torch.float32, device=params[0].device)
                gflat = torch.zeros_like(pflat)
            for p, o in zip(params, offs):
                view = pflat[o:o + p.numel()].view_as(p)
                view.copy_(p.data)
                p.data = view
                g = gflat[o:o + p.numel()].view_as(p)
                if p.grad is not None:
                    g.copy_(p.grad)
                p.grad = g
            self._flat = (pflat, gflat)
        self._layer_of = {}
        self._grad_ptr = {}
        for layer, p in enumerate(params, start=1):
            # Gradients live in fixed storage the runtime packs from; zero_grad
            # zeroes in place instead of dropping it.
            if p.grad is None:
                p.grad = torch.zeros_like(p)
            self.runtime.register(layer, p.data, p.grad)
            self._grad_ptr[layer] = p.grad.data_ptr()
            self._layer_of[id(p)] = layer
        self.runtime.finalize()
        self._hooks = []
        for p in params:
            self._hooks.append(p.register_post_accumulate_grad_hook(self._make_grad_hook(p)))
        if model is not None:
            for m in model.modules():
                layers = [self._layer_of[id(p)] for p in m.parameters(recurse=False)
                          if id(p) in self._layer_of]
                if layers:
                    self._hooks.append(m.register_forward_pre_hook(self._make_ff_hook(layers)))

    def _make_grad_hook(self, p):
        layer = self._layer_of[id(p)]

        def hook(param):
            if param.grad is None or param.grad.data_ptr() != self._grad_ptr[layer]:
                raise RuntimeError(f"gradient storage of layer {layer} changed; use "
                                   "DistOptim.zero_grad() (in-place) instead of set_to_none")
            if not self._in_backward:
                # First gradient of the iteration: this iteration's updates are
                # enqueued from now on, so the current LR must be on the device.
                self._in_backward = True
                self._sync_lr()
            self.runtime.grad_ready(layer)
        return hook

    def _make_ff_hook(self, layers):
        def hook(module, args):
            for layer in layers:
                self.runtime.param_wait(layer)
        return hook

    def _sync_lr(self):
        lr = float(self.optimizer.param_groups[0]["lr"])
        if lr != self._lr:
            self.runtime.set_lr(lr)  # stream-ordered on the comm stream, no host sync
            self._lr = lr

    def step(self, closure=None):
        if closure is not None:
            raise ValueError("closures are not supported")
        self._in_backward = False
        self.runtime.step(self._stream)
        # The wrapped optimizer's update ran on the GPU: tell LR schedulers so.
        self.optimizer._opt_called = True
        if self.model is None:
            # No forward pre-hooks gate the parameters: make the caller's
            # stream wait for the all-gathers that rewrite them.
            self.runtime.join(self._stream)

    def zero_grad(self, set_to_none: bool = False):
        for p in self.params:
            p.grad.zero_()

    def synchronize(self):
        self.runtime.synchronize()

    def check_replicas(self) -> bool:
        return self.runtime.check_replicas()

    @property
    def param_groups(self):
        return self.optimizer.param_groups

    def close(self):
        for h in self._hooks:
            h.remove()
        self._hooks = []
        self.runtime.close()
        if self._heap is not None:
            # the parameters live in the heap: give them private storage first
            for p in self.params:
                p.data = p.data.clone()
                p.grad = p.grad.clone()
            self._flat = None
            self._heap.close()
            self._heap = None


def init(group=None) -> Communicator | None:
    """Create the NCCL communicator for the current torch.distributed job
    (None when not distributed / single rank)."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    return Communicator.from_torch_distributed(group)
