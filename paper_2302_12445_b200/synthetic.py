"""Synthetic per-layer compute for the DeAR benchmarks (BASELINE configs 2-4).

The reference models a layer only by its parameter count and compute
durations (LayerSpec, model.hpp:26-34); BASELINE.json asks for "synthetic
layer compute" that the collectives overlap with. Here every learnable tensor
of a preset (proj/src/model.cpp:111-168 sizes, layer 1 = input side) is a
linear map on `tokens` rows of width `hidden`:

    its n_l fp32 parameters, viewed row-major as W_l[R_l, hidden] with
    R_l = ceil(n_l / hidden) (the last row partial, zero-padded in the bf16
    compute copy), so
    FF_l     Y_l  = X  W_l^T          [T, R_l]    2 T R_l H flops
    BP_l     dX   = dY W_l            [T, H]      2 T R_l H flops  (dgrad)
             G_l += dY^T X            [R_l, H]    2 T R_l H flops  (wgrad, fp32,
                                                  written into the flat grad)
All three are the hand-written tcgen05 GEMM (gemm.py). Per layer FF costs
2 n_l T flops and BP twice that, i.e. the 6 * params * tokens of a dense
network and the paper's t_bp = 2 t_ff (§VI-H).

What is synthetic: the input X and the upstream gradient dY are fixed seeded
tensors shared by all layers (layers are not chained numerically), so there
is no loss function. Parameters and gradients are real: W_l is the bf16 copy
of the parameters that DeAR's unpack kernel refreshes after every update, and
G_l is the true weight gradient of Y_l = X W_l^T for upstream dY.
"""
from __future__ import annotations

import math
import os

import torch

from .gemm import GemmPlan


def _round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


class SyntheticModel:
    def __init__(self, numels: list[int], hidden: int, tokens: int, device="cuda", seed: int = 0,
                 tune: bool = True, wgrad_split: int = 0, symmetric: bool = False):
        self.numels = [int(n) for n in numels]
        self.L = len(self.numels)
        self.H = int(hidden)
        self.T = int(tokens)
        if self.H % 64 or self.T % 64:
            raise ValueError("hidden and tokens must be multiples of 64")
        dev = torch.device(device)
        H, T = self.H, self.T
        self.rows = [max(1, math.ceil(n / H)) for n in self.numels]
        # Flat fp32 parameter / gradient storage, each layer 256-byte aligned.
        self.offsets, off = [], 0
        for n in self.numels:
            self.offsets.append(off)
            off += _round_up(max(n, 1), 64)
        self.flat_elems = off
        g = torch.Generator(device="cpu").manual_seed(seed)
        rows = [max(1, math.ceil(n / H)) for n in self.numels]
        # symmetric=True: parameters, gradients and bf16 copies in an NVLS
        # symmetric heap (collective over torch.distributed), for the nvls backend.
        self.heap = None
        if symmetric:
            from .runtime import SymmetricHeap

            self.heap = SymmetricHeap(8 * off + 2 * sum(r * H for r in rows) + (1 << 20))
            self.params_flat = self.heap.tensor(off)
            self.params_flat.copy_((torch.rand(off, generator=g) * 2 - 1).mul_(0.02))
            self.grads_flat = self.heap.tensor(off).zero_()
        else:
            self.params_flat = (torch.rand(off, generator=g) * 2 - 1).mul_(0.02).to(dev)
            self.grads_flat = torch.zeros(off, device=dev)
        self.params = [self.params_flat[o:o + n] for o, n in zip(self.offsets, self.numels)]
        self.grads = [self.grads_flat[o:o + n] for o, n in zip(self.offsets, self.numels)]
        # bf16 compute copies, full rows (zero pad past n_l).
        self.w_offsets, woff = [], 0
        for r in self.rows:
            self.w_offsets.append(woff)
            woff += r * H
        self.shadow_flat = (self.heap.tensor(woff, torch.bfloat16).zero_() if self.heap is not None
                            else torch.zeros(woff, dtype=torch.bfloat16, device=dev))
        self.shadows = [self.shadow_flat[o:o + r * H] for o, r in zip(self.w_offsets, self.rows)]
        for p, s in zip(self.params, self.shadows):
            s[: p.numel()].copy_(p.to(torch.bfloat16))
        rmax = max(self.rows)
        self.rpad = _round_up(rmax, 64)
        # Activations / upstream gradient (synthetic, seeded).
        self.x = (torch.rand(T, H, generator=g) * 2 - 1).to(torch.bfloat16).to(dev)
        self.xt = self.x.t().contiguous()
        self.dy = (torch.rand(T, self.rpad, generator=g) * 2 - 1).mul_(1e-3).to(torch.bfloat16).to(dev)
        self.dyt = self.dy.t().contiguous()
        self.y = torch.empty(T, self.rpad, dtype=torch.bfloat16, device=dev)
        # FF output in the transposed orientation (Y^T = W X^T), when the tile
        # tuner finds it faster (narrow layers: one wave of wide tiles).
        self.yt = torch.empty(self.rpad, T, dtype=torch.bfloat16, device=dev)
        self.ff_transposed = False
        self.dx = torch.empty(T, H, dtype=torch.bfloat16, device=dev)
        self.wgrad_split = int(wgrad_split)
        self.bp_split = os.environ.get("DEAR_BP_SPLIT", "0") == "1"
        self._build_plans()
        self.tiles = self.tune_tiles() if tune else None

    def _build_plans(self):
        H, T = self.H, self.T
        self.ff, self.dgrad, self.wgrad, self.ff_t = [], [], [], []
        for l in range(self.L):
            R, n = self.rows[l], self.numels[l]
            W = self.shadows[l]
            # No layer GEMM reads what another one writes (X, dY and the
            # bf16 weights are read-only across the GEMM chain; W is refreshed
            # by unpack on the comm stream behind an event), so operands may
            # stream under the previous GEMM's tail.
            self.ff.append(GemmPlan(self.x, W, self.y, T, R, H, lda=H, ldb=H, ldd=self.rpad,
                                    early_operands=True))
            self.ff_t.append(GemmPlan(W, self.x, self.yt, R, T, H, lda=H, ldb=H, ldd=T,
                                      early_operands=True))
            self.dgrad.append(GemmPlan(self.dy, W, self.dx, T, H, R, b_mn_major=True,
                                       lda=self.rpad, ldb=H, ldd=H, early_operands=True))
            self.wgrad.append(GemmPlan(self.dyt, self.xt, self.grads[l] if n > 0 else self.grads_flat,
                                       R, H, T, lda=T, ldb=T, ldd=H, d_limit=n,
                                       accumulate=True, early_operands=True,
                                       split_k=self.wgrad_split))

    def tune_tiles(self, chain: int = 16) -> dict:
        """Plan-time tile autotuning (gemm.autotune): FF as a chain of FF
        launches; wgrad (scratch output) and dgrad as chains of their own to
        rank tiles, then backprop on the real chain of grouped launches over
        every layer (top-2 x top-2 tiles x split-K counts). Runs once, outside
        any timed region; the gradients are zeroed afterwards."""
        from .gemm import autotune, tile_candidates

        H, T = self.H, self.T
        k = min(self.L, 8)
        R = max(set(self.rows), key=self.rows.count)
        n = R * H
        s = torch.cuda.Stream()
        ff = autotune(self.ff[:k], tile_candidates(T, R, False), chain, s)
        fft = autotune(self.ff_t[:k], tile_candidates(R, T, False), chain, s)
        if fft[0][0] < ff[0][0]:
            # same flops, output stored transposed (y is synthetic scratch)
            self.ff, self.ff_t = self.ff_t, self.ff
            self.ff_transposed = True
            ff = fft
        dg = autotune(self.dgrad[:k], tile_candidates(T, H, True), chain, s)
        scratch = torch.zeros(n + 64, device=self.x.device)
        wgs = [GemmPlan(self.dyt, self.xt, scratch, R, H, T, lda=T, ldb=T, ldd=H, d_limit=n,
                        accumulate=True, early_operands=True, split_k=self.wgrad_split)]
        wg = autotune(wgs, tile_candidates(R, H, False), chain, s)
        best_ff = ff[0][1:]
        for l in range(self.L):
            self.ff[l].set_tile(*best_ff)
        wgs[0].close()
        # Backprop on the real chain: every layer's grouped wgrad+dgrad into
        # the real (freshly zeroed, mostly cold) gradients, as in a step. The
        # scratch chain above cannot see the split-K reductions' cost on cold
        # lines, so the weight-gradient tile, split count and reduction path,
        # then the dgrad tile, are chosen here.
        from .gemm import time_chain

        L = self.L
        split0 = self.wgrad[0].info()["splits"]
        num_kb = (T + 63) // 64
        splits = ([self.wgrad_split] if self.wgrad_split > 0 else
                  sorted({x for x in (split0, 4, 6, 8, 10, 12, 16) if 1 <= x <= num_kb}))

        def bp_real(i):
            if i == 0:
                self.zero_grad()
            l = L - 1 - (i % L)
            self._run_bp(l, s)

        def set_bp(wc, sp, red, dc):
            for l in range(L):
                self.wgrad[l].set_tile(*wc)
                self.wgrad[l].set_splits(sp)
                self.wgrad[l].set_red_add(red)
                self.dgrad[l].set_tile(*dc)

        # stage 1: weight-gradient tile x split-K x reduction path (TMA reduce
        # or red.add), dgrad at its best chain tile
        max_bn = int(os.environ.get("DEAR_GEMM_MAX_BN", "256"))  # see gemm.tile_candidates
        wtiles = list(dict.fromkeys([c[1:] for c in wg[:2]] +
                                    [t for t in ((128, 0), (176, 0), (256, 0), (128, 1),
                                                 (256, 1)) if t[0] <= max_bn and
                                     (t[1] == 0 or R > 128)]))
        trials = []
        for wc in wtiles:
            for sp in splits:
                for red in (False, True):
                    set_bp(wc, sp, red, dg[0][1:])
                    trials.append((time_chain(bp_real, L, s, reps=2), wc, sp, red, dg[0][1:]))
        trials.sort(key=lambda t: t[0])
        _, wc, sp, red, _ = trials[0]
        # stage 2: dgrad tile with that weight-gradient configuration
        for dc in [c[1:] for c in dg[1:3]]:
            set_bp(wc, sp, red, dc)
            trials.append((time_chain(bp_real, L, s, reps=2), wc, sp, red, dc))
        trials.sort(key=lambda t: t[0])
        us, best_wg, best_sp, best_red, best_dg = trials[0]
        # Multi-rank: every rank runs rank 0's choice. Per-rank tuning noise
        # would otherwise give the ranks different layer times, and the
        # reduce-scatter of every bucket waits for the slowest rank.
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            pick = [(best_ff, self.ff_transposed, best_wg, best_sp, best_red, best_dg, us,
                     ff[0][0])]
            dist.broadcast_object_list(pick, 0)
            best_ff, transposed, best_wg, best_sp, best_red, best_dg, us, ff_us = pick[0]
            if transposed != self.ff_transposed:
                self.ff, self.ff_t = self.ff_t, self.ff
                self.ff_transposed = transposed
            for l in range(self.L):
                self.ff[l].set_tile(*best_ff)
            ff = [(ff_us,) + tuple(best_ff)] + list(ff[1:])
        set_bp(best_wg, best_sp, best_red, best_dg)
        self.zero_grad()
        torch.cuda.synchronize()
        return {"ff": {"bn": best_ff[0], "pair": best_ff[1], "us": round(ff[0][0], 2),
                       "transposed": self.ff_transposed},
                "wgrad": {"bn": best_wg[0], "pair": best_wg[1], "splits": best_sp,
                          "reduce": "red.add" if best_red else "tma"},
                "dgrad": {"bn": best_dg[0], "pair": best_dg[1]},
                "bp_group_us": round(us, 2),
                "candidates": {"ff": len(ff), "wgrad": len(wg), "dgrad": len(dg),
                               "bp_real_chain": len(trials)}}

    def gemm_launches_per_step(self) -> int:
        bp = sum(2 if self.bp_split or w.info()["pair"] != d.info()["pair"] else 1
                 for w, d in zip(self.wgrad, self.dgrad))
        return self.L + bp

    # -- flops ---------------------------------------------------------------
    def ff_flops(self) -> int:
        return sum(2 * self.T * r * self.H for r in self.rows)

    def bp_flops(self) -> int:
        return 2 * self.ff_flops()

    # -- one iteration's compute, stream-ordered ----------------------------
    def set_input(self, x_host: torch.Tensor | None, stream=None) -> None:
        """Copy this step's input batch (pinned host -> device) and derive X^T."""
        if x_host is not None:
            self.x.copy_(x_host, non_blocking=True)
        self.xt.copy_(self.x.t())

    def forward_layer(self, l: int, stream=None) -> None:
        self.ff[l - 1].run(stream)

    def backward_layer(self, l: int, stream=None) -> None:
        # wgrad and dgrad are independent: one persistent launch computes both.
        self._run_bp(l - 1, stream)

    def _run_bp(self, i: int, stream) -> None:
        if self.bp_split:  # two chained launches (DEAR_BP_SPLIT=1, A/B experiments)
            self.wgrad[i].run(stream)
            self.dgrad[i].run(stream)
        else:
            GemmPlan.run_group([self.wgrad[i], self.dgrad[i]], stream)

    def zero_grad(self) -> None:
        self.grads_flat.zero_()

    def result_scalar(self) -> torch.Tensor:
        """A device scalar standing for the step's loss (read back by e2e)."""
        return self.yt[0, 0] if self.ff_transposed else self.y[0, 0]

    def close(self):
        for p in self.ff + self.ff_t + self.dgrad + self.wgrad:
            p.close()
        if self.heap is not None:
            self.params = self.grads = self.shadows = None
            self.params_flat = self.grads_flat = self.shadow_flat = None
            self.heap.close()
            self.heap = None
