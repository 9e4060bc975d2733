"""Multi-GPU tile-band sharding of the fit.

One process per GPU.  The image's ceil(H/16) block rows are split into
contiguous bands, one per rank; every rank holds all K kernels (replicated)
and the full target, runs a1-a7 on its band only (``smoe_set_band`` +
``smoe_grad``), the per-rank gradients and loss partials are summed with one
NCCL all-reduce each, and every rank applies the identical Adam update
(``smoe_apply``), so parameters stay bit-identical across ranks.

The gradient sum is the method's only exchange: per-band gradients of the
1/(H W C)-normalised loss add up to the full-image gradient (pinned in
tests/test_oracle.py::test_band_additivity).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def band_rows(ny: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block-row band of ``rank``: the first ny % world ranks get
    one extra row (e.g. 270 rows on 8 ranks -> 34,34,34,34,34,34,33,33)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(ny, world)
    r0 = rank * base + min(rank, extra)
    r1 = r0 + base + (1 if rank < extra else 0)
    return r0, r1


def allreduce_grads(grad: torch.Tensor, sums: torch.Tensor | None, group=None) -> None:
    """Sum per-band gradients [K, Pk] (fp32) and, if given, loss partials [3]
    (fp64) over the ranks, in place."""
    dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    if sums is not None:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)


class BandedFit:
    """Data-parallel fit of one image across the ranks of ``group``."""

    def __init__(self, handle, rank: int, world: int, group=None):
        from . import smoe
        self.h = handle
        self.rank, self.world, self.group = rank, world, group
        ny = (handle.H + 15) // 16
        self.band = band_rows(ny, rank, world)
        if self.band[1] > self.band[0]:
            handle.set_band(*self.band)
        dev = f"cuda:{handle.device}"
        self.grad = torch.zeros((handle.K, handle.Pk), dtype=torch.float32, device=dev)
        self.sums = torch.zeros(3, dtype=torch.float64, device=dev)
        self._smoe = smoe

    def step(self, params, target, lr, stats: bool = True):
        """One fit iteration; returns the all-reduced loss partials (SSE,
        clamped SSE, uncovered pixels), or None with stats=False (the loss
        partials then stay per band: one collective per step, the gradient's)."""
        if self.band[1] > self.band[0]:
            self.h.grad(params, target, self.grad, self.sums)
        else:  # more ranks than block rows: this rank contributes nothing
            self.grad.zero_()
            self.sums.zero_()
        allreduce_grads(self.grad, self.sums if stats else None, self.group)
        self.h.apply(params, self.grad, lr)
        return self.sums if stats else None
