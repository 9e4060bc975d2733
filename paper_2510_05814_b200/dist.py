"""Multi-GPU tile-band sharding of the fit.

One process per GPU.  The image's ceil(H/16) block rows are split into
contiguous bands, one per rank; every rank holds all K kernels and runs
a1-a7 on its band only (``smoe_set_band`` + ``smoe_grad``: the preprocess
writes records only for kernels whose box meets the band, and only the
band's blocks are binned and rasterised).  The per-band gradients of the
1/(H W C)-normalised loss add up to the full-image gradient (pinned in
tests/test_oracle.py::test_band_additivity), so the method's one exchange is
that sum, done as

  1. reduce-scatter of grad[Kpad][Pk] (fp32, NCCL over NVLink/NVSwitch): rank
     r receives the summed rows of its kernel shard [r Ks, (r+1) Ks),
     Ks = ceil(K / world);
  2. all-reduce of the band loss partials sums[4] = (SSE, clamped SSE,
     uncovered, skipped) (fp64, 32 bytes);
  3. Adam on the rank's shard only (``smoe_apply_ex(k0, k1, sums)``; skipped
     on every rank alike when any rank's binning overflowed, sums[3] > 0);
  4. all-gather of the four parameter arrays, padded to Kpad rows (packed
     into one collective), so every rank holds the identical updated
     parameters.

Bytes moved equal the all-reduce's (reduce-scatter + all-gather), the Adam
work per rank is 1/world of the replicated form, and the Adam moments of
other shards are never touched.
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


def shard_rows(K: int, rank: int, world: int) -> tuple[int, int, int]:
    """Kernel shard of ``rank`` for the reduce-scatter / all-gather: rows
    [k0, k1) of the K kernels (clipped), and Ks = ceil(K / world), the padded
    shard size (every rank's chunk of the padded [Kpad = world Ks] buffers)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    Ks = -(-K // world)
    return min(K, rank * Ks), min(K, (rank + 1) * Ks), Ks


def allreduce_grads(grad: torch.Tensor, sums: torch.Tensor | None, group=None) -> None:
    """Sum per-band gradients and, if given, loss partials over the ranks,
    in place (the replicated-update form; kept for reference and tests)."""
    dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
    if sums is not None:
        dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)


def reduce_scatter_grads(grad_pad: torch.Tensor, shard: torch.Tensor, sums: torch.Tensor, group=None) -> None:
    """Steps 1-2: ``shard`` [Ks, Pk] <- sum over ranks of this rank's rows of
    ``grad_pad`` [world Ks, Pk]; ``sums`` all-reduced in place."""
    dist.reduce_scatter_tensor(shard, grad_pad, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)


def allgather_params(arrays, rank: int, world: int, Ks: int, group=None) -> None:
    """Step 4: in-place all-gather of parameter arrays padded to world*Ks
    rows; rank r contributes rows [r Ks, (r+1) Ks) of each array.  ONE
    collective: the rank's shard rows of every array are packed side by side
    into a [Ks, W] send buffer (W = the arrays' row widths summed: 6 + C E),
    gathered into [world, Ks, W] and unpacked (one collective launch and
    latency instead of four; the bytes are the same)."""
    views = [a.view(world, Ks, -1) for a in arrays]
    widths = [v.shape[2] for v in views]
    send = torch.cat([v[rank] for v in views], dim=1)
    recv = torch.empty((world,) + tuple(send.shape), dtype=send.dtype, device=send.device)
    dist.all_gather_into_tensor(recv.view(-1), send.view(-1), group=group)
    off = 0
    for v, w in zip(views, widths):
        v.copy_(recv[:, :, off:off + w])
        off += w


def padded(params, world: int):
    """A copy of ``params`` (smoe.Params) whose four arrays have
    Kpad = world ceil(K / world) rows (pad rows zero; the library reads only
    the first K), as the in-place all-gather needs."""
    from .smoe import Params
    K = params.mu.shape[0]
    Kpad = world * (-(-K // world))

    def pad(t):
        out = torch.zeros((Kpad,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        out[:K].copy_(t)
        return out

    return Params(pad(params.mu), pad(params.chol), pad(params.log_pi), pad(params.expert))


class BandedFit:
    """Data-parallel fit of one image across the ranks of ``group``.

    ``params`` passed to :meth:`step` must come from :func:`padded` (arrays of
    Kpad rows) so that the parameter all-gather works in place."""

    def __init__(self, handle, rank: int, world: int, group=None):
        self.h = handle
        self.rank, self.world, self.group = rank, world, group
        ny = (handle.H + 15) // 16
        self.band = band_rows(ny, rank, world)
        if self.band[1] > self.band[0]:
            handle.set_band(*self.band)
        self.k0, self.k1, self.Ks = shard_rows(handle.K, rank, world)
        dev = f"cuda:{handle.device}"
        Kpad = world * self.Ks
        self.grad_pad = torch.zeros((Kpad, handle.Pk), dtype=torch.float32, device=dev)
        self.grad = self.grad_pad[:handle.K]          # the library's [K, Pk] view (contiguous)
        self.shard = torch.zeros((self.Ks, handle.Pk), dtype=torch.float32, device=dev)
        self.sums = torch.zeros(4, dtype=torch.float64, device=dev)

    def _once(self, params, target, lr):
        if self.band[1] > self.band[0]:
            self.h.grad(params, target, self.grad, self.sums)
        else:  # more ranks than block rows: this rank contributes nothing
            self.grad.zero_()
            self.sums.zero_()
        reduce_scatter_grads(self.grad_pad, self.shard, self.sums, self.group)
        self.h.apply(params, self.shard[:self.k1 - self.k0], lr, self.k0, self.k1, sums=self.sums)
        allgather_params((params.mu, params.chol, params.log_pi, params.expert), self.rank, self.world,
                         self.Ks, self.group)

    def step(self, params, target, lr, check: bool = False):
        """One fit iteration, asynchronous.  Returns the all-reduced band sums
        (SSE, clamped SSE, uncovered pixels, skipped) as a device tensor.  A
        step that some rank's list overflow made every rank skip alike
        surfaces at the next ``sync``; with ``check`` the call synchronises
        instead and, on a skip, grows the lists and redoes the step."""
        for attempt in range(4):
            self._once(params, target, lr)
            if not check or float(self.sums[3]) == 0.0 or attempt == 3:
                return self.sums
            self.sync(grow=True)

    def sync(self, grow: bool = False):
        """Synchronise the rank's handle; with ``grow`` a capacity report
        (this rank's lists were grown) is expected and swallowed."""
        from .smoe import ERR_CAPACITY, SmoeError
        try:
            return self.h.sync()
        except SmoeError as e:
            if grow and e.status == ERR_CAPACITY:
                return None
            raise
