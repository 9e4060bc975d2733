"""Multi-model R-SMoE (MM-RSMoE) for denoising.

P:279-310: H independently trained SMoE models of the same noisy image are
fused by averaging their predictions, y_m(x) = (1/H) sum_h y'_h(x) (Eq. 11),
which divides the variance of the model noise by H (Eq. 14).  The paper's
hypotheses come from shifted block windows; here every hypothesis
h is a full-image fit whose random kernel pool is drawn with its own seed and
whose centres are displaced by the hypothesis' shift (the paper's window
shifts [2, 4, ..., 16] px), so the hypotheses differ in initialisation the
way the shifted windows do.  Each hypothesis has its own library handle and
CUDA stream; the H fits run concurrently on one GPU (replicas across GPUs
need no collective).  The fusion runs in the render kernel
(smoe_render_ex with accumulate = 1/H).
"""
from __future__ import annotations

import numpy as np
import torch

from . import smoe, synth


def hypothesis_shifts(H: int, step: int = 2) -> list[tuple[int, int]]:
    """Window shifts (dx, dy) of the H hypotheses: multiples of ``step`` px
    (P:310 uses 2-pixel steps up to 16), row-major over a square grid."""
    n = int(np.ceil(np.sqrt(H)))
    return [((i % n) * step, (i // n) * step) for i in range(H)]


def init_hypotheses(target: np.ndarray, K: int, H: int, seed: int, order: int = 0):
    """Per-hypothesis kernel pools: paper init with seed
    seed + h, centres shifted by the hypothesis' window shift (mod image)."""
    C, Hh, Ww = target.shape
    pools = []
    for h, (dx, dy) in enumerate(hypothesis_shifts(H)):
        p = synth.paper_init(target, K, seed + h, order)
        p.mu[:, 0] = np.mod(p.mu[:, 0] + dx, Ww).astype(np.float32)
        p.mu[:, 1] = np.mod(p.mu[:, 1] + dy, Hh).astype(np.float32)
        pools.append(p)
    return pools


class MultiModel:
    """H concurrent fits of one image and their fused render."""

    def __init__(self, H: int, K: int, height: int, width: int, C: int, order: int = 0, **kw):
        self.H = H
        self.handles = [smoe.SMoE(K, height, width, C, order, **kw) for _ in range(H)]
        self.streams = [torch.cuda.Stream() for _ in range(H)]
        self.shape = (C, height, width)

    def step(self, params: list, target: torch.Tensor, lr: smoe.LR):
        """One asynchronous iteration of every hypothesis, each on its stream."""
        cur = torch.cuda.current_stream()
        for h, s in zip(self.handles, self.streams):
            s.wait_stream(cur)
        for h, s, p in zip(self.handles, self.streams, params):
            with torch.cuda.stream(s):
                h.step(p, target, lr, stats=False)
        for s in self.streams:
            cur.wait_stream(s)

    def fit(self, params: list, target: torch.Tensor, T: int):
        for t in range(T):
            self.step(params, target, smoe.LR.paper(t, T))
        for h in self.handles:
            h.sync()

    def render(self, params: list, out_H: int | None = None, out_W: int | None = None, sharpen: float = 1.0):
        """Fused prediction y_m = (1/H) sum_h y_h (Eq. 11) on out_H x out_W."""
        C, Hh, Ww = self.shape
        out_H = Hh if out_H is None else out_H
        out_W = Ww if out_W is None else out_W
        out = torch.zeros((C, out_H, out_W), dtype=torch.float32, device="cuda")
        for h, p in zip(self.handles, params):
            h.render(p, out_H, out_W, out=out, sharpen=sharpen, accumulate=1.0 / self.H)
        return out
