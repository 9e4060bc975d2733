"""Seeded synthetic inputs shared by the tests, the bench and smoke().

This module holds NO arithmetic of the method (no kernels, gates, boxes,
gradients or optimiser): only random numbers and image synthesis.  Both the
CUDA path and the CPU oracle receive the arrays it produces.  The recipe is
stated in DESIGN.md ("Input recipe"); the shapes follow BASELINE.json configs:

* target images: piecewise-smooth "natural-like" content -- a Voronoi
  partition with about H*W/4000 regions, each with a base colour plus a
  linear shading ramp, 1-px anti-aliased region edges, plus a band-limited
  texture (8 random sinusoids, amplitude 0.03), clamped to [0, 1];
* additive Gaussian noise N(0, sigma^2), unclamped (config 4, sigma=25/255);
* kernel pools: the paper's random round init (centres
  uniform over the image, isotropic 5 px scale, expert = target colour at the
  nearest pixel, log_pi = 0, slopes 0) and, for parity, anisotropic pools
  (l11, l22 ~ U[1.5, 8], l21 ~ U[-4, 4]).

Seeds: image ``1234 + cfg``, kernels ``seed + 1``, noise ``seed + 2``.  The
generator is numpy's counter-based Philox.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(int(seed)))


def image(H: int, W: int, C: int, seed: int) -> np.ndarray:
    """Planar float32 [C][H][W] image in [0,1] (recipe in the module doc)."""
    from scipy.spatial import cKDTree

    g = rng(seed)
    n_reg = max(2, (H * W) // 4000)
    seeds = np.stack([g.uniform(0, W, n_reg), g.uniform(0, H, n_reg)], 1)
    base = g.uniform(0.05, 0.95, (n_reg, C))
    ramp = g.normal(0, 0.004, (n_reg, C, 2))
    tree = cKDTree(seeds)
    out = np.empty((C, H, W), np.float32)
    k_freq = g.uniform(0.02, 0.6, (8, 2)) * g.choice([-1, 1], (8, 2))
    k_phase = g.uniform(0, 2 * np.pi, (8, C))
    rows = max(1, (1 << 22) // max(W, 1))        # process in row chunks
    xs = np.arange(W, dtype=np.float64)
    for r0 in range(0, H, rows):
        r1 = min(H, r0 + rows)
        yy, xx = np.meshgrid(np.arange(r0, r1, dtype=np.float64), xs, indexing="ij")
        pts = np.stack([xx.ravel(), yy.ravel()], 1)
        dist, idx = tree.query(pts, k=2, workers=-1)
        i1, i2 = idx[:, 0], idx[:, 1]
        # signed distance to the bisector of the two nearest seeds -> 1 px AA
        sep = np.linalg.norm(seeds[i1] - seeds[i2], axis=1) + 1e-9
        bis = (dist[:, 1] ** 2 - dist[:, 0] ** 2) / (2.0 * sep)
        alpha = np.clip(0.5 + bis, 0.0, 1.0)[:, None]

        def shade(i):
            off = pts - seeds[i]
            return base[i] + ramp[i, :, 0] * off[:, 0:1] + ramp[i, :, 1] * off[:, 1:2]

        col = alpha * shade(i1) + (1.0 - alpha) * shade(i2)
        tex = np.zeros_like(col)
        for s in range(8):
            ph = xx.ravel() * k_freq[s, 0] + yy.ravel() * k_freq[s, 1]
            tex += 0.03 / 8 * np.sin(ph[:, None] + k_phase[s][None, :])
        col = np.clip(col + tex, 0.0, 1.0)
        out[:, r0:r1, :] = col.T.reshape(C, r1 - r0, W).astype(np.float32)
    return out


def noisy(img: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """img + N(0, sigma^2), unclamped (reading Q21)."""
    g = rng(seed)
    return (img + g.normal(0.0, sigma, img.shape)).astype(np.float32)


@dataclass
class Pool:
    """Kernel parameters, float32, in the C-ABI layout."""
    mu: np.ndarray       # [K,2]
    chol: np.ndarray     # [K,3] (l11, l21, l22)
    log_pi: np.ndarray   # [K]
    expert: np.ndarray   # [K,C,E]

    @property
    def K(self):
        return self.mu.shape[0]

    def copy(self):
        return Pool(self.mu.copy(), self.chol.copy(), self.log_pi.copy(), self.expert.copy())


def paper_init(target: np.ndarray, K: int, seed: int, order: int = 0, scale_px: float = 5.0) -> Pool:
    """Random round kernels with the fixed 5 px scale."""
    C, H, W = target.shape
    g = rng(seed)
    mu = np.stack([g.uniform(0, W, K), g.uniform(0, H, K)], 1).astype(np.float32)
    chol = np.tile(np.array([scale_px, 0.0, scale_px], np.float32), (K, 1))
    log_pi = np.zeros(K, np.float32)
    E = 1 + 2 * order
    expert = np.zeros((K, C, E), np.float32)
    ix = np.clip(np.rint(mu[:, 0]).astype(np.int64), 0, W - 1)
    iy = np.clip(np.rint(mu[:, 1]).astype(np.int64), 0, H - 1)
    expert[:, :, 0] = target[:, iy, ix].T
    return Pool(mu, chol, log_pi, expert)


def aniso_pool(H: int, W: int, C: int, K: int, seed: int, order: int = 0,
               l_range=(1.5, 8.0), shear=4.0, log_pi_sd=0.0, slope_sd=0.02,
               margin_px: float = 0.0) -> Pool:
    """Anisotropic parity pool: l11, l22 ~ U[l_range], l21 ~ U[-shear, shear],
    centres uniform over the image widened by ``margin_px`` on each side."""
    g = rng(seed)
    mu = np.stack([g.uniform(-margin_px, W + margin_px, K),
                   g.uniform(-margin_px, H + margin_px, K)], 1).astype(np.float32)
    chol = np.stack([g.uniform(*l_range, K), g.uniform(-shear, shear, K),
                     g.uniform(*l_range, K)], 1).astype(np.float32)
    log_pi = (g.normal(0.0, log_pi_sd, K) if log_pi_sd > 0 else np.zeros(K)).astype(np.float32)
    E = 1 + 2 * order
    expert = np.zeros((K, C, E), np.float32)
    expert[:, :, 0] = g.uniform(0.0, 1.0, (K, C))
    if order == 1:
        expert[:, :, 1:] = g.normal(0.0, slope_sd, (K, C, 2))
    return Pool(mu, chol, log_pi, expert.astype(np.float32))


# BASELINE.json configs (shape only; the recipe above fills them).
CONFIGS = {
    "tiny":   dict(cfg=1, H=64, W=64, C=1, K=64, order=0, iters=20),
    "kodak":  dict(cfg=2, H=512, W=768, C=3, K=10_000, order=1, iters=2000),
    "div2k":  dict(cfg=3, H=1356, W=2040, C=3, K=100_000, order=0, iters=2000, sr=4),
    "denoise": dict(cfg=4, H=512, W=512, C=3, K=20_000, order=0, iters=2000, noise=25 / 255, sr=2),
    "8k":     dict(cfg=5, H=4320, W=7680, C=3, K=1_000_000, order=0, iters=2000),
}


def workload(name: str, K: int = 0):
    """(target, clean_image_or_None, pool) for a named BASELINE.json config
    (K > 0 overrides the kernel count: density sweeps)."""
    c = dict(CONFIGS[name])
    if K > 0:
        c["K"] = K
    s = 1234 + c["cfg"]
    img = image(c["H"], c["W"], c["C"], s)
    target = noisy(img, c["noise"], s + 2) if "noise" in c else img
    pool = paper_init(target, c["K"], s + 1, c["order"])
    return target, img, pool
