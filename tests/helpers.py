"""Shared test helpers: margin conditioning (rule P1) and tolerance checks.

Rule P1: generated parity inputs
are re-jittered until every (pixel, kernel) pair is at least tau_d from the
cull boundary d^2 = R2 and every box edge at least tau_b px from an integer,
so that fp32 and fp64 take the same discrete decisions.  The check uses the
oracle's fp64 margins (tests may call the oracle).
"""
import numpy as np

import oracle as O


def conditioned(pool, H, W, out_H=None, out_W=None, seed=0, tau_d=1e-4, tau_b=1e-3, rounds=30):
    g = np.random.default_rng(seed)
    pool = pool.copy()
    for _ in range(rounds):
        dg, eg = O.margins(O.Params.from_any(pool), H, W, out_H, out_W)
        bad = (dg <= tau_d) | (eg <= tau_b)
        if not bad.any():
            return pool
        pool.mu[bad] += g.uniform(-0.5, 0.5, (int(bad.sum()), 2)).astype(np.float32)
    raise AssertionError("could not margin-condition the pool")


def conditioned_multi(pool, H, W, rasters, **kw):
    """Condition for several output rasters at once."""
    for _ in range(10):
        for (oH, oW) in rasters:
            pool = conditioned(pool, H, W, oH, oW, **kw)
        ok = True
        for (oH, oW) in rasters:
            dg, eg = O.margins(O.Params.from_any(pool), H, W, oH, oW)
            ok &= bool(((dg > kw.get("tau_d", 1e-4)) & (eg > kw.get("tau_b", 1e-3))).all())
        if ok:
            return pool
    raise AssertionError("multi-raster conditioning failed")


def assert_pixels(y, y_ref, rel=1e-5, abs_=1e-6, what="pixels"):
    """North-star pixel tolerance: |dy| <= 1e-5 |y_ref| + 1e-6."""
    y = np.asarray(y, np.float64)
    d = np.abs(y - y_ref)
    tol = rel * np.abs(y_ref) + abs_
    bad = d > tol
    assert not bad.any(), f"{what}: {bad.sum()} of {bad.size} out of tolerance, worst {d.max():.3e}"


def assert_grads(g, g_ref, a_ref, rel=1e-4, floor=1e-5, what="grad"):
    """North-star gradient tolerance 1e-4 relative with the floor 1e-5 A_ref
    (A_ref = sum over pixels of |per-pixel term|), SURVEY §8(c)."""
    g = np.asarray(g, np.float64)
    d = np.abs(g - g_ref)
    tol = rel * np.abs(g_ref) + floor * a_ref
    bad = d > tol
    if bad.any():
        i = np.unravel_index(np.argmax(d / np.maximum(tol, 1e-300)), d.shape)
        raise AssertionError(f"{what}: {bad.sum()} of {bad.size} out of tolerance; worst at {i}: "
                             f"gpu {g[i]:.6e} ref {g_ref[i]:.6e} A {a_ref[i]:.3e}")
