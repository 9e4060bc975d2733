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


def assert_grads(g, g_ref, a_ref, rel=1e-4, floor=1e-5, what="grad", b_ref=None, opnd=2.0 ** -20):
    """North-star gradient tolerance 1e-4 relative with the floor 1e-5 A_ref
    (A_ref = sum over pixels of |per-pixel term|), plus
    16 fp32 ulps (2^-20) of the operand scale B_ref (the same sum with every
    difference inside a term -- y - t, m_j(x) - y -- replaced by the sum of
    its operands' magnitudes; O.loss_grad's grad_opnd): a
    term whose residual or expert-minus-output nearly cancels carries the
    rounding error of its operands, not of its value."""
    g = np.asarray(g, np.float64)
    d = np.abs(g - g_ref)
    tol = rel * np.abs(g_ref) + floor * a_ref
    if b_ref is not None:
        tol = tol + opnd * b_ref
    bad = d > tol
    if bad.any():
        i = np.unravel_index(np.argmax(d / np.maximum(tol, 1e-300)), d.shape)
        raise AssertionError(f"{what}: {bad.sum()} of {bad.size} out of tolerance; worst at {i}: "
                             f"gpu {g[i]:.6e} ref {g_ref[i]:.6e} A {a_ref[i]:.3e}")


def oracle_fit_with_tolerance(op, target, T, lr_of_t, R2=None, rel=1e-4, floor=1e-5, tau_d=1e-4):
    """Oracle fit (dense loss + analytic gradient + Adam per step) that
    also returns, per parameter component, how far an fp32 run may drift from
    it after T steps when its gradient meets the north-star tolerance
    tol_g = rel|g| + floor A_ref at every step ("Trajectory
    tolerance").  Adam divides the first moment by sqrt(v), so a gradient
    error tol_g moves a step by at most lr * 2 tol_g / sqrt(v) (first-order
    in m and v), and never by more than 2 lr max(1, |m^|/sqrt(v^)) (two
    updates of opposite sign: a component whose gradient is below tol_g has
    an undetermined sign).  fp32 storage adds half an ulp of the parameter
    per step.

    Rule P1 holds for the initial parameters only: as the fit moves them, a
    (pixel, kernel) pair can come within fp32 reach of the cull boundary
    d^2 = R2 at some step, where fp32 and fp64 may decide it differently and
    every gradient that pixel feeds is undetermined.  At each step the
    oracle's margins (O.margins) flag such kernels, with the threshold
    widened by how far the fp32 parameters may already be off (d^2 moves by
    <= 2 R |dmu| / s_min + 2 R2 |dL| / s_min, s_min the smaller singular
    value of L); that step's update of every kernel whose box overlaps a
    flagged kernel's box gets the undetermined-sign bound.
    Returns (params, trace[(loss, psnr)], tol[K][Pk])."""
    R2v = O.R2_99() if R2 is None else R2
    C, H, W = np.asarray(target).shape
    opt = O.Adam(op.K, op.Pk)
    p = op.copy()
    tol = np.zeros((op.K, op.Pk))
    trace = []
    for t in range(T):
        lg = O.loss_grad(p, target, R2=R2)
        trace.append((lg.loss, lg.psnr))
        affected = np.zeros(op.K, bool)
        if np.isfinite(R2v):
            dg, _ = O.margins(p, H, W, R2=R2v)
            ch = p.chol
            # smallest singular value of L = [[l11, 0], [l21, l22]]
            a2 = ch[:, 0] ** 2 + ch[:, 1] ** 2 + ch[:, 2] ** 2
            det = np.abs(ch[:, 0] * ch[:, 2])
            smin = np.sqrt(np.maximum((a2 - np.sqrt(np.maximum(a2 ** 2 - 4 * det ** 2, 0))) / 2, 1e-30))
            R = np.sqrt(R2v)
            reach = tau_d + (2 * R * tol[:, 0:2].sum(1) + 2 * R2v * tol[:, 2:5].sum(1)) / smin
            flag = np.flatnonzero(dg < reach)
            if flag.size:
                pb, _, _ = O.boxes(p, H, W, R2=R2v)
                ok = pb[:, 0] >= 0
                for k in flag:
                    if pb[k, 0] < 0:
                        continue
                    affected |= ok & (pb[:, 0] <= pb[k, 1]) & (pb[:, 1] >= pb[k, 0]) & \
                        (pb[:, 2] <= pb[k, 3]) & (pb[:, 3] >= pb[k, 2])
        lr = lr_of_t(t)
        lrv = lr.vector(op.C, op.order)[None, :]
        p = opt.step(p, lg.grad, lr)
        mhat = opt.m1 / (1.0 - O.BETA1 ** opt.t)
        rms = np.sqrt(opt.m2 / (1.0 - O.BETA2 ** opt.t)) + O.EPS
        tg = rel * np.abs(lg.grad) + floor * lg.grad_abs + 2.0 ** -20 * lg.grad_opnd
        cap = 2.0 * np.maximum(1.0, np.abs(mhat) / rms)
        step = np.minimum(cap, 2.0 * tg / rms)
        step[affected] = cap[affected]
        tol += lrv * step + 2.0 ** -24 * np.abs(p.flat())
    return p, trace, tol


def assert_params(got, ref, tol, factor=2.0, what="params"):
    """Every component within factor x tol (no outlier budget); the factor
    covers the feedback of parameter differences into later gradients, which
    the first-order tol of oracle_fit_with_tolerance leaves out."""
    got = np.asarray(got, np.float64)
    d = np.abs(got - ref)
    lim = factor * tol
    bad = d > lim
    if bad.any():
        i = np.unravel_index(np.argmax(d / np.maximum(lim, 1e-300)), d.shape)
        raise AssertionError(f"{what}: {bad.sum()} of {bad.size} beyond {factor} x tol; worst at {i}: "
                             f"gpu {got[i]:.8e} ref {ref[i]:.8e} tol {tol[i]:.3e}")
    return float((d / np.maximum(lim, 1e-300)).max())


def conditioned_mode(pool, H, W, out_H=None, out_W=None, mode="square", seed=0, tau_d=1e-4, tau_b=1e-3,
                     rounds=40):
    """Rule P1 for a box mode: also keep the mode's box edges tau_b from an
    integer and (mode "exact") every candidate block's rectangle minimum of
    d^2 tau_d from R2, so fp32 and fp64 list the same blocks."""
    g = np.random.default_rng(seed)
    pool = pool.copy()
    for _ in range(rounds):
        p = O.Params.from_any(pool)
        dg, eg = O.margins(p, H, W, out_H, out_W)
        em, rm = O.mode_margins(p, H, W, out_H, out_W, mode=mode)
        bad = (dg <= tau_d) | (eg <= tau_b) | (em <= tau_b) | (rm <= tau_d)
        if not bad.any():
            return pool
        pool.mu[bad] += g.uniform(-0.5, 0.5, (int(bad.sum()), 2)).astype(np.float32)
    raise AssertionError("could not margin-condition the pool for the box mode")
