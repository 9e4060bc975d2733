"""Pins for the CPU oracle (CPU only, no GPU).

Each test checks the oracle against something OTHER than its own formula:
worked examples printed in SPEC.md / constants in PAPER.md
(tests/golden/spec_examples.json, each entry cited), closed forms,
library routines (numpy eigvalsh / inv), brute-force enumeration and central
finite differences, and invariants of the model.  The comments name which
plausible mistake each pin would catch.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
from paper_2510_05814_b200 import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
INF = float("inf")


def chol_of(S):
    """Cholesky factor (l11, l21, l22) of a 2x2 SPD matrix via numpy."""
    L = np.linalg.cholesky(np.asarray(S, float))
    return np.array([L[0, 0], L[1, 0], L[1, 1]])


def params(mus, chols, ms, log_pi=None, order=0):
    mus = np.asarray(mus, float).reshape(-1, 2)
    K = mus.shape[0]
    ms = np.asarray(ms, float).reshape(K, -1)
    C = ms.shape[1]
    E = 1 + 2 * order
    ex = np.zeros((K, C, E))
    ex[:, :, 0] = ms
    lp = np.zeros(K) if log_pi is None else np.asarray(log_pi, float)
    return O.Params(mus, np.asarray(chols, float).reshape(K, 3), lp, ex)


def pool_params(pool):
    return O.Params.from_any(pool)


def conditioned(pool, H, W, out_H=None, out_W=None, seed=0, tau_d=1e-4, tau_b=1e-3):
    """Rule P1: re-jitter centres until every (pixel, kernel)
    pair is at least tau_d from the cull boundary and every box edge at least
    tau_b px from an integer.  Works on the float32 pool."""
    g = np.random.default_rng(seed)
    pool = pool.copy()
    for _ in range(20):
        dg, eg = O.margins(pool_params(pool), H, W, out_H, out_W)
        bad = (dg <= tau_d) | (eg <= tau_b)
        if not bad.any():
            return pool
        pool.mu[bad] += g.uniform(-0.5, 0.5, (bad.sum(), 2)).astype(np.float32)
    raise AssertionError("could not margin-condition the pool")


# ------------------------------------------------------------ constants ----

def test_R2_closed_form():
    # chi2_2 CDF 1-exp(-x/2): the 99% quantile puts K = exp(-R2/2) at 0.01 exactly
    R2 = O.R2_99()
    assert abs(math.exp(-R2 / 2) - 0.01) < 1e-16
    assert abs(R2 - GOLD["chi2_99_2dof"]["R2"]) < 5e-5          # S:187/S:210 table value
    # an R2 mistake (e.g. R=3 -> 9, or chi2 with 1 dof 6.63) is caught here


def test_cov_from_chol_spec():
    for ex in GOLD["cov_from_chol"]:
        np.testing.assert_allclose(O.cov(ex["chol"]), ex["sigma"], atol=0, rtol=0, err_msg=ex["cite"])


def test_mahalanobis_and_kernel_eval_spec():
    for ex in GOLD["mahalanobis2"]:
        d2 = O.d2([0.0, 0.0], chol_of(ex["sigma"]), *ex["offset"])
        assert abs(d2 - ex["d2"]) < 1e-12, ex["cite"]
    for ex in GOLD["kernel_eval"]:
        d2 = O.d2(ex["mu"], chol_of(ex["sigma"]), *ex["x"])
        assert abs(math.exp(-0.5 * d2) - ex["K"]) < 5e-6, ex["cite"]


def test_d2_matches_numpy_inverse_random():
    # transposed-operand / sign mistakes in the adjugate fail against np.linalg.inv
    g = np.random.default_rng(1)
    for _ in range(200):
        ch = np.array([g.uniform(0.3, 9), g.uniform(-5, 5), g.uniform(0.3, 9)])
        L = np.array([[ch[0], 0], [ch[1], ch[2]]])
        S = L @ L.T
        mu = g.uniform(-10, 10, 2)
        x = g.uniform(-20, 20, 2)
        ref = (x - mu) @ np.linalg.inv(S) @ (x - mu)
        assert abs(O.d2(mu, ch, *x) - ref) <= 1e-10 * max(1, ref)


def test_lambda_max_spec_and_eigvalsh():
    for ex in GOLD["eig2x2_lambda_max"]:
        assert abs(O.lambda_max(chol_of(ex["sigma"])) - ex["lmax"]) < 1e-12, ex["cite"]
    g = np.random.default_rng(2)
    for _ in range(200):
        ch = np.array([g.uniform(0.3, 9), g.uniform(-5, 5), g.uniform(0.3, 9)])
        L = np.array([[ch[0], 0], [ch[1], ch[2]]])
        ref = np.linalg.eigvalsh(L @ L.T).max()
        assert abs(O.lambda_max(ch) - ref) <= 1e-11 * ref


def test_box_side_spec():
    for ex in GOLD["bounding_box_side"]:
        p = params([[100.0, 100.0]], [chol_of(ex["sigma"])], [[0.5]])
        _, _, hs = O.boxes(p, 256, 256)
        assert abs(2 * hs[0] - ex["side"]) < 5e-4, ex["cite"]
    # Sigma scaled by 4 -> side doubles
    p1 = params([[50.0, 50.0]], [[1.3, 0.4, 0.9]], [[0.5]])
    p4 = params([[50.0, 50.0]], [[2.6, 0.8, 1.8]], [[0.5]])
    assert abs(O.boxes(p4, 128, 128)[2][0] - 2 * O.boxes(p1, 128, 128)[2][0]) < 1e-12


def test_tile_index_spec_example():
    ex = GOLD["tile_index"]
    l = ex["half_side"] / math.sqrt(O.R2_99())
    p = params([ex["mu"]], [[l, 0.0, l]], [[0.5]])
    _, tb, _ = O.boxes(p, ex["H"], ex["W"])
    assert list(range(tb[0, 0], tb[0, 1] + 1)) == ex["blocks_x"]
    assert list(range(tb[0, 2], tb[0, 3] + 1)) == ex["blocks_y"]


@pytest.mark.parametrize("scale", [1.0, 2.0, 4.0, 0.5, 1.5])
def test_tiles_brute_force(scale):
    """Tile lists vs brute force: enumerate every output pixel whose sample
    point lies in the square box (half side from numpy eigvalsh), collect its
    block; also check the coverage invariant: every pixel with
    d2 <= R2 has the kernel in its block's list."""
    H, W = 37, 53
    oH, oW = int(round(H * scale)), int(round(W * scale))
    pool = synth.aniso_pool(H, W, 1, 40, seed=11, margin_px=6)
    pool = conditioned(pool, H, W, oH, oW)
    p = pool_params(pool)
    R2 = O.R2_99()
    nx, ny = -(-oW // 16), -(-oH // 16)
    _, tb, _ = O.boxes(p, H, W, oH, oW)
    rng_, ids = O.tile_list(tb, nx, ny)
    lists = [set(ids[rng_[n]:rng_[n + 1]].tolist()) for n in range(nx * ny)]
    xs = (np.arange(oW) + 0.5) * W / oW - 0.5
    ys = (np.arange(oH) + 0.5) * H / oH - 0.5
    for k in range(p.K):
        L = np.array([[p.chol[k, 0], 0], [p.chol[k, 1], p.chol[k, 2]]])
        S = L @ L.T
        r = math.sqrt(R2 * np.linalg.eigvalsh(S).max())
        inx = np.nonzero(np.abs(xs - p.mu[k, 0]) <= r)[0]
        iny = np.nonzero(np.abs(ys - p.mu[k, 1]) <= r)[0]
        bf = {(iy // 16) * nx + ix // 16 for iy in iny for ix in inx}
        got = {n for n in range(nx * ny) if k in lists[n]}
        assert bf == got, f"kernel {k}"
        Si = np.linalg.inv(S)
        for iy in iny:
            for ix in inx:
                dvec = np.array([xs[ix], ys[iy]]) - p.mu[k]
                if dvec @ Si @ dvec <= R2:
                    assert k in lists[(iy // 16) * nx + ix // 16]
    # canonical order: ascending tile, ascending kernel within a tile
    for n in range(nx * ny):
        seg = ids[rng_[n]:rng_[n + 1]]
        assert np.all(np.diff(seg) > 0)


def test_tile_list_band_restriction():
    H, W = 64, 48
    pool = synth.aniso_pool(H, W, 1, 30, seed=3)
    p = pool_params(pool)
    _, tb, _ = O.boxes(p, H, W)
    nx, ny = 3, 4
    full_r, full_ids = O.tile_list(tb, nx, ny)
    for ty0, ty1 in [(0, 1), (1, 3), (3, 4)]:
        r, ids = O.tile_list(tb, nx, ny, (ty0, ty1))
        a, b = full_r[ty0 * nx], full_r[ty1 * nx]
        np.testing.assert_array_equal(ids, full_ids[a:b])


# --------------------------------------------------------------- render ----

def test_gates_and_render_point_spec():
    ex = GOLD["gates_at"][0]
    p = params(ex["mus"], [[1, 0, 1]] * 2, [[0.0], [0.0]])
    w, _ = O.gates(p, *ex["x"], R2=INF)
    np.testing.assert_allclose(w, ex["w"], rtol=1e-12, err_msg=ex["cite"])
    for ex in GOLD["render_point"]:
        K = len(ex["mus"])
        p = params(ex["mus"], [[1, 0, 1]] * K, [[m] for m in ex["m"]])
        y, _ = O.render_points(p, [ex["x"][0]], [ex["x"][1]], R2=INF)
        assert abs(y[0, 0] - ex["y"]) < 1e-12, ex["cite"]
    # with truncation both kernels of S:141 are culled at (0,0): d2 = 25 > R2 -> Q7 gives 0
    p = params([[-5, 0], [5, 0]], [[1, 0, 1]] * 2, [[0.1], [0.9]])
    y, D = O.render_points(p, [0.0], [0.0])
    assert y[0, 0] == 0.0 and D[0] == 0.0


def test_partition_of_unity_and_convex_hull():
    H, W = 24, 31
    pool = synth.aniso_pool(H, W, 3, 25, seed=5, log_pi_sd=0.7)
    p = pool_params(pool)
    g = np.random.default_rng(0)
    for _ in range(300):
        x, y = g.uniform(-2, W + 1), g.uniform(-2, H + 1)
        w, D = O.gates(p, x, y)
        if D > 0:
            assert abs(w.sum() - 1.0) < 1e-12
            assert np.all(w >= 0)
        else:
            assert np.all(w == 0)
    y, D = O.render(p, H, W)
    cov = D > 0
    m = p.expert[:, :, 0]
    # SMoE output is a convex combination of the experts
    for c in range(3):
        assert np.all(y[c][cov] >= m[:, c].min() - 1e-12)
        assert np.all(y[c][cov] <= m[:, c].max() + 1e-12)
        assert np.all(y[c][~cov] == 0.0)


def test_pi_shift_invariance():
    H, W = 20, 20
    pool = synth.aniso_pool(H, W, 1, 15, seed=6, log_pi_sd=0.5)
    p = pool_params(pool)
    q = p.copy()
    q.log_pi = q.log_pi + 1.7
    y1, D1 = O.render(p, H, W)
    y2, D2 = O.render(q, H, W)
    np.testing.assert_allclose(y1, y2, atol=1e-12)
    np.testing.assert_allclose(D2, D1 * math.exp(1.7), rtol=1e-12)


def test_single_kernel_closed_form():
    """One kernel: gate = 1 inside the ellipse (d2 from numpy inv), so
    y = m (constant) or m + W(x-mu) (linear) inside and 0 outside."""
    H, W = 30, 26
    mu = np.array([12.3, 14.6])
    ch = np.array([4.0, 1.5, 2.5])
    for order in (0, 1):
        p = params([mu], [ch], [[0.3, 0.6, 0.9]], order=order)
        if order:
            p.expert[0, :, 1] = [0.01, -0.02, 0.03]
            p.expert[0, :, 2] = [-0.015, 0.005, 0.02]
        y, D = O.render(p, H, W)
        L = np.array([[ch[0], 0], [ch[1], ch[2]]])
        Si = np.linalg.inv(L @ L.T)
        R2 = O.R2_99()
        for i in range(H):
            for j in range(W):
                dv = np.array([j, i]) - mu
                inside = dv @ Si @ dv <= R2
                for c in range(3):
                    e = p.expert[0, c]
                    ref = (e[0] + (e[1] * dv[0] + e[2] * dv[1] if order else 0.0)) if inside else 0.0
                    assert abs(y[c, i, j] - ref) < 1e-12


def test_two_kernel_logistic_closed_form():
    """Equal isotropic sigma at (x0 -+ a, y0) with experts m1, m2 give
    y = m1 + (m2-m1) * logistic(2 a (x - x0) / sigma^2) where both are uncut."""
    x0, y0, a, s = 20.0, 15.0, 2.5, 3.0
    m1, m2 = 0.2, 0.85
    p = params([[x0 - a, y0], [x0 + a, y0]], [[s, 0, s]] * 2, [[m1], [m2]])
    xs = np.linspace(x0 - 4, x0 + 4, 41)
    ys = np.full_like(xs, y0 + 1.0)
    y, _ = O.render_points(p, xs, ys)
    ref = m1 + (m2 - m1) / (1 + np.exp(-2 * a * (xs - x0) / s ** 2))
    np.testing.assert_allclose(y[:, 0], ref, atol=1e-14)


def test_truncation_bound_vs_untruncated():
    """Dense untruncated brute force (R2=inf) vs the truncated model:
    y_full - y_trunc = sum_{culled} g_j (m_j - y_trunc) / D_full, hence
    |y_trunc - y_full| <= (D_cut / D_full) max_{culled} |m_j - y_trunc|."""
    H, W = 14, 12
    pool = synth.aniso_pool(H, W, 1, 12, seed=7, l_range=(1.0, 3.0), shear=1.0)
    p = pool_params(pool)
    yt, Dt = O.render(p, H, W)
    yf, Df = O.render(p, H, W, R2=INF)
    # independent numpy brute force of the untruncated model (Eqs. 2-4)
    m = p.expert[:, 0, 0]
    R2 = O.R2_99()
    worst = 0.0
    for i in range(H):
        for j in range(W):
            gs, d2s = [], []
            for k in range(p.K):
                L = np.array([[p.chol[k, 0], 0], [p.chol[k, 1], p.chol[k, 2]]])
                dv = np.array([j, i]) - p.mu[k]
                d2 = dv @ np.linalg.inv(L @ L.T) @ dv
                gs.append(math.exp(p.log_pi[k] - d2 / 2))
                d2s.append(d2)
            gs, d2s = np.array(gs), np.array(d2s)
            assert abs(yf[0, i, j] - (gs @ m) / gs.sum()) < 1e-12
            cut = d2s > R2
            if Dt[i, j] > 0 and cut.any():
                bound = gs[cut].sum() / gs.sum() * np.abs(m[cut] - yt[0, i, j]).max()
                assert abs(yt[0, i, j] - yf[0, i, j]) <= bound + 1e-14
                worst = max(worst, abs(yt[0, i, j] - yf[0, i, j]))
            # each culled term is < 0.01 pi_j (kernel value below the 99% level)
            assert np.all(gs[cut] < 0.01 * np.exp(p.log_pi[cut]) + 1e-18)
    assert worst > 0  # the instance really exercises the truncation


# ----------------------------------------------------------- loss, PSNR ----

def test_loss_and_psnr_spec():
    ex = GOLD["loss"]
    H, W = 16, 16
    p = params([[7.5, 7.5]], [[40, 0, 40]], [[ex["render"]]])
    t = np.full((1, H, W), ex["target"])
    lg = O.loss_grad(p, t)
    assert abs(lg.loss - ex["mse"]) < 1e-15
    for e in GOLD["psnr"]:
        assert abs(O.psnr_from_mse(e["mse"]) - e["db"]) < 1e-12, e["cite"]
    assert O.psnr_from_mse(0.0) == float("inf")


def test_noisy_psnr_anchor():
    # noisy input at sigma^2 = 0.01 scores 20.28 dB on Kodak; our
    # generator + clamped PSNR must land near it (loose anchor: content
    # dependent through clipping, so +-0.5 dB on the mean of three images)
    vals = []
    for s in (99, 5, 7):
        img = synth.image(256, 256, 3, s)
        noisy = synth.noisy(img, 0.1, s + 1)
        vals.append(O.psnr_from_mse(np.mean((np.clip(noisy, 0, 1) - img) ** 2)))
    assert abs(np.mean(vals) - GOLD["noisy_psnr_sigma2_0.01"]["db"]) < 0.5


# ------------------------------------------------------------ gradients ----

def fd_grad(p, t, k, i, h=1e-6):
    v = p.flat()
    vp, vm = v.copy(), v.copy()
    vp[k, i] += h
    vm[k, i] -= h
    lp = O.loss_grad(O.Params.unflat(vp, p.C, p.order), t).loss
    lm = O.loss_grad(O.Params.unflat(vm, p.C, p.order), t).loss
    return (lp - lm) / (2 * h)


@pytest.mark.parametrize("C,order", [(1, 0), (3, 0), (3, 1)])
def test_gradient_central_fd(C, order):
    """Analytic gradient vs central FD on margin-conditioned
    anisotropic instances with l21 != 0, log_pi != 0 and linear slopes:
    catches a dropped chain-rule term (e.g. -a b Gb in dL/dl11), a sign
    or a transposed index."""
    H, W = 20, 23
    pool = synth.aniso_pool(H, W, C, 9, seed=20 + C + order, order=order, log_pi_sd=0.4,
                            l_range=(2.0, 6.0), slope_sd=0.05)
    pool = conditioned(pool, H, W, tau_d=1e-3)
    p = pool_params(pool)
    t = synth.image(H, W, C, 5).astype(np.float64)
    lg = O.loss_grad(p, t)
    assert lg.uncovered < H * W
    scale = np.abs(lg.grad).max()
    for k in range(p.K):
        for i in range(p.Pk):
            fd = fd_grad(p, t, k, i)
            assert abs(lg.grad[k, i] - fd) <= 1e-5 * abs(fd) + 1e-7 * scale, (k, i, lg.grad[k, i], fd)


def test_log_pi_gradient_sums_to_zero():
    # sum_j w_j (m_j(x) - y) = 0 at every covered pixel, truncation included
    H, W = 24, 24
    pool = synth.aniso_pool(H, W, 3, 30, seed=8, order=1, log_pi_sd=0.5)
    p = pool_params(pool)
    t = synth.image(H, W, 3, 9).astype(np.float64)
    lg = O.loss_grad(p, t)
    assert abs(lg.grad[:, 5].sum()) < 1e-14 * max(1.0, np.abs(lg.grad_abs[:, 5]).sum())
    assert np.abs(lg.grad[:, 5]).max() > 1e-6


def test_single_kernel_gradients():
    """One kernel covering the image partly: the gate is 1 wherever it is
    nonzero, so all geometric gradients vanish and
    dL/dm_c = 2 (n_E m_c - sum_E t_c) / (H W C), n_E = ellipse pixel count."""
    H, W, C = 20, 20, 3
    mu = np.array([9.2, 10.7])
    ch = np.array([3.0, 0.8, 2.0])
    p = params([mu], [ch], [[0.2, 0.5, 0.7]])
    t = synth.image(H, W, C, 4).astype(np.float64)
    lg = O.loss_grad(p, t)
    assert np.all(np.abs(lg.grad[0, :6]) < 1e-16)   # y = g m / g: zero up to rounding
    L = np.array([[ch[0], 0], [ch[1], ch[2]]])
    Si = np.linalg.inv(L @ L.T)
    ins = np.zeros((H, W), bool)
    for i in range(H):
        for j in range(W):
            dv = np.array([j, i]) - mu
            ins[i, j] = dv @ Si @ dv <= O.R2_99()
    nE = ins.sum()
    for c in range(C):
        ref = 2 * (nE * p.expert[0, c, 0] - t[c][ins].sum()) / (H * W * C)
        assert abs(lg.grad[0, 6 + c] - ref) < 1e-15


def test_symmetric_pair_opposite_mu_gradient():
    # mirror-symmetric configuration and target -> equal and opposite dmu_x
    H, W = 16, 31
    # mirror about x = 15 maps kernel 0 onto kernel 1 (Wx -> -Wx)
    p = params([[12.0, 7.5], [18.0, 7.5]], [[3, 0.7, 3], [3, -0.7, 3]], [[0.3], [0.3]], order=1)
    p.mu[:, 1] = 7.5
    p.expert[0, 0, 1], p.expert[1, 0, 1] = 0.05, -0.05
    p.expert[:, 0, 2] = 0.02
    xs = np.arange(W)
    t = np.tile(np.where(xs < 15, 0.1, np.where(xs > 15, 0.1, 0.9)), (H, 1))[None]
    lg = O.loss_grad(p, t)
    assert abs(lg.grad[0, 0] + lg.grad[1, 0]) < 1e-15
    assert abs(lg.grad[0, 0]) > 1e-6


def test_band_additivity():
    # gradients of disjoint row bands add up to the full gradient
    H, W = 48, 20
    pool = synth.aniso_pool(H, W, 3, 20, seed=12, order=1)
    p = pool_params(pool)
    t = synth.image(H, W, 3, 13).astype(np.float64)
    full = O.loss_grad(p, t)
    parts = [O.loss_grad(p, t, rows=r) for r in [(0, 16), (16, 32), (32, 48)]]
    np.testing.assert_allclose(sum(q.grad for q in parts), full.grad, atol=1e-16, rtol=1e-12)
    assert abs(sum(q.sse for q in parts) - full.sse) < 1e-12


def test_grad_kernels_subset_matches_full():
    H, W = 26, 22
    pool = synth.aniso_pool(H, W, 3, 15, seed=14, order=1)
    p = pool_params(pool)
    t = synth.image(H, W, 3, 15).astype(np.float64)
    full = O.loss_grad(p, t)
    sel = np.array([0, 3, 7, 14])
    g, a = O.grad_kernels(p, t, sel)
    np.testing.assert_allclose(g, full.grad[sel], rtol=1e-12, atol=1e-18)


# -------------------------------------------------------------- optimiser --

def test_adam_spec_examples():
    ex = GOLD["adam_first_step"]
    p = params([[5.0, 5.0]], [[2, 0, 2]], [[0.5]])
    opt = O.Adam(1, p.Pk)
    g = np.zeros((1, p.Pk))
    g[0, 0] = ex["g"]
    q = opt.step(p, g, O.LR(mu=ex["lr"]))
    assert abs((q.mu[0, 0] - p.mu[0, 0]) - ex["delta"]) < 1e-9
    np.testing.assert_array_equal(q.flat()[0, 1:], p.flat()[0, 1:])  # g = 0 -> unchanged
    # second step with the same gradient keeps m_hat / sqrt(v_hat) = 1
    q2 = opt.step(q, g, O.LR(mu=ex["lr"]))
    assert abs((q2.mu[0, 0] - q.mu[0, 0]) - ex["delta"]) < 1e-9


def test_adam_against_textbook_loop_and_clamp():
    # scalar Adam written out step by step (Kingma & Ba Algorithm 1)
    g = np.random.default_rng(3)
    grads = g.normal(0, 1, 30)
    x, m, v = 0.7, 0.0, 0.0
    p = params([[x, 0.0]], [[2, 0, 2]], [[0.5]])
    opt = O.Adam(1, p.Pk)
    for t, gr in enumerate(grads, 1):
        m = 0.9 * m + 0.1 * gr
        v = 0.999 * v + 0.001 * gr * gr
        x = x - 0.01 * (m / (1 - 0.9 ** t)) / (math.sqrt(v / (1 - 0.999 ** t)) + 1e-8)
        G = np.zeros((1, p.Pk))
        G[0, 0] = gr
        p = opt.step(p, G, O.LR())
    assert abs(p.mu[0, 0] - x) < 1e-14
    # clamp: a large positive l11/l22 gradient cannot push them below 1e-3
    p = params([[0.0, 0.0]], [[0.0015, 0.0, 0.0012]], [[0.5]])
    opt = O.Adam(1, p.Pk)
    G = np.zeros((1, p.Pk))
    G[0, 2] = G[0, 4] = 5.0
    q = opt.step(p, G, O.LR())
    assert q.chol[0, 0] == 1e-3 and q.chol[0, 2] == 1e-3


def test_lr_schedule_spec():
    T = 10000
    for ex in GOLD["lr_schedule"]:
        assert abs(O.lr_mu_schedule(int(ex["t_frac"] * T), T) - ex["lr"]) <= 1e-4 * ex["lr"], ex["cite"]


def test_fit_constant_target_single_kernel():
    # S:357 in spirit: a trivially fittable target converges, loss decreasing
    H, W = 16, 16
    p = params([[7.5, 7.5]], [[30, 0, 30]], [[0.45]])
    t = np.full((1, H, W), 0.5)
    q, trace = O.fit(p, t, 100)
    assert trace[-1][0] < 1e-6
    assert trace[-1][0] < trace[0][0]


# ------------------------------------------------ NEXT rows f1, f2 (oracle) --

def test_rbf_head_spec_and_closed_form():
    """Eq. (1): y = sum_j m_j K_j(x).  S:142: one kernel m = 0.8,
    Sigma = I: 0.8 at mu and 0.8 exp(-1/2) one pixel away."""
    p = params([[5.0, 5.0]], [[1, 0, 1]], [[0.8]])
    with O.head("rbf"):
        y, _ = O.render_points(p, [5.0, 6.0], [5.0, 5.0])
    assert abs(y[0, 0] - 0.8) < 1e-15
    assert abs(y[1, 0] - 0.8 * math.exp(-0.5)) < 1e-15
    assert abs(y[1, 0] - 0.48522) < 5e-6                         # printed value
    # two overlapping kernels simply add (no normalisation, unlike Eq. 4)
    p2 = params([[5.0, 5.0], [6.0, 5.0]], [[1, 0, 1]] * 2, [[0.3], [0.5]])
    with O.head("rbf"):
        y2, _ = O.render_points(p2, [5.5], [5.0])
    assert abs(y2[0, 0] - 0.8 * math.exp(-0.125)) < 1e-15


@pytest.mark.parametrize("C,order", [(1, 0), (3, 1)])
def test_rbf_gradient_central_fd(C, order):
    H, W = 18, 21
    pool = synth.aniso_pool(H, W, C, 8, seed=70 + C, order=order, log_pi_sd=0.3, l_range=(2.0, 5.0))
    pool = conditioned(pool, H, W, tau_d=1e-3)
    p = pool_params(pool)
    t = synth.image(H, W, C, 71).astype(np.float64)
    with O.head("rbf"):
        lg = O.loss_grad(p, t)
        scale = np.abs(lg.grad).max()
        for k in range(p.K):
            for i in range(p.Pk):
                fd = fd_grad(p, t, k, i)
                assert abs(lg.grad[k, i] - fd) <= 1e-5 * abs(fd) + 1e-7 * scale, (k, i)


def test_sharpening_spec_examples():
    """Kernel editing: Sigma -> s Sigma.  s = 1 is the
    identity; s = 1/4 halves every box side exactly; gates stay a partition
    of unity; a constant-expert model stays exactly constant where covered."""
    H, W = 30, 34
    pool = synth.aniso_pool(H, W, 1, 20, seed=80)
    p = pool_params(pool)
    np.testing.assert_array_equal(O.sharpened(p, 1.0).chol, p.chol)
    _, _, hs = O.boxes(p, H, W)
    _, _, hs4 = O.boxes(O.sharpened(p, 0.25), H, W)
    np.testing.assert_allclose(hs4, hs / 2, rtol=1e-15)
    q = O.sharpened(p, 0.3)
    for (x, y) in [(3.2, 4.1), (17.0, 15.5), (30.3, 2.2)]:
        w, D = O.gates(q, x, y)
        if D > 0:
            assert abs(w.sum() - 1) < 1e-12
    q.expert[:] = 0.625
    yq, Dq = O.render(q, H, W, 60, 68)
    assert np.all(np.abs(yq[0][Dq > 0] - 0.625) < 1e-15)


def test_sr_sampling_downsample_consistency_linear():
    """SR sample mapping of oracle_render (S:547 half-pixel convention; P:162,
    P:314).  A single untruncated (R2 = inf) linear-expert kernel renders the
    plane y = m + W (x - mu) exactly at every sample.  Averaging each k x k
    block of the k-times render must give the 1x render exactly: the mean of
    the k output sample positions (j+1/2)/k - 1/2 of source pixel i is i.
    S:565's low-frequency consistency check, exact for a linear model.  A
    mapping x = j/k (offset -(k-1)/(2k)) or the corner-aligned
    j (W-1)/(kW-1) fails it by far more than rounding."""
    H, W = 7, 9
    p = params([[3.3, 2.6]], [[4.0, 0.7, 3.0]], [[0.4]], order=1)
    p.expert[0, 0, 1:] = [0.031, -0.017]         # Wx, Wy
    y1, _ = O.render(p, H, W, R2=INF)
    for k in (2, 3, 4):
        yk, Dk = O.render(p, H, W, k * H, k * W, R2=INF)
        assert (Dk > 0).all()
        down = yk.reshape(1, H, k, W, k).mean(axis=(2, 4))
        np.testing.assert_allclose(down, y1, rtol=0, atol=1e-13)
    # the same plane at a non-integer scale: every sample is the plane at
    # its mapped point, so the output is itself a plane whose values at the
    # two outermost samples are symmetric about the image centre
    y15, _ = O.render(p, H, W, 11, 14, R2=INF)
    row = y15[0, 5]
    np.testing.assert_allclose(row[0] + row[-1], 2 * row.mean(), atol=1e-13)


def test_sr_sampling_mirror_symmetry():
    """A model mirror-symmetric about the image's vertical centre line
    x = (W-1)/2 must render mirror-symmetric at any output size, integer or
    not, when samples are centred.  Checks the mapping itself with a
    nonlinear, truncated, anisotropic model (not only planes)."""
    H, W = 20, 26
    g = np.random.default_rng(5)
    K = 12
    mu = np.stack([g.uniform(2, 11, K), g.uniform(2, 18, K)], 1)
    ch = np.stack([g.uniform(1.5, 3.5, K), g.uniform(-1.0, 1.0, K), g.uniform(1.5, 3.5, K)], 1)
    m = g.uniform(0.1, 0.9, (K, 2))
    mir_mu = np.stack([(W - 1) - mu[:, 0], mu[:, 1]], 1)
    mir_ch = ch * np.array([1.0, -1.0, 1.0])     # Sigma_xy -> -Sigma_xy under x -> -x
    p = params(np.concatenate([mu, mir_mu]), np.concatenate([ch, mir_ch]), np.concatenate([m, m]))
    for oH, oW in [(20, 26), (40, 52), (31, 37), (50, 61)]:
        y, _ = O.render(p, H, W, oH, oW)
        np.testing.assert_allclose(y, y[:, :, ::-1], rtol=0, atol=1e-12)


def test_point_margins_against_numpy():
    """O.point_margins (sampled-parity conditioning) equals the minimum over
    kernels of |delta^T Sigma^-1 delta - R2| computed with numpy's inverse of
    Sigma = L L^T; a point on a kernel's ellipse has margin 0 and a kernel
    centre alone gives R2."""
    g = np.random.default_rng(11)
    K = 25
    mu = g.uniform(0, 30, (K, 2))
    ch = np.stack([g.uniform(1, 4, K), g.uniform(-2, 2, K), g.uniform(1, 4, K)], 1)
    p = params(mu, ch, g.uniform(0, 1, K))
    xs, ys = g.uniform(-3, 33, 200), g.uniform(-3, 33, 200)
    R2 = O.R2_99()
    ref = np.full(200, np.inf)
    for k in range(K):
        L = np.array([[ch[k, 0], 0], [ch[k, 1], ch[k, 2]]])
        Si = np.linalg.inv(L @ L.T)
        d = np.stack([xs - mu[k, 0], ys - mu[k, 1]], 1)
        ref = np.minimum(ref, np.abs(np.einsum("ni,ij,nj->n", d, Si, d) - R2))
    np.testing.assert_allclose(O.point_margins(p, xs, ys), ref, rtol=1e-12, atol=1e-12)
    one = params([[5.0, 7.0]], [[2.0, 0.5, 1.5]], [0.3])
    L = np.array([[2.0, 0.0], [0.5, 1.5]])
    v = L @ np.array([np.cos(0.7), np.sin(0.7)]) * np.sqrt(R2)     # on the ellipse
    assert O.point_margins(one, [5.0 + v[0]], [7.0 + v[1]])[0] < 1e-12
    assert abs(O.point_margins(one, [5.0], [7.0])[0] - R2) < 1e-12


def test_operand_scale_bounds_term_scale():
    """B_ref (O.loss_grad grad_opnd, a tolerance scale) replaces every
    difference inside a per-pixel term by the sum of its operands'
    magnitudes, so it bounds A_ref (sum of |terms|) from above, and the two
    coincide for the expert terms of a model whose residuals cannot cancel
    (target 0, non-negative experts)."""
    H, W = 20, 24
    pool = synth.aniso_pool(H, W, 3, 30, 31, order=1, log_pi_sd=0.3)
    p = pool_params(pool)
    t = synth.image(H, W, 3, 32).astype(np.float64)
    lg = O.loss_grad(p, t)
    assert (lg.grad_opnd >= lg.grad_abs * (1 - 1e-12)).all()
    g, a, b = O.grad_kernels(p, t, np.arange(0, 30, 7), opnd=True)
    np.testing.assert_allclose(b, lg.grad_opnd[0:30:7], rtol=1e-12)
    q = p.copy()
    q.expert[:, :, 1:] = 0.0
    q.expert[:, :, 0] = np.abs(q.expert[:, :, 0])
    lz = O.loss_grad(q, np.zeros((3, H, W)))
    m = slice(6, None, 3)                         # m_c components: g eD_c, no inner difference
    np.testing.assert_allclose(lz.grad_opnd[:, m], lz.grad_abs[:, m], rtol=1e-12, atol=0)


def test_box_modes_closed_forms_nesting_and_coverage():
    """Box modes (reading Q4): the aabb half sides are the
    ellipse's extents R l11 and R sqrt(l21^2 + l22^2) (checked by sampling
    the ellipse boundary x = mu + R L (cos t, sin t)); the lists nest
    exact <= aabb <= square; square mode equals the boxes/tile_list route;
    and every (pixel, kernel) pair inside the ellipse is listed in every
    mode (coverage invariant), at 1x and at an SR raster."""
    H, W = 57, 70
    pool = synth.aniso_pool(H, W, 1, 60, 21, margin_px=6)
    p = pool_params(pool)
    R2 = O.R2_99()
    t = np.linspace(0, 2 * np.pi, 20001)
    for k in range(5):
        l11, l21, l22 = p.chol[k]
        L = np.array([[l11, 0.0], [l21, l22]])
        pts = np.sqrt(R2) * (L @ np.stack([np.cos(t), np.sin(t)]))
        assert abs(np.abs(pts[0]).max() - np.sqrt(R2) * l11) < 1e-6
        assert abs(np.abs(pts[1]).max() - np.sqrt(R2 * (l21 ** 2 + l22 ** 2))) < 1e-6
    for (oH, oW) in [(H, W), (2 * H, 2 * W), (40, 50)]:
        lists = {m: O.block_lists(p, H, W, oH, oW, mode=m) for m in ("square", "aabb", "exact")}
        pairs = {m: set(zip(np.repeat(np.arange(len(r) - 1), np.diff(r)).tolist(), ids.tolist()))
                 for m, (r, ids, _) in lists.items()}
        assert pairs["exact"] <= pairs["aabb"] <= pairs["square"]
        assert len(pairs["exact"]) < len(pairs["square"])
        _, tb, _ = O.boxes(p, H, W, oH, oW)
        r0, i0 = O.tile_list(tb, -(-oW // 16), -(-oH // 16))
        np.testing.assert_array_equal(lists["square"][0], r0)
        np.testing.assert_array_equal(lists["square"][1], i0)
        nx = -(-oW // 16)
        for i in range(oH):
            for j in range(oW):
                xs, ys = (j + 0.5) * W / oW - 0.5, (i + 0.5) * H / oH - 0.5
                tile = (i // 16) * nx + j // 16
                for k in range(p.K):
                    if O.d2(p.mu[k], p.chol[k], xs, ys) <= R2:
                        for m in pairs:
                            assert (tile, k) in pairs[m], (m, i, j, k)


def test_rect_min_d2_against_dense_sampling():
    """oracle_rect_min_d2 (exact box mode) equals the minimum of d^2 over a
    fine grid of the rectangle up to the grid's resolution, never exceeds
    it, and is 0 with the centre inside."""
    g = np.random.default_rng(4)
    for _ in range(40):
        mu = g.uniform(-5, 25, 2)
        ch = np.array([g.uniform(0.5, 4), g.uniform(-2, 2), g.uniform(0.5, 4)])
        x0, y0 = g.uniform(0, 10, 2)
        x1, y1 = x0 + g.uniform(0.5, 15), y0 + g.uniform(0.5, 15)
        v = O.rect_min_d2(mu, ch, x0, x1, y0, y1)
        xs, ys = np.meshgrid(np.linspace(x0, x1, 401), np.linspace(y0, y1, 401))
        L = np.array([[ch[0], 0], [ch[1], ch[2]]])
        Si = np.linalg.inv(L @ L.T)
        d = np.stack([xs - mu[0], ys - mu[1]], -1)
        dense = np.einsum("...i,ij,...j->...", d, Si, d).min()
        assert v <= dense + 1e-9
        assert dense - v <= 0.05 * max(1.0, dense)
        if x0 <= mu[0] <= x1 and y0 <= mu[1] <= y1:
            assert v == 0.0
