"""CPU oracle for the Rasterized SMoE hot path (arxiv 2510.05814).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_2510_05814_b200`` never imports it, and
it imports nothing from the product package.

The dense per-pixel arithmetic lives in ``smoe_oracle.c`` (plain C, fp64,
single-threaded, every pixel against every kernel).  This module adds the
pieces whose plain definition is a library primitive or a few lines of numpy:

* the canonical per-block kernel lists ``K_n`` (Eq. 5): every
  (block, kernel) pair whose square box contains a pixel centre
  of the block, sorted lexicographically (readings Q5, Q18);
* Adam ("optimized using Adam"; constants of reading Q9) with the
  per-group learning rates of P:426 and the Cholesky clamp of S:29;
* the exponential mu learning-rate decay 0.01 -> 1e-5;
* PSNR and the fit loop.

Parity status: every function here is pinned by ``tests/test_oracle.py``
(closed forms, SPEC worked examples, brute force, finite differences,
invariants) except ``fit`` whose 100-iteration trajectory has no paper value:
"parity unpinned" for the trajectory itself (its per-step pieces are pinned).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

TILE = 16  # 16x16 pixel blocks


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        src = os.path.join(_HERE, "smoe_oracle.c")
        if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
            subprocess.check_call(["make", "-s", "-C", _HERE])
        lib = ctypes.CDLL(path)
        D = ctypes.c_double
        I = ctypes.c_int
        P = ctypes.c_void_p
        lib.oracle_R2_99.restype = D
        lib.oracle_R2_99.argtypes = []
        lib.oracle_d2.restype = D
        lib.oracle_d2.argtypes = [P, P, D, D]
        lib.oracle_lambda_max.restype = D
        lib.oracle_lambda_max.argtypes = [P]
        lib.oracle_cov.restype = None
        lib.oracle_cov.argtypes = [P, P, P, P]
        lib.oracle_boxes.restype = None
        lib.oracle_boxes.argtypes = [I, P, P, D, I, I, I, I, P, P, P]
        lib.oracle_gates.restype = None
        lib.oracle_gates.argtypes = [I, P, P, P, D, D, D, P, P]
        lib.oracle_render.restype = None
        lib.oracle_render.argtypes = [I, I, I, P, P, P, P, I, I, I, I, I, I, D, P, P]
        lib.oracle_render_points.restype = None
        lib.oracle_render_points.argtypes = [I, I, I, P, P, P, P, I, P, P, D, P, P]
        lib.oracle_loss_grad.restype = None
        lib.oracle_loss_grad.argtypes = [I, I, I, P, P, P, P, I, I, P, I, I, D, P, P, P, P]
        lib.oracle_grad_kernels.restype = None
        lib.oracle_grad_kernels.argtypes = [I, I, I, P, P, P, P, I, I, P, D, I, P, P, P, P]
        lib.oracle_margins.restype = None
        lib.oracle_margins.argtypes = [I, P, P, D, I, I, I, I, P, P]
        lib.oracle_rect_min_d2.restype = D
        lib.oracle_rect_min_d2.argtypes = [P, P, D, D, D, D]
        lib.oracle_block_pairs.restype = ctypes.c_longlong
        lib.oracle_block_pairs.argtypes = [I, P, P, D, I, I, I, I, I, P, P, P, ctypes.c_longlong]
        lib.oracle_mode_margins.restype = None
        lib.oracle_mode_margins.argtypes = [I, P, P, D, I, I, I, I, I, P, P]
        lib.oracle_point_margins.restype = None
        lib.oracle_point_margins.argtypes = [I, P, P, D, I, P, P, P]
        lib.oracle_set_head.restype = None
        lib.oracle_set_head.argtypes = [I]
        _LIB = lib
    return _LIB


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class head:
    """Context manager selecting the regression head of the dense oracle:
    "smoe" (Eq. 2/4, default) or "rbf" (Eq. 1)."""

    def __init__(self, name: str):
        self.v = {"smoe": 0, "rbf": 1}[name]

    def __enter__(self):
        _lib().oracle_set_head(self.v)
        return self

    def __exit__(self, *a):
        _lib().oracle_set_head(0)


def sharpened(p: "Params", s: float) -> "Params":
    """Kernel editing for sharpening: Sigma -> s Sigma,
    i.e. every Cholesky factor times sqrt(s); centres, gates, experts kept."""
    q = p.copy()
    q.chol = q.chol * np.sqrt(s)
    return q


def R2_99() -> float:
    """chi^2_2 quantile at 0.99 = 2 ln 100 (reading Q1)."""
    return _lib().oracle_R2_99()


@dataclass
class Params:
    """Kernel parameters in fp64: mu[K,2], chol[K,3]=(l11,l21,l22), log_pi[K],
    expert[K,C,E] with E = 1 (constant) or 3 (linear: m, Wx, Wy)."""
    mu: np.ndarray
    chol: np.ndarray
    log_pi: np.ndarray
    expert: np.ndarray

    @property
    def K(self):
        return self.mu.shape[0]

    @property
    def C(self):
        return self.expert.shape[1]

    @property
    def order(self):
        return (self.expert.shape[2] - 1) // 2

    @property
    def Pk(self):
        return 6 + self.expert.shape[1] * self.expert.shape[2]

    def copy(self):
        return Params(self.mu.copy(), self.chol.copy(), self.log_pi.copy(), self.expert.copy())

    @staticmethod
    def from_any(p) -> "Params":
        """Accept any object with mu/chol/log_pi/expert attributes (or a dict)."""
        get = (lambda k: p[k]) if isinstance(p, dict) else (lambda k: getattr(p, k))
        conv = lambda a: _f64(a.cpu().numpy() if hasattr(a, "cpu") else a)
        return Params(conv(get("mu")).reshape(-1, 2), conv(get("chol")).reshape(-1, 3),
                      conv(get("log_pi")).reshape(-1), conv(get("expert")))

    def flat(self) -> np.ndarray:
        """[K][Pk] in the gradient layout (mu, l11, l21, l22, log_pi, expert)."""
        K = self.K
        return np.concatenate([self.mu, self.chol, self.log_pi[:, None],
                               self.expert.reshape(K, -1)], axis=1)

    @staticmethod
    def unflat(v: np.ndarray, C: int, order: int) -> "Params":
        K = v.shape[0]
        E = 1 + 2 * order
        return Params(v[:, 0:2].copy(), v[:, 2:5].copy(), v[:, 5].copy(),
                      v[:, 6:].reshape(K, C, E).copy())


def _args(p: Params):
    mu, ch, lp, ex = _f64(p.mu), _f64(p.chol), _f64(p.log_pi), _f64(p.expert)
    return (mu, ch, lp, ex)


def d2(mu, chol, px, py) -> float:
    """(x-mu)^T Sigma^-1 (x-mu), Sigma = L L^T (Eq. 3 exponent)."""
    return _lib().oracle_d2(_ptr(_f64(mu)), _ptr(_f64(chol)), float(px), float(py))


def cov(chol):
    out = [ctypes.c_double() for _ in range(3)]
    _lib().oracle_cov(_ptr(_f64(chol)), *[ctypes.byref(o) for o in out])
    return np.array([[out[0].value, out[1].value], [out[1].value, out[2].value]])


def lambda_max(chol) -> float:
    return _lib().oracle_lambda_max(_ptr(_f64(chol)))


def boxes(p: Params, H, W, out_H=None, out_W=None, R2=None):
    """Square 99% boxes mapped to the out_H x out_W raster.
    Returns pixbox[K,4]=(x_lo,x_hi,y_lo,y_hi), tilebox[K,4]=(tx0,tx1,ty0,ty1)
    (-1 rows when the box misses the image) and the half side r[K]."""
    out_H = H if out_H is None else out_H
    out_W = W if out_W is None else out_W
    R2 = R2_99() if R2 is None else R2
    K = p.K
    pb = np.zeros((K, 4), np.int32)
    tb = np.zeros((K, 4), np.int32)
    hs = np.zeros(K)
    mu, ch, _, _ = _args(p)
    _lib().oracle_boxes(K, _ptr(mu), _ptr(ch), R2, H, W, out_H, out_W, _ptr(pb), _ptr(tb), _ptr(hs))
    return pb, tb, hs


def tile_list(tilebox: np.ndarray, nx: int, ny: int, ty_range=None):
    """Per-block subsets K_n (Eq. 5) as the canonical sorted list.

    Every block b_n = (tx, ty) inside a kernel's tile box is recorded as
    affected by it; the pairs (n = ty*nx + tx, k) are sorted
    lexicographically (np.lexsort is the library sort step).  ty_range limits
    the blocks to rows [ty0, ty1) (a multi-GPU band).  Returns
    (tile_range[nx*ny+1], ids[P])."""
    ty0, ty1 = (0, ny) if ty_range is None else ty_range
    tiles, kers = [], []
    for k in range(tilebox.shape[0]):
        tx0, tx1, by0, by1 = (int(v) for v in tilebox[k])
        if tx0 < 0:
            continue
        by0, by1 = max(by0, ty0), min(by1, ty1 - 1)
        for ty in range(by0, by1 + 1):
            for tx in range(tx0, tx1 + 1):
                tiles.append(ty * nx + tx)
                kers.append(k)
    tiles = np.asarray(tiles, np.int64)
    kers = np.asarray(kers, np.int64)
    order = np.lexsort((kers, tiles))
    tiles, kers = tiles[order], kers[order]
    counts = np.bincount(tiles, minlength=nx * ny) if tiles.size else np.zeros(nx * ny, np.int64)
    rng = np.zeros(nx * ny + 1, np.int64)
    rng[1:] = np.cumsum(counts)
    return rng, kers


BOX_MODES = {"square": 0, "aabb": 1, "exact": 2}


def rect_min_d2(mu, chol, x0, x1, y0, y1) -> float:
    """min of (x-mu)^T Sigma^-1 (x-mu) over the rectangle [x0,x1] x [y0,y1]."""
    return _lib().oracle_rect_min_d2(_ptr(_f64(mu)), _ptr(_f64(chol)), float(x0), float(x1), float(y0), float(y1))


def block_lists(p: Params, H, W, out_H=None, out_W=None, mode="square", R2=None):
    """Canonical per-block lists K_n under a box mode (reading Q4): returns
    (tile_range[n_tiles+1], ids[P], tilebox[K,4]).  Mode "square" equals
    tile_list(boxes(...)); "aabb" uses the ellipse's axis-aligned box;
    "exact" keeps the aabb blocks whose pixel-centre rectangle meets the
    ellipse (smoe_oracle.c oracle_block_pairs)."""
    out_H = H if out_H is None else out_H
    out_W = W if out_W is None else out_W
    R2 = R2_99() if R2 is None else R2
    mu, ch, _, _ = _args(p)
    tb = np.zeros((p.K, 4), np.int32)
    m = BOX_MODES[mode]
    n = _lib().oracle_block_pairs(p.K, _ptr(mu), _ptr(ch), R2, H, W, out_H, out_W, m, _ptr(tb), None, None, 0)
    tiles = np.zeros(max(n, 1), np.int32)
    kers = np.zeros(max(n, 1), np.int32)
    _lib().oracle_block_pairs(p.K, _ptr(mu), _ptr(ch), R2, H, W, out_H, out_W, m, _ptr(tb), _ptr(tiles),
                              _ptr(kers), n)
    tiles, kers = tiles[:n].astype(np.int64), kers[:n].astype(np.int64)
    order = np.lexsort((kers, tiles))        # library sort step (Q18 tie order)
    tiles, kers = tiles[order], kers[order]
    nx, ny = -(-out_W // 16), -(-out_H // 16)
    rng = np.zeros(nx * ny + 1, np.int64)
    rng[1:] = np.cumsum(np.bincount(tiles, minlength=nx * ny))
    return rng, kers, tb


def mode_margins(p: Params, H, W, out_H=None, out_W=None, mode="square", R2=None):
    """Per kernel: box-edge distance to an integer under the mode, and (mode
    exact) the smallest |rect_min_d2 - R2| over its candidate blocks."""
    out_H = H if out_H is None else out_H
    out_W = W if out_W is None else out_W
    R2 = R2_99() if R2 is None else R2
    mu, ch, _, _ = _args(p)
    eg = np.zeros(p.K)
    rg = np.zeros(p.K)
    _lib().oracle_mode_margins(p.K, _ptr(mu), _ptr(ch), R2, H, W, out_H, out_W, BOX_MODES[mode], _ptr(eg), _ptr(rg))
    return eg, rg


def gates(p: Params, px, py, R2=None):
    """Gates w_j(x) of Eq. (4) normalised over the truncated set, and D."""
    R2 = R2_99() if R2 is None else R2
    mu, ch, lp, _ = _args(p)
    w = np.zeros(p.K)
    D = ctypes.c_double()
    _lib().oracle_gates(p.K, _ptr(mu), _ptr(ch), _ptr(lp), float(px), float(py), R2, _ptr(w), ctypes.byref(D))
    return w, D.value


def render(p: Params, H, W, out_H=None, out_W=None, rows=None, R2=None):
    """Dense render y[C][rows][out_W] (Eq. 2/5 with truncation) and D."""
    out_H = H if out_H is None else out_H
    out_W = W if out_W is None else out_W
    r0, r1 = (0, out_H) if rows is None else rows
    R2 = R2_99() if R2 is None else R2
    mu, ch, lp, ex = _args(p)
    y = np.zeros((p.C, r1 - r0, out_W))
    D = np.zeros((r1 - r0, out_W))
    _lib().oracle_render(p.K, p.C, p.order, _ptr(mu), _ptr(ch), _ptr(lp), _ptr(ex),
                         H, W, out_H, out_W, r0, r1, R2, _ptr(y), _ptr(D))
    return y, D


def render_points(p: Params, xs, ys, R2=None):
    """y at arbitrary source-space points: returns y[n,C], D[n]."""
    R2 = R2_99() if R2 is None else R2
    xs, ys = _f64(xs), _f64(ys)
    n = xs.size
    mu, ch, lp, ex = _args(p)
    y = np.zeros((n, p.C))
    D = np.zeros(n)
    _lib().oracle_render_points(p.K, p.C, p.order, _ptr(mu), _ptr(ch), _ptr(lp), _ptr(ex),
                                n, _ptr(xs), _ptr(ys), R2, _ptr(y), _ptr(D))
    return y, D


@dataclass
class LossGrad:
    grad: np.ndarray       # [K, Pk]
    grad_abs: np.ndarray   # [K, Pk]  sum over pixels of |per-pixel term| (A_ref)
    grad_opnd: np.ndarray  # [K, Pk]  operand scale B_ref (test tolerance only, see smoe_oracle.c)
    sse: float
    sse_clamped: float
    uncovered: int
    n: int                 # H*W*C

    @property
    def loss(self):
        return self.sse / self.n

    @property
    def psnr(self):
        return psnr_from_mse(self.sse_clamped / self.n)


def loss_grad(p: Params, target, rows=None, R2=None) -> LossGrad:
    """MSE loss (reading Q8), PSNR sums and the analytic gradient (rows r0..r1)."""
    t = _f64(target)
    C, H, W = t.shape
    assert C == p.C
    r0, r1 = (0, H) if rows is None else rows
    R2 = R2_99() if R2 is None else R2
    mu, ch, lp, ex = _args(p)
    g = np.zeros((p.K, p.Pk))
    a = np.zeros((p.K, p.Pk))
    b = np.zeros((p.K, p.Pk))
    st = np.zeros(3)
    _lib().oracle_loss_grad(p.K, p.C, p.order, _ptr(mu), _ptr(ch), _ptr(lp), _ptr(ex),
                            H, W, _ptr(t), r0, r1, R2, _ptr(g), _ptr(a), _ptr(b), _ptr(st))
    return LossGrad(g, a, b, st[0], st[1], int(st[2]), C * H * W)


def grad_kernels(p: Params, target, sel, R2=None, opnd=False):
    """Full-image gradient rows for the kernels in ``sel`` only: (grad,
    A_ref) or, with ``opnd``, (grad, A_ref, B_ref)."""
    t = _f64(target)
    C, H, W = t.shape
    R2 = R2_99() if R2 is None else R2
    sel = np.ascontiguousarray(sel, np.int32)
    mu, ch, lp, ex = _args(p)
    g = np.zeros((sel.size, p.Pk))
    a = np.zeros((sel.size, p.Pk))
    b = np.zeros((sel.size, p.Pk))
    _lib().oracle_grad_kernels(p.K, p.C, p.order, _ptr(mu), _ptr(ch), _ptr(lp), _ptr(ex),
                               H, W, _ptr(t), R2, sel.size, _ptr(sel), _ptr(g), _ptr(a), _ptr(b))
    return (g, a, b) if opnd else (g, a)


def margins(p: Params, H, W, out_H=None, out_W=None, R2=None):
    """Per kernel: min |d^2 - R2| near its box, min box-edge distance to Z."""
    out_H = H if out_H is None else out_H
    out_W = W if out_W is None else out_W
    R2 = R2_99() if R2 is None else R2
    mu, ch, _, _ = _args(p)
    dg = np.zeros(p.K)
    eg = np.zeros(p.K)
    _lib().oracle_margins(p.K, _ptr(mu), _ptr(ch), R2, H, W, out_H, out_W, _ptr(dg), _ptr(eg))
    return dg, eg


def point_margins(p: Params, xs, ys, R2=None):
    """Per source-space point: min over every kernel of |d^2 - R2| (dense);
    used to keep sampled parity away from the cull discontinuity."""
    R2 = R2_99() if R2 is None else R2
    xs, ys = _f64(xs).ravel(), _f64(ys).ravel()
    mu, ch, _, _ = _args(p)
    gap = np.zeros(xs.size)
    _lib().oracle_point_margins(p.K, _ptr(mu), _ptr(ch), R2, xs.size, _ptr(xs), _ptr(ys), _ptr(gap))
    return gap


# ---------------------------------------------------------------- metrics ---

def psnr_from_mse(mse: float) -> float:
    """PSNR = 10 log10(1/MSE) for [0,1] images."""
    if mse <= 0.0:
        return float("inf")
    return 10.0 * np.log10(1.0 / mse)


# ------------------------------------------------------------- optimiser ---

BETA1, BETA2, EPS = 0.9, 0.999, 1e-8   # reading Q9
CHOL_MIN = 1e-3                         # S:29 clamp


def lr_mu_schedule(t0: int, T: int, lr0: float = 0.01, lr_end: float = 1e-5) -> float:
    """mu learning rate decaying exponentially 0.01 -> 1e-5:
    lr(t0) = lr0 * (lr_end/lr0)^(t0/T), t0 the 0-based step."""
    return lr0 * (lr_end / lr0) ** (t0 / T)


@dataclass
class LR:
    """Per-group learning rates: mu 0.01 (scheduled), Sigma 1e-3,
    m 1e-3; log_pi frozen (reading Q11); linear slopes 2e-4 (reading Q13)."""
    mu: float = 0.01
    chol: float = 1e-3
    log_pi: float = 0.0
    expert: float = 1e-3
    slope: float = 2e-4

    def vector(self, C: int, order: int) -> np.ndarray:
        E = 1 + 2 * order
        ex = np.tile(np.array([self.expert] + [self.slope] * (E - 1)), C)
        return np.concatenate([[self.mu] * 2, [self.chol] * 3, [self.log_pi], ex])


class Adam:
    """Bias-corrected Adam (Kingma & Ba), eps outside the sqrt, state
    per scalar parameter, 1-based step t; then l11, l22 >= 1e-3."""

    def __init__(self, K: int, Pk: int):
        self.m1 = np.zeros((K, Pk))
        self.m2 = np.zeros((K, Pk))
        self.t = 0

    def step(self, p: Params, grad: np.ndarray, lr: LR) -> Params:
        self.t += 1
        t = self.t
        self.m1 = BETA1 * self.m1 + (1.0 - BETA1) * grad
        self.m2 = BETA2 * self.m2 + (1.0 - BETA2) * grad * grad
        mhat = self.m1 / (1.0 - BETA1 ** t)
        vhat = self.m2 / (1.0 - BETA2 ** t)
        lrv = lr.vector(p.C, p.order)[None, :]
        v = p.flat() - lrv * mhat / (np.sqrt(vhat) + EPS)
        v[:, 2] = np.maximum(v[:, 2], CHOL_MIN)   # l11
        v[:, 4] = np.maximum(v[:, 4], CHOL_MIN)   # l22
        return Params.unflat(v, p.C, p.order)


def fit(p: Params, target, T: int, lr: LR | None = None, schedule_T: int | None = None,
        round_fp32: bool = False, R2=None):
    """T iterations of {loss+gradient, Adam}.  Returns (params, trace)
    with trace[i] = (loss, psnr) of iteration i measured BEFORE its update.
    ``round_fp32`` rounds parameters to fp32 after each update (an optional
    mode for comparison with fp32 state).  Parity unpinned: the paper prints
    no trajectory; each step's pieces are pinned individually."""
    lr = LR() if lr is None else lr
    schedule_T = T if schedule_T is None else schedule_T
    opt = Adam(p.K, p.Pk)
    trace = []
    p = p.copy()
    for t0 in range(T):
        lg = loss_grad(p, target, R2=R2)
        trace.append((lg.loss, lg.psnr))
        lr_t = LR(lr_mu_schedule(t0, schedule_T, lr.mu), lr.chol, lr.log_pi, lr.expert, lr.slope)
        p = opt.step(p, lg.grad, lr_t)
        if round_fp32:
            p = Params.unflat(p.flat().astype(np.float32).astype(np.float64), p.C, p.order)
    return p, trace
