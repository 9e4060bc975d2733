"""Thin Python binding of the C-ABI library ``libsmoe.so`` (include/smoe.h).

Argument marshalling only: every step of the hot path runs in the CUDA
kernels behind the ABI.  PyTorch provides device memory and streams.  There
is no fallback: if ``libsmoe.so`` is missing or no CUDA device is present the
calls fail loudly.

The function names mirror the C entry points (``smoe_create``, ``smoe_step``,
``smoe_render``, ...); :class:`SMoE` wraps a handle with the same methods.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SMOE_LIB") or os.path.join(_HERE, "libsmoe.so")   # SMOE_LIB: A/B builds
_LIB = None

OK, ERR_INVALID_ARG, ERR_CUDA, ERR_OUT_OF_MEMORY, ERR_NONFINITE, ERR_CAPACITY, ERR_BAD_HANDLE = range(7)


class SmoeError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


class c_params(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_void_p), ("chol", ctypes.c_void_p),
                ("log_pi", ctypes.c_void_p), ("expert", ctypes.c_void_p)]


class c_lr(ctypes.Structure):
    _fields_ = [("mu", ctypes.c_float), ("chol", ctypes.c_float), ("log_pi", ctypes.c_float),
                ("expert", ctypes.c_float), ("slope", ctypes.c_float)]


class c_stats(ctypes.Structure):
    _fields_ = [("loss", ctypes.c_double), ("psnr_db", ctypes.c_double), ("sse", ctypes.c_double),
                ("sse_clamped", ctypes.c_double), ("pairs", ctypes.c_longlong),
                ("uncovered_px", ctypes.c_longlong), ("n_tiles", ctypes.c_longlong)]


class c_kernel_time(ctypes.Structure):
    _fields_ = [("total_ms", ctypes.c_double), ("launches", ctypes.c_longlong)]


class c_work(ctypes.Structure):
    _fields_ = [("tested_pairs", ctypes.c_longlong), ("hit_pairs", ctypes.c_longlong),
                ("sort_cycles", ctypes.c_longlong), ("cta_cycles", ctypes.c_longlong)]


KERNEL_COUNT = 8


class c_raw_stats(ctypes.Structure):
    _fields_ = [("sse", ctypes.c_double), ("sse_clamped", ctypes.c_double), ("uncovered", ctypes.c_double),
                ("pairs", ctypes.c_longlong)]


class c_options(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int), ("H", ctypes.c_int), ("W", ctypes.c_int), ("C", ctypes.c_int),
                ("expert_order", ctypes.c_int), ("R2", ctypes.c_double), ("device", ctypes.c_int),
                ("pair_capacity", ctypes.c_longlong), ("backward_mode", ctypes.c_int),
                ("use_graphs", ctypes.c_int), ("head", ctypes.c_int), ("box_mode", ctypes.c_int)]


class c_render_options(ctypes.Structure):
    _fields_ = [("sharpen", ctypes.c_float), ("accumulate", ctypes.c_float), ("vector_stores", ctypes.c_int)]


def lib():
    """Load libsmoe.so (fails loudly when the extension was not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build the CUDA extension (python -c "
                          "'import __graft_entry__ as g; g.build()')")
    L = ctypes.CDLL(LIB_PATH)
    H = ctypes.c_void_p
    P = ctypes.c_void_p
    I = ctypes.c_int
    st = ctypes.c_int
    sig = {
        "smoe_default_options": (st, [ctypes.POINTER(c_options)]),
        "smoe_create": (st, [I, I, I, I, I, ctypes.POINTER(H)]),
        "smoe_create_ex": (st, [ctypes.POINTER(c_options), ctypes.POINTER(H)]),
        "smoe_destroy": (st, [H]),
        "smoe_set_stream": (st, [H, P]),
        "smoe_render": (st, [H, ctypes.POINTER(c_params), I, I, P]),
        "smoe_render_ex": (st, [H, ctypes.POINTER(c_params), I, I, P, ctypes.POINTER(c_render_options)]),
        "smoe_step": (st, [H, ctypes.POINTER(c_params), P, ctypes.POINTER(c_lr), ctypes.POINTER(c_stats)]),
        "smoe_set_band": (st, [H, I, I]),
        "smoe_invalidate": (st, [H]),
        "smoe_grad": (st, [H, ctypes.POINTER(c_params), P, P, P]),
        "smoe_apply": (st, [H, ctypes.POINTER(c_params), P, ctypes.POINTER(c_lr)]),
        "smoe_apply_ex": (st, [H, ctypes.POINTER(c_params), P, ctypes.POINTER(c_lr), I, I, P]),
        "smoe_reset_adam": (st, [H]),
        "smoe_sync": (st, [H, ctypes.POINTER(c_stats)]),
        "smoe_bin": (st, [H, ctypes.POINTER(c_params), I, I, P, P, ctypes.c_longlong,
                          ctypes.POINTER(ctypes.c_longlong), P]),
        "smoe_paper_lr": (c_lr, [I, I]),
        "smoe_launch_count": (ctypes.c_longlong, [H]),
        "smoe_profile_begin": (st, [H, I, ctypes.c_uint]),
        "smoe_profile_end": (st, [H, P, ctypes.POINTER(c_work)]),
        "smoe_kernel_name": (ctypes.c_char_p, [I]),
        "smoe_status_string": (ctypes.c_char_p, [st]),
        "smoe_last_error": (ctypes.c_char_p, [H]),
        "smoe_abi_version": (I, []),
        "smoe_stats_async": (st, [H, P]),
        "smoe_get_adam": (st, [H, P, P, ctypes.POINTER(ctypes.c_longlong)]),
        "smoe_set_adam": (st, [H, P, P, ctypes.c_longlong]),
        "smoe_stats_from_raw": (st, [H, P, ctypes.POINTER(c_stats)]),
        "smoe_segment": (st, [P, I, I, I, ctypes.c_float, I, P, ctypes.POINTER(I)]),
        "smoe_segment_init": (st, [P, I, I, I, P, I, I, I, ctypes.c_ulonglong, ctypes.c_float, P, P, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _LIB = L
    return L


def _check(status: int, handle=None):
    if status != OK:
        msg = lib().smoe_last_error(handle).decode(errors="replace")
        raise SmoeError(status, msg or lib().smoe_status_string(status).decode())


@dataclass
class Params:
    """Kernel parameters as float32 CUDA tensors in the ABI layout:
    mu[K,2], chol[K,3] = (l11, l21, l22), log_pi[K], expert[K,C,E]."""
    mu: torch.Tensor
    chol: torch.Tensor
    log_pi: torch.Tensor
    expert: torch.Tensor

    @staticmethod
    def from_numpy(pool, device="cuda") -> "Params":
        t = lambda a: torch.as_tensor(a, dtype=torch.float32).contiguous().to(device)
        return Params(t(pool.mu), t(pool.chol), t(pool.log_pi), t(pool.expert))

    def clone(self) -> "Params":
        return Params(self.mu.clone(), self.chol.clone(), self.log_pi.clone(), self.expert.clone())

    def flat(self) -> torch.Tensor:
        K = self.mu.shape[0]
        return torch.cat([self.mu, self.chol, self.log_pi[:, None], self.expert.reshape(K, -1)], 1)

    def c(self, K: int | None = None, C: int | None = None, E: int | None = None,
          device: int | None = None) -> c_params:
        for t in (self.mu, self.chol, self.log_pi, self.expert):
            if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()):
                raise SmoeError(ERR_INVALID_ARG, "params must be contiguous float32 CUDA tensors")
            if device is not None and t.device.index != device:
                raise SmoeError(ERR_INVALID_ARG, f"params on {t.device}, the handle is on cuda:{device}")
        if K is not None:
            want = {"mu": 2 * K, "chol": 3 * K, "log_pi": K, "expert": K * C * E}
            for name, n in want.items():
                if getattr(self, name).numel() < n:
                    raise SmoeError(ERR_INVALID_ARG, f"params.{name}: {getattr(self, name).numel()} "
                                                     f"elements, expected {n}")
        return c_params(self.mu.data_ptr(), self.chol.data_ptr(), self.log_pi.data_ptr(),
                        self.expert.data_ptr())


@dataclass
class LR:
    """Per-group learning rates of one step (readings Q11, Q13)."""
    mu: float = 0.01
    chol: float = 1e-3
    log_pi: float = 0.0
    expert: float = 1e-3
    slope: float = 2e-4

    def c(self) -> c_lr:
        return c_lr(self.mu, self.chol, self.log_pi, self.expert, self.slope)

    @staticmethod
    def paper(t: int, T: int) -> "LR":
        l = lib().smoe_paper_lr(int(t), int(T))
        return LR(l.mu, l.chol, l.log_pi, l.expert, l.slope)


@dataclass
class Stats:
    loss: float
    psnr_db: float
    sse: float
    sse_clamped: float
    pairs: int
    uncovered_px: int
    n_tiles: int

    @staticmethod
    def of(s: c_stats) -> "Stats":
        return Stats(s.loss, s.psnr_db, s.sse, s.sse_clamped, s.pairs, s.uncovered_px, s.n_tiles)


def _ptr(x, what="buffer", dtype=torch.float32, numel=None, device=None):
    """Raw address of a contiguous torch tensor or numpy array (host or
    device) after checking what the library will read through it: dtype,
    element count (at least ``numel``) and, for CUDA tensors, the handle's
    device.  A mismatch raises ERR_INVALID_ARG instead of letting the library
    read the wrong bytes or copy past the end of a host buffer."""
    if x is None:
        return None
    if isinstance(x, torch.Tensor):
        if not x.is_contiguous():
            raise SmoeError(ERR_INVALID_ARG, f"{what}: must be contiguous")
        if x.dtype != dtype:
            raise SmoeError(ERR_INVALID_ARG, f"{what}: dtype {x.dtype}, expected {dtype}")
        if numel is not None and x.numel() < numel:
            raise SmoeError(ERR_INVALID_ARG, f"{what}: {x.numel()} elements, expected {numel}")
        if x.is_cuda and device is not None and x.device.index != device:
            raise SmoeError(ERR_INVALID_ARG, f"{what}: on {x.device}, the handle is on cuda:{device}")
        return x.data_ptr()
    if hasattr(x, "ctypes") and hasattr(x, "flags"):
        import numpy as np
        if not x.flags["C_CONTIGUOUS"]:
            raise SmoeError(ERR_INVALID_ARG, f"{what}: must be contiguous")
        want = np.float32 if dtype == torch.float32 else np.float64
        if x.dtype != want:
            raise SmoeError(ERR_INVALID_ARG, f"{what}: dtype {x.dtype}, expected {np.dtype(want)}")
        if numel is not None and x.size < numel:
            raise SmoeError(ERR_INVALID_ARG, f"{what}: {x.size} elements, expected {numel}")
        return x.ctypes.data
    raise SmoeError(ERR_INVALID_ARG, f"{what}: expected a torch tensor or numpy array")


class SMoE:
    """A library handle: K kernels fitting an H x W x C image with constant
    (order 0) or linear (order 1) experts (B.json smoe_create)."""

    def __init__(self, K: int, H: int, W: int, C: int, expert_order: int = 0, R2: float | None = None,
                 device: int | None = None, pair_capacity: int = 0, backward_mode: int = -1,
                 use_graphs: bool = True, head: str = "smoe", box_mode: str | None = None):
        L = lib()
        o = c_options()
        _check(L.smoe_default_options(ctypes.byref(o)))
        o.K, o.H, o.W, o.C, o.expert_order = K, H, W, C, expert_order
        if R2 is not None:
            o.R2 = R2
        o.device = torch.cuda.current_device() if device is None else device
        o.pair_capacity = pair_capacity
        o.backward_mode = backward_mode
        o.use_graphs = int(bool(use_graphs))
        o.head = {"smoe": 0, "rbf": 1}[head]
        if box_mode is not None:      # None: the library default (aabb)
            o.box_mode = {"square": 0, "aabb": 1, "exact": 2}[box_mode]
        h = ctypes.c_void_p()
        _check(L.smoe_create_ex(ctypes.byref(o), ctypes.byref(h)))
        self.h = h
        self.K, self.H, self.W, self.C, self.order = K, H, W, C, expert_order
        self.E = 1 + 2 * expert_order
        self.Pk = 6 + C * self.E
        self.device = o.device

    def close(self):
        if getattr(self, "h", None):
            lib().smoe_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _stream(self):
        s = torch.cuda.current_stream(self.device).cuda_stream
        _check(lib().smoe_set_stream(self.h, ctypes.c_void_p(s)), self.h)

    def _p(self, params: Params) -> c_params:
        return params.c(self.K, self.C, self.E, self.device)

    def _fresh(self, params: Params):
        """Fused records (smoe_invalidate): tell the library when the caller
        wrote the parameter tensors since the last step (their version
        counters moved; the library's own writes do not move them)."""
        key = tuple((t.data_ptr(), t._version) for t in (params.mu, params.chol, params.log_pi, params.expert))
        if key != getattr(self, "_pkey", None):
            _check(lib().smoe_invalidate(self.h), self.h)
        self._pkey = key

    def _target(self, target):
        return _ptr(target, "target", torch.float32, self.C * self.H * self.W, self.device)

    def step(self, params: Params, target, lr: LR | None = None, stats: bool = True):
        """smoe_step: one fit iteration in place on ``params``; returns the
        pre-update Stats when ``stats`` (synchronising), else None."""
        self._stream()
        lr = lr or LR()
        p = self._p(params)
        t = self._target(target)
        self._fresh(params)
        if stats:
            s = c_stats()
            _check(lib().smoe_step(self.h, ctypes.byref(p), t, ctypes.byref(lr.c()), ctypes.byref(s)), self.h)
            return Stats.of(s)
        _check(lib().smoe_step(self.h, ctypes.byref(p), t, ctypes.byref(lr.c()), None), self.h)
        return None

    def render(self, params: Params, out_H: int | None = None, out_W: int | None = None, out=None,
               sharpen: float = 1.0, accumulate: float = 0.0, vector_stores: bool = False):
        """smoe_render(_ex): y on an out_H x out_W raster -> [C, out_H, out_W];
        ``sharpen`` = s < 1 renders with Sigma -> s Sigma (kernel editing);
        ``accumulate`` = w != 0 adds w y into ``out`` (multi-model fusion)."""
        self._stream()
        out_H = self.H if out_H is None else out_H
        out_W = self.W if out_W is None else out_W
        own = out is None
        if own:
            out = torch.empty((self.C, out_H, out_W), dtype=torch.float32, device=f"cuda:{self.device}")
        ro = c_render_options(sharpen, accumulate, int(bool(vector_stores)))
        args = (self.h, ctypes.byref(self._p(params)), out_H, out_W,
                _ptr(out, "out", torch.float32, self.C * out_H * out_W, self.device), ctypes.byref(ro))
        _check(lib().smoe_render_ex(*args), self.h)
        if own:
            # the output is ours: make sure the render was not skipped by a
            # list overflow (the library grows its lists and we render again)
            for attempt in range(3):
                try:
                    self.sync()
                    break
                except SmoeError as e:
                    if e.status != ERR_CAPACITY or attempt == 2:
                        raise
                    _check(lib().smoe_render_ex(*args), self.h)
        return out

    def invalidate(self):
        """smoe_invalidate: the caller wrote the parameter buffers outside the
        tensors' version counters (e.g. through ``.data`` or raw pointers);
        the next step re-derives the kernel records."""
        _check(lib().smoe_invalidate(self.h), self.h)

    def set_band(self, tile_row0: int, tile_row1: int):
        _check(lib().smoe_set_band(self.h, tile_row0, tile_row1), self.h)

    def grad(self, params: Params, target, grad=None, sums=None):
        """smoe_grad: (grad[K,Pk], sums[3] = SSE, clamped SSE, uncovered)."""
        self._stream()
        dev = f"cuda:{self.device}"
        if grad is None:
            grad = torch.empty((self.K, self.Pk), dtype=torch.float32, device=dev)
        if sums is None:
            sums = torch.empty(4, dtype=torch.float64, device=dev)
        self._fresh(params)
        _check(lib().smoe_grad(self.h, ctypes.byref(self._p(params)), self._target(target),
                               _ptr(grad, "grad", torch.float32, self.K * self.Pk, self.device),
                               _ptr(sums, "sums", torch.float64, 4, self.device)), self.h)
        return grad, sums

    def apply(self, params: Params, grad, lr: LR | None = None, k0: int = 0, k1: int | None = None,
              sums=None):
        """smoe_apply / smoe_apply_ex: Adam update of kernels [k0, k1) with
        grad[(k1-k0), Pk]; ``sums`` (the all-reduced smoe_grad sums[4]) makes
        the update conditional on no rank having skipped its band."""
        self._stream()
        k1 = self.K if k1 is None else k1
        _check(lib().smoe_apply_ex(self.h, ctypes.byref(self._p(params)),
                                   _ptr(grad, "grad", torch.float32, (k1 - k0) * self.Pk, self.device),
                                   ctypes.byref((lr or LR()).c()), int(k0), int(k1),
                                   _ptr(sums, "sums", torch.float64, 4, self.device)), self.h)

    def reset_adam(self):
        _check(lib().smoe_reset_adam(self.h), self.h)

    def get_adam(self):
        """smoe_get_adam -> (m1[K,Pk], m2[K,Pk], t): optimiser checkpoint."""
        m1 = torch.empty((self.K, self.Pk), dtype=torch.float32)
        m2 = torch.empty((self.K, self.Pk), dtype=torch.float32)
        t = ctypes.c_longlong()
        _check(lib().smoe_get_adam(self.h, m1.data_ptr(), m2.data_ptr(), ctypes.byref(t)), self.h)
        return m1, m2, t.value

    def set_adam(self, m1, m2, t: int):
        """smoe_set_adam: restore an optimiser checkpoint."""
        m1 = m1.contiguous().float()
        m2 = m2.contiguous().float()
        n = self.K * self.Pk
        _check(lib().smoe_set_adam(self.h, _ptr(m1, "m1", numel=n, device=self.device),
                                   _ptr(m2, "m2", numel=n, device=self.device), int(t)), self.h)

    def stats_async(self, dst_ptr: int):
        """smoe_stats_async: enqueue the D2H copy of the last step's raw
        statistics into host memory at dst_ptr (a c_raw_stats, ideally pinned)."""
        self._stream()
        _check(lib().smoe_stats_async(self.h, ctypes.c_void_p(dst_ptr)), self.h)

    def stats_from_raw(self, src_ptr: int) -> Stats:
        s = c_stats()
        _check(lib().smoe_stats_from_raw(self.h, ctypes.c_void_p(src_ptr), ctypes.byref(s)), self.h)
        return Stats.of(s)

    def sync(self) -> Stats:
        s = c_stats()
        _check(lib().smoe_sync(self.h, ctypes.byref(s)), self.h)
        return Stats.of(s)

    def bin(self, params: Params, out_H: int | None = None, out_W: int | None = None):
        """smoe_bin: (tile_range[n_tiles+1], ids[P], tilebox[K,4]) as int64 CPU tensors."""
        self._stream()
        out_H = self.H if out_H is None else out_H
        out_W = self.W if out_W is None else out_W
        nt = ((out_H + 15) // 16) * ((out_W + 15) // 16)
        rng = torch.empty(nt + 1, dtype=torch.int32)
        tb = torch.empty((self.K, 4), dtype=torch.int32)
        n = ctypes.c_longlong()
        _check(lib().smoe_bin(self.h, ctypes.byref(self._p(params)), out_H, out_W, rng.data_ptr(), None, 0,
                              ctypes.byref(n), tb.data_ptr()), self.h)
        ids = torch.empty(max(1, n.value), dtype=torch.int32)
        _check(lib().smoe_bin(self.h, ctypes.byref(self._p(params)), out_H, out_W, rng.data_ptr(), ids.data_ptr(),
                              ids.numel(), ctypes.byref(n), tb.data_ptr()), self.h)
        return rng.long(), ids[:n.value].long(), tb.long()

    def launch_count(self) -> int:
        return int(lib().smoe_launch_count(self.h))

    def profile_begin(self, max_launches: int, kernels=None, count_work: bool = False):
        """smoe_profile_begin: time the next launches of ``kernels`` (names,
        None = all) with CUDA event pairs on the handle's stream; with
        ``count_work`` the raster also counts tested / hit pairs."""
        mask = 0
        if kernels:
            names = [lib().smoe_kernel_name(i).decode() for i in range(KERNEL_COUNT)]
            for k in kernels:
                mask |= 1 << names.index(k)
        else:
            mask = (1 << KERNEL_COUNT) - 1
        if count_work:
            mask |= 0x80000000
        _check(lib().smoe_profile_begin(self.h, int(max_launches), mask), self.h)

    def profile_end(self):
        """smoe_profile_end -> ({kernel name: (total_ms, launches)}, (tested, hit)).
        ``self.last_work`` keeps the full counters (tested, hit, sort cycles,
        CTA cycles)."""
        arr = (c_kernel_time * KERNEL_COUNT)()
        w = c_work()
        _check(lib().smoe_profile_end(self.h, ctypes.cast(arr, ctypes.c_void_p), ctypes.byref(w)), self.h)
        out = {}
        for i in range(KERNEL_COUNT):
            if arr[i].launches:
                out[lib().smoe_kernel_name(i).decode()] = (arr[i].total_ms, arr[i].launches)
        self.last_work = (w.tested_pairs, w.hit_pairs, w.sort_cycles, w.cta_cycles)
        return out, (w.tested_pairs, w.hit_pairs)


# C-named module-level wrappers (the binding keeps the ABI's names).
def smoe_create(K, H, W, C, expert_order=0, **kw) -> SMoE:
    return SMoE(K, H, W, C, expert_order, **kw)


def smoe_step(h: SMoE, params, target, lr=None, stats=True):
    return h.step(params, target, lr, stats)


def smoe_render(h: SMoE, params, out_H=None, out_W=None, out=None):
    return h.render(params, out_H, out_W, out)


def smoe_grad(h: SMoE, params, target, grad=None, sums=None):
    return h.grad(params, target, grad, sums)


def smoe_apply(h: SMoE, params, grad, lr=None):
    return h.apply(params, grad, lr)


def smoe_set_band(h: SMoE, r0, r1):
    return h.set_band(r0, r1)


def smoe_sync(h: SMoE):
    return h.sync()


def smoe_bin(h: SMoE, params, out_H=None, out_W=None):
    return h.bin(params, out_H, out_W)


def smoe_destroy(h: SMoE):
    h.close()


def segment(image, threshold: float = 10.0, min_size: int = 16):
    """smoe_segment: region labels [H, W] (int32 numpy) and the segment count
    for a [C, H, W] float32 host image in [0, 1]."""
    import numpy as np
    img = np.ascontiguousarray(image, dtype=np.float32)
    C, H, W = img.shape
    labels = np.empty((H, W), np.int32)
    n = ctypes.c_int()
    _check(lib().smoe_segment(img.ctypes.data, H, W, C, float(threshold), int(min_size), labels.ctypes.data,
                              ctypes.byref(n)))
    return labels, n.value


def segment_init(image, labels, n_segments: int, K: int, order: int = 0, seed: int = 0, scale_px: float = 5.0):
    """smoe_segment_init: a kernel pool (numpy, smoe_params layout) spread
    over the segments by Eq. 9 with the experts at the segment colours."""
    import numpy as np
    from .synth import Pool
    img = np.ascontiguousarray(image, dtype=np.float32)
    C, H, W = img.shape
    E = 1 + 2 * order
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    mu = np.empty((K, 2), np.float32)
    chol = np.empty((K, 3), np.float32)
    lp = np.empty(K, np.float32)
    ex = np.empty((K, C, E), np.float32)
    _check(lib().smoe_segment_init(img.ctypes.data, H, W, C, lab.ctypes.data, int(n_segments), int(K), int(order),
                                   int(seed), float(scale_px), mu.ctypes.data, chol.ctypes.data, lp.ctypes.data,
                                   ex.ctypes.data))
    return Pool(mu, chol, lp, ex)
