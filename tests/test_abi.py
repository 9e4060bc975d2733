"""CPU-side checks of the C-ABI library (no device compute): it loads, exports
every entry point include/smoe.h declares, and its host-only functions behave
(status strings, options, the paper lr schedule, graceful failure without a
device)."""
import ctypes
import math
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "smoe.h")


@pytest.fixture(scope="module")
def L():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "paper_2510_05814_b200", "csrc")])
    from paper_2510_05814_b200 import smoe
    return smoe.lib()


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(smoe_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared()
    for n in ("smoe_create", "smoe_render", "smoe_step", "smoe_grad", "smoe_apply", "smoe_set_band"):
        assert n in names


def test_every_declared_symbol_is_exported(L):
    names = declared()
    assert len(names) >= 15
    out = subprocess.check_output(["nm", "-D", "--defined-only",
                                   os.path.join(ROOT, "paper_2510_05814_b200", "libsmoe.so")]).decode()
    exported = set(re.findall(r"\bT (smoe_\w+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        getattr(L, n)


def test_library_is_sm100a(L):
    out = subprocess.check_output(["cuobjdump", "--list-elf",
                                   os.path.join(ROOT, "paper_2510_05814_b200", "libsmoe.so")]).decode()
    assert "sm_100a" in out


def test_host_only_functions(L):
    from paper_2510_05814_b200 import smoe
    assert L.smoe_abi_version() == 2
    names = [L.smoe_kernel_name(i).decode() for i in range(smoe.KERNEL_COUNT)]
    assert names == ["k_preprocess", "k_scatter", "k_raster<train>", "k_raster<render>", "k_adam", "k_bin",
                     "k_scan_lookback", "k_emit"]
    assert L.smoe_kernel_name(smoe.KERNEL_COUNT) == b"?"
    assert L.smoe_apply_ex(None, None, None, None, 0, 0, None) == smoe.ERR_BAD_HANDLE
    assert L.smoe_status_string(0) == b"ok"
    assert L.smoe_status_string(5) == b"pair capacity exceeded"
    o = smoe.c_options()
    assert L.smoe_default_options(ctypes.byref(o)) == 0
    assert abs(o.R2 - 2 * math.log(100.0)) < 1e-15 and o.device == -1 and o.box_mode == 1
    # paper lr schedule
    assert abs(L.smoe_paper_lr(0, 10000).mu - 0.01) < 1e-9
    assert abs(L.smoe_paper_lr(5000, 10000).mu - 3.1623e-4) < 1e-7
    assert abs(L.smoe_paper_lr(10000, 10000).mu - 1e-5) < 1e-10
    lr = L.smoe_paper_lr(3, 10)
    assert lr.chol == pytest.approx(1e-3) and lr.expert == pytest.approx(1e-3) and lr.log_pi == 0.0


def test_invalid_arguments_and_no_device(L):
    from paper_2510_05814_b200 import smoe
    h = ctypes.c_void_p()
    assert L.smoe_create(0, 8, 8, 1, 0, ctypes.byref(h)) == smoe.ERR_INVALID_ARG
    assert L.smoe_create(4, 8, 8, 2, 0, ctypes.byref(h)) == smoe.ERR_INVALID_ARG
    assert L.smoe_create(4, 8, 8, 1, 2, ctypes.byref(h)) == smoe.ERR_INVALID_ARG
    assert L.smoe_step(None, None, None, None, None) == smoe.ERR_BAD_HANDLE
    assert L.smoe_destroy(None) == smoe.ERR_BAD_HANDLE
    import torch
    if not torch.cuda.is_available():
        st = L.smoe_create(4, 8, 8, 1, 0, ctypes.byref(h))
        assert st == smoe.ERR_CUDA and not h.value


def test_binding_validates_buffers():
    """ADVICE (round 1): the binding checks dtype, element count and layout
    of what it hands the library (no GPU needed: the checks run first)."""
    import numpy as np
    import torch
    from paper_2510_05814_b200 import smoe
    with pytest.raises(smoe.SmoeError) as e:
        smoe._ptr(torch.zeros(4, dtype=torch.float64), "target", torch.float32, 4)
    assert e.value.status == smoe.ERR_INVALID_ARG
    with pytest.raises(smoe.SmoeError):
        smoe._ptr(np.zeros(3), "sums", torch.float64, 4)          # host sums too short
    with pytest.raises(smoe.SmoeError):
        smoe._ptr(np.zeros(8, np.float64), "grad", torch.float32, 8)
    with pytest.raises(smoe.SmoeError):
        smoe._ptr(torch.zeros(4, 4).t(), "out", torch.float32, 16)  # not contiguous
    with pytest.raises(smoe.SmoeError):
        smoe._ptr([1.0, 2.0], "grad")
    assert smoe._ptr(np.zeros(4), "sums", torch.float64, 4) != 0
    assert smoe._ptr(None) is None


def test_segment_init_rejects_empty_segments_and_bad_shape(L):
    """ADVICE (round 1): a segment id with no pixel, or H/W < 1, is an
    invalid argument (no out-of-bounds read)."""
    import numpy as np
    from paper_2510_05814_b200 import smoe
    H, W, C, K = 4, 5, 1, 6
    img = np.zeros((C, H, W), np.float32)
    lab = np.zeros((H, W), np.int32)
    lab[:, 3:] = 2                               # ids 0 and 2 used, 1 empty
    with pytest.raises(smoe.SmoeError) as e:
        smoe.segment_init(img, lab, 3, K)
    assert e.value.status == smoe.ERR_INVALID_ARG
    mu = np.zeros((K, 2), np.float32)
    P = lambda a: a.ctypes.data
    ch, lp, ex = np.zeros((K, 3), np.float32), np.zeros(K, np.float32), np.zeros((K, C, 1), np.float32)
    assert L.smoe_segment_init(P(img), 0, W, C, P(lab), 1, K, 0, 0, 5.0, P(mu), P(ch), P(lp), P(ex)) == smoe.ERR_INVALID_ARG
    pool = smoe.segment_init(img, np.minimum(lab, 1), 2, K)
    assert pool.mu.shape == (K, 2)


def test_binding_fails_loudly_without_library(tmp_path, monkeypatch):
    from paper_2510_05814_b200 import smoe
    monkeypatch.setattr(smoe, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(smoe, "_LIB", None)
    with pytest.raises(ImportError):
        smoe.lib()
