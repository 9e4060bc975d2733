"""Fused records (include/smoe.h smoe_invalidate): with the
two-stage binning the Adam of smoe_step writes the next step's kernel
records and tile boxes (the geometry of P:215-221) for the parameters it
just updated, and the next step on the same parameters skips k_records.

A pass that uses the fused records must see exactly the lists, pixels and
loss of a fresh binning of the same parameters: the gradient pass of the
stepped handle (warm: no k_records) is compared with a new handle's (cold),
right after each call that must invalidate the fused records (an in-place
parameter edit by the caller, a render, smoe_apply, a band change).  The
loss partials are fp64 sums of deterministic per-block values (equal to
~1e-15); gradients are float atomics in a nondeterministic order, so they
are compared at 1e-5 relative (stale records would move them by the
parameter step, ~1e-2).  Element-wise parity of the fused path against the
oracle is in test_gpu_adam.py (its K >= 16 384 pools run it)."""
import numpy as np
import pytest
import torch

from paper_2510_05814_b200 import smoe, synth

pytestmark = pytest.mark.gpu

H, W, K = 72, 104, 400


def _grad(h, prm, tgt):
    g, s = h.grad(prm, tgt)
    torch.cuda.synchronize()
    return g.cpu().numpy().astype(np.float64), s.cpu().numpy()


# binning -> (SMOE_PERM, launches of a warm step, of a cold step); one-pass
# binning (SMOE_PERM=0 at this K) has no fused form: every step is cold
BINNINGS = {"two_stage": ("1", 3, 4), "one_pass": ("0", 3, 3)}


@pytest.mark.parametrize("binning", list(BINNINGS))
@pytest.mark.parametrize("C,order", [(3, 0), (1, 1)])
@pytest.mark.parametrize("event", [None, "edit", "render", "apply", "band"])
def test_fused_records_match_fresh_binning(monkeypatch, binning, C, order, event):
    perm, warm, cold = BINNINGS[binning]
    monkeypatch.setenv("SMOE_PERM", perm)                    # two-stage binning even at this small K, or not
    monkeypatch.setenv("SMOE_FUSE_REC", "1")
    pool = synth.aniso_pool(H, W, C, K, 3, order=order)
    prm = smoe.Params.from_numpy(pool, "cuda:0")
    tgt = torch.as_tensor(synth.image(H, W, C, 4)).cuda()
    h = smoe.SMoE(K, H, W, C, order)
    launches = []
    for it in range(6):
        n0 = h.launch_count()
        h.step(prm, tgt, smoe.LR(), stats=(it == 0))
        torch.cuda.synchronize()
        launches.append(h.launch_count() - n0)
    # steady state: (k_emit,) raster, Adam (the Adam wrote the records)
    assert launches[3:] == [warm] * 3, launches
    band = None
    if event == "edit":
        prm.mu.add_(0.37)                                    # the caller writes the parameters
    elif event == "render":
        h.render(prm, 2 * H, 2 * W)
    elif event == "apply":
        g, _ = h.grad(prm, tgt)
        h.apply(prm, g, smoe.LR())
    elif event == "band":
        band = (1, (H + 15) // 16)
        h.set_band(*band)
    n0 = h.launch_count()
    g1, s1 = _grad(h, prm, tgt)
    # warm only when nothing invalidated
    assert h.launch_count() - n0 == (warm if event is None else cold)
    h2 = smoe.SMoE(K, H, W, C, order)
    if band:
        h2.set_band(*band)
    g2, s2 = _grad(h2, prm.clone(), tgt)
    h.close()
    h2.close()
    np.testing.assert_allclose(s1[:3], s2[:3], rtol=1e-12, atol=0)
    assert s1[3] == s2[3] == 0.0
    tol = 1e-5 * np.abs(g2) + 1e-6 * np.abs(g2).max()
    bad = np.abs(g1 - g2) > tol
    assert not bad.any(), f"{bad.sum()} gradient entries differ, worst {np.abs(g1 - g2).max():.3e}"


@pytest.mark.parametrize("binning", list(BINNINGS))
def test_fused_records_off_launches_k_records(monkeypatch, binning):
    """SMOE_FUSE_REC=0: every step runs its own preprocessing."""
    perm, warm, cold = BINNINGS[binning]
    monkeypatch.setenv("SMOE_PERM", perm)
    monkeypatch.setenv("SMOE_FUSE_REC", "0")
    C, order = 3, 0
    pool = synth.aniso_pool(H, W, C, K, 3, order=order)
    prm = smoe.Params.from_numpy(pool, "cuda:0")
    tgt = torch.as_tensor(synth.image(H, W, C, 4)).cuda()
    h = smoe.SMoE(K, H, W, C, order)
    launches = []
    for it in range(5):
        n0 = h.launch_count()
        h.step(prm, tgt, smoe.LR(), stats=False)
        torch.cuda.synchronize()
        launches.append(h.launch_count() - n0)
    h.close()
    assert launches[2:] == [cold] * 3, launches


@pytest.mark.parametrize("binning", list(BINNINGS))
def test_fused_emission_overflow_recovers(monkeypatch, binning):
    """A step whose update grows the kernels past the bucket capacity: the
    next step's binning (on fused or fresh records) overflows, is skipped,
    grown and redone; the trajectory must match the unfused one."""
    perm = BINNINGS[binning][0]
    monkeypatch.setenv("SMOE_PERM", perm)
    C, order = 3, 0
    pool = synth.aniso_pool(H, W, C, K, 5, order=order)
    tgt = torch.as_tensor(synth.image(H, W, C, 6)).cuda()
    big = smoe.LR(mu=0.01, chol=1.5, log_pi=0.01, expert=0.01, slope=0.0)   # Cholesky factors jump by ~1.5 px
    runs = []
    for fuse in ("0", "1"):
        monkeypatch.setenv("SMOE_FUSE_REC", fuse)
        prm = smoe.Params.from_numpy(pool, "cuda:0")
        h = smoe.SMoE(K, H, W, C, order)
        losses, pairs = [], []
        for it in range(10):
            st = h.step(prm, tgt, big if it == 4 else smoe.LR())
            losses.append(st.loss)
            pairs.append(st.pairs)
        runs.append(([t.cpu().numpy().astype(np.float64) for t in (prm.mu, prm.chol, prm.log_pi, prm.expert)],
                     np.array(losses)))
        h.close()
    (pa, la), (pb, lb) = runs
    np.testing.assert_allclose(lb, la, rtol=1e-4)
    for x, y in zip(pa, pb):
        np.testing.assert_allclose(y, x, rtol=1e-3, atol=1e-4)


def test_explicit_invalidate_after_untracked_write(monkeypatch):
    """A write the binding cannot see (through ``.data``, which does not move
    the tensor's version counter) followed by ``smoe_invalidate``: the next
    gradient pass bins afresh (cold launch count) and equals a new handle's."""
    perm, warm, cold = BINNINGS["two_stage"]
    monkeypatch.setenv("SMOE_PERM", perm)
    monkeypatch.setenv("SMOE_FUSE_REC", "1")
    C, order = 3, 0
    pool = synth.aniso_pool(H, W, C, K, 3, order=order)
    prm = smoe.Params.from_numpy(pool, "cuda:0")
    tgt = torch.as_tensor(synth.image(H, W, C, 4)).cuda()
    h = smoe.SMoE(K, H, W, C, order)
    for it in range(5):
        h.step(prm, tgt, smoe.LR(), stats=(it == 0))
    torch.cuda.synchronize()
    v0 = prm.mu._version
    prm.mu.data.add_(0.37)
    assert prm.mu._version == v0                      # invisible to the binding
    h.invalidate()
    n0 = h.launch_count()
    g1, s1 = _grad(h, prm, tgt)
    assert h.launch_count() - n0 == cold
    h2 = smoe.SMoE(K, H, W, C, order)
    g2, s2 = _grad(h2, prm.clone(), tgt)
    h.close()
    h2.close()
    np.testing.assert_allclose(s1[:3], s2[:3], rtol=1e-12, atol=0)
    tol = 1e-5 * np.abs(g2) + 1e-6 * np.abs(g2).max()
    assert not (np.abs(g1 - g2) > tol).any()
