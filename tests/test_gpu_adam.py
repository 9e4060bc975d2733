"""GPU parity of a8 (Adam + clamp) on the kernel-per-thread
k_adam_kt that runs for large pools (K > 8 x 148 x 256 / V: 18 944 kernels
for C = 3 constant experts, 37 888 for C = 1, i.e. configs 3, 4 and 5), the
sharded update of the multi-GPU path (smoe_apply_ex on a kernel range) and
the capacity-overflow protocol of smoe_grad / smoe_apply / smoe_render with
device buffers.  Everything goes through the C ABI; references come from
the oracle only."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_05814_b200 import smoe, synth
from helpers import assert_params, conditioned, oracle_fit_with_tolerance

pytestmark = pytest.mark.gpu

# (C, order, K, H, W): pools above the element-parallel limit of k_adam
KT_CASES = [(3, 0, 20_000, 96, 96), (1, 0, 40_000, 96, 96)]


def _v(C, order):
    P = 6 + C * (1 + 2 * order)
    return 8 if P <= 8 else 16


def _kt_pool(C, order, K, H, W, seed):
    # small anisotropic kernels (sigma ~ 0.3-0.9 px) so the dense oracle stays
    # cheap at K = 40 000; log pi != 0 and l21 != 0 exercise every term
    pool = synth.aniso_pool(H, W, C, K, seed, order=order, l_range=(0.35, 0.9), shear=0.3, log_pi_sd=0.3,
                            margin_px=1)
    return conditioned(pool, H, W)


@pytest.mark.parametrize("C,order,K,H,W", KT_CASES)
def test_adam_kt_one_step_matches_oracle(C, order, K, H, W):
    """MODE 0 (smoe_step): raw sums -> chain rule -> Adam -> clamp on the
    large-pool kernel, against the oracle's gradient and Adam (same
    per-element bar as test_step_matches_oracle_adam)."""
    assert K > 8 * 148 * (256 // _v(C, order))        # k_adam_kt, not the element-parallel form
    pool = _kt_pool(C, order, K, H, W, 40 + C)
    target = synth.image(H, W, C, 41)
    h = smoe.SMoE(K, H, W, C, order)
    p = smoe.Params.from_numpy(pool, "cuda")
    lr = smoe.LR(mu=0.01, chol=1e-3, log_pi=1e-3, expert=1e-3, slope=2e-4)
    st = h.step(p, torch.as_tensor(target).cuda(), lr)
    op = O.Params.from_any(pool)
    lg = O.loss_grad(op, target.astype(np.float64))
    assert abs(st.loss - lg.loss) <= 1e-5 * lg.loss
    opt = O.Adam(K, op.Pk)
    olr = O.LR(0.01, 1e-3, 1e-3, 1e-3, 2e-4)
    ref = opt.step(op, lg.grad, olr).flat()
    got = p.flat().cpu().numpy().astype(np.float64)
    tol = 1e-3 * olr.vector(C, order)[None, :] + 2e-7 * np.abs(ref)
    small = np.abs(lg.grad) < 1e-5 * lg.grad_abs + 1e-7         # sign not determined
    bad = (np.abs(got - ref) > tol) & ~small
    assert not bad.any(), np.argwhere(bad)[:5]
    assert (~small).mean() > 0.5
    # Adam state: moments of the determined components, step counter
    m1, m2, t = h.get_adam()
    assert t == 1
    det = ~small
    np.testing.assert_allclose(m1.numpy()[det], opt.m1[det], rtol=1e-3, atol=0)
    np.testing.assert_allclose(m2.numpy()[det], opt.m2[det], rtol=2e-3, atol=0)


@pytest.mark.parametrize("C,order,K,H,W", KT_CASES)
def test_adam_kt_fit_trajectory(C, order, K, H, W):
    """MODE 0 over a 5-step fit with the paper's schedule: per-step PSNR
    within 0.01 dB and every parameter within the trajectory tolerance."""
    T = 5
    pool = _kt_pool(C, order, K, H, W, 50 + C)
    target = synth.image(H, W, C, 51)
    h = smoe.SMoE(K, H, W, C, order)
    p = smoe.Params.from_numpy(pool, "cuda")
    tg = torch.as_tensor(target).cuda()
    trace = [h.step(p, tg, smoe.LR.paper(t, T)).psnr_db for t in range(T)]
    q, otrace, tol = oracle_fit_with_tolerance(O.Params.from_any(pool), target.astype(np.float64), T,
                                               lambda t: O.LR(O.lr_mu_schedule(t, T)))
    assert max(abs(a - b[1]) for a, b in zip(trace, otrace)) < 0.01
    assert_params(p.flat().cpu().numpy(), q.flat(), tol)


def _grad_sequence(K, Pk, T, seed):
    """Seeded gradient sequence with |g| bounded away from 0 (so Adam's
    normalised update is determined) and mixed signs/scales per component."""
    g = np.random.default_rng(seed)
    scale = 10.0 ** g.uniform(-6, -2, (1, K, Pk))
    x = g.normal(0, 1, (T, K, Pk))
    x = np.where(np.abs(x) < 0.2, np.sign(x + 1e-12) * 0.2, x)
    return (x * scale).astype(np.float32)


@pytest.mark.parametrize("C,order,K", [(3, 0, 20_000), (1, 0, 40_000), (3, 1, 300)])
def test_apply_trajectory_matches_oracle_adam(C, order, K):
    """MODE 2 (smoe_apply) for 20 steps with seeded gradients: parameters,
    both moments and the step counter follow the oracle's Adam to fp32
    rounding; l11/l22 start near the 1e-3 clamp so it engages."""
    H = W = 64
    T = 20
    pool = synth.aniso_pool(H, W, C, K, 60 + C, order=order, log_pi_sd=0.3)
    pool.chol[::3, 0] = 1.5e-3
    pool.chol[1::3, 2] = 1.2e-3
    Pk = 6 + C * (1 + 2 * order)
    G = _grad_sequence(K, Pk, T, 61)
    h = smoe.SMoE(K, H, W, C, order)
    p = smoe.Params.from_numpy(pool, "cuda")
    op = O.Params.from_any(pool)
    opt = O.Adam(K, Pk)
    tol = np.zeros((K, Pk))
    for t in range(T):
        lr = smoe.LR.paper(t, T)
        lr.log_pi = 1e-3
        h.apply(p, torch.as_tensor(G[t]).cuda(), lr)
        olr = O.LR(lr.mu, lr.chol, lr.log_pi, lr.expert, lr.slope)
        op = opt.step(op, G[t].astype(np.float64), olr)
        # fp32 parameter storage (half an ulp per step) + fp32 Adam arithmetic
        tol += 2.0 ** -24 * np.abs(op.flat()) + 1e-5 * olr.vector(C, order)[None, :]
    assert_params(p.flat().cpu().numpy(), op.flat(), tol, factor=1.0)
    c = p.chol.cpu().numpy()
    assert (c[:, 0] >= 1e-3).all() and (c[:, 2] >= 1e-3).all()
    assert (np.abs(op.chol[:, 0] - 1e-3) < 1e-12).any()          # the clamp engaged
    m1, m2, tt = h.get_adam()
    assert tt == T
    # fp32 accumulation of the moments: relative to the largest term of the
    # (possibly cancelling) sum, per component
    gmax = np.abs(G).max(axis=0).astype(np.float64)
    assert (np.abs(m1.numpy() - opt.m1) <= 1e-5 * np.abs(opt.m1) + 1e-6 * gmax).all()
    assert (np.abs(m2.numpy() - opt.m2) <= 1e-5 * np.abs(opt.m2) + 1e-6 * gmax ** 2).all()


@pytest.mark.parametrize("K", [300, 20_000])
def test_sharded_apply_equals_full_apply(K):
    """smoe_apply_ex on kernel shards (the multi-GPU reduce-scatter -> per-rank
    Adam path) updates exactly the shard's parameters and gives bit-identical
    results to the full update, step after step."""
    H = W = 64
    C, order = 3, 0
    pool = synth.aniso_pool(H, W, C, K, 70, order=order)
    Pk = 9
    G = _grad_sequence(K, Pk, 3, 71)
    full = smoe.Params.from_numpy(pool, "cuda")
    shard = smoe.Params.from_numpy(pool, "cuda")
    cuts = [0, K // 3, K // 3 + 1, K]                  # includes a one-kernel shard
    hf = smoe.SMoE(K, H, W, C, order)
    hs = [smoe.SMoE(K, H, W, C, order) for _ in range(len(cuts) - 1)]   # one handle per "rank"
    for t in range(3):
        lr = smoe.LR.paper(t, 3)
        g = torch.as_tensor(G[t]).cuda()
        hf.apply(full, g, lr)
        before = shard.flat().clone()
        for i, hh in enumerate(hs):
            k0, k1 = cuts[i], cuts[i + 1]
            hh.apply(shard, g[k0:k1].contiguous(), lr, k0, k1)
            after = shard.flat()
            if i == 0:    # rows beyond the first shard untouched so far
                assert torch.equal(after[k1:], before[k1:])
        assert torch.equal(shard.flat(), full.flat())


def test_apply_skips_when_a_rank_overflowed():
    """The all-reduced sums[3] (skipped flag) gates the update on the device
    (and on the host for a host sums array)."""
    H = W = 32
    K = 50
    pool = synth.aniso_pool(H, W, 1, K, 80)
    h = smoe.SMoE(K, H, W, 1, 0)
    p = smoe.Params.from_numpy(pool, "cuda")
    g = torch.full((K, 7), 1e-3, device="cuda")
    before = p.flat().clone()
    h.apply(p, g, smoe.LR(), sums=torch.tensor([0.0, 0.0, 0.0, 1.0], dtype=torch.float64, device="cuda"))
    h.apply(p, g, smoe.LR(), sums=np.array([0.0, 0.0, 0.0, 2.0]))
    torch.cuda.synchronize()
    assert torch.equal(p.flat(), before)
    assert h.get_adam()[2] == 0
    h.apply(p, g, smoe.LR(), sums=torch.zeros(4, dtype=torch.float64, device="cuda"))
    assert not torch.equal(p.flat(), before) and h.get_adam()[2] == 1


def test_grad_and_render_overflow_with_device_buffers():
    """ADVICE (round 1): an overflowing binning on the asynchronous paths.
    smoe_grad with device grad/sums writes a zero gradient and sums[3] = 1,
    an update gated by those sums does nothing, smoe_sync reports
    SMOE_ERR_CAPACITY after growing the lists, and the next call is correct;
    a render into a device buffer leaves NaN (never stale memory)."""
    H = W = 256
    K = 400
    pool = conditioned(synth.aniso_pool(H, W, 1, K, 12), H, W)
    target = torch.as_tensor(synth.image(H, W, 1, 13)).cuda()
    h = smoe.SMoE(K, H, W, 1, 0)
    p = smoe.Params.from_numpy(pool, "cuda")
    h.grad(p, target)                                  # calibrates the training grid
    out = torch.zeros((1, H, W), device="cuda")
    h.render(p, out=out)                               # calibrates the render grid
    h.sync()
    big = p.clone()
    big.chol *= 8.0                                    # ~64x more pairs
    g, s = h.grad(big, target)
    out.zero_()
    h.render(big, out=out)
    torch.cuda.synchronize()
    assert float(s[3]) == 1.0 and float(s[0]) == 0.0
    assert float(g.abs().max()) == 0.0
    assert bool(torch.isnan(out).all())
    before = big.flat().clone()
    h.apply(big, g, smoe.LR(), sums=s)
    torch.cuda.synchronize()
    assert torch.equal(big.flat(), before)
    with pytest.raises(smoe.SmoeError) as e:
        h.sync()
    assert e.value.status == smoe.ERR_CAPACITY
    g2, s2 = h.grad(big, target)
    y = h.render(big)
    ref = smoe.SMoE(K, H, W, 1, 0)
    g3, s3 = ref.grad(big, target)
    torch.cuda.synchronize()
    assert float(s2[3]) == 0.0 and abs(float(s2[0]) - float(s3[0])) <= 1e-9 * float(s3[0])
    assert torch.allclose(g2, g3, rtol=1e-4, atol=1e-6 * float(g3.abs().max()))
    assert bool(torch.isfinite(y).all())
