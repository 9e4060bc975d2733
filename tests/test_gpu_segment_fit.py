"""f4 on the GPU path (Eq. 9): a denoising fit whose
kernel pool comes from the segmentation initialisation (smoe_segment +
smoe_segment_init, host C++) follows the oracle's fit of the same pool --
PSNR trace within the north-star 0.01 dB and every parameter within the
trajectory tolerance after T steps.  The segmentation itself
is pinned label-exact against oracle/segment.py in tests/test_segment.py;
this is the fit it feeds, through the C ABI."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_05814_b200 import smoe, synth
from helpers import assert_params, conditioned, oracle_fit_with_tolerance

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("order", [0, 1])
def test_segmentation_init_fit_matches_oracle(order):
    H, W, C, T = 44, 52, 3, 20
    clean = synth.image(H, W, C, 21)
    noisy = synth.noisy(clean, 25.0 / 255.0, 22)
    labels, n = smoe.segment(noisy, 10.0, 16)
    K = 2 * n + 40
    pool = smoe.segment_init(noisy, labels, n, K, order=order, seed=3, scale_px=2.5)
    pool = conditioned(pool, H, W)                      # rule P1 (fp32 and fp64 take the same cull decisions)
    target = noisy.astype(np.float32)
    h = smoe.SMoE(K, H, W, C, order)
    p = smoe.Params.from_numpy(pool, "cuda")
    tg = torch.as_tensor(target).cuda()
    trace = [h.step(p, tg, smoe.LR.paper(t, T)).psnr_db for t in range(T)]
    q, otrace, tol = oracle_fit_with_tolerance(O.Params.from_any(pool), target.astype(np.float64), T,
                                               lambda t: O.LR(O.lr_mu_schedule(t, T)))
    h.close()
    assert max(abs(a - b[1]) for a, b in zip(trace, otrace)) < 0.01
    assert_params(p.flat().cpu().numpy(), q.flat(), tol)
