"""Both render raster forms against the oracle, whichever the host picks:
the two-pixels-per-lane k_raster<render> (4 warps per 16x16 block) and the
four-pixels-per-lane k_render4 (2 warps per block; chosen for grids with
short buckets).  SMOE_RENDER4=0/1 forces the form per launch."""
import numpy as np
import pytest
import torch

import oracle as O
from paper_2510_05814_b200 import smoe, synth
from helpers import assert_pixels, conditioned

pytestmark = pytest.mark.gpu

@pytest.mark.parametrize("form", ["0", "1"])
@pytest.mark.parametrize("scale", [1.0, 2.0, 0.5, 1.5])
def test_render_forms_parity(scale, form, monkeypatch):
    monkeypatch.setenv("SMOE_RENDER4", form)
    H, W, C, K = 45, 61, 3, 120
    oH, oW = int(round(H * scale)), int(round(W * scale))
    pool = synth.aniso_pool(H, W, C, K, 400, order=1, margin_px=6, log_pi_sd=0.5)
    pool = conditioned(pool, H, W, oH, oW)
    h = smoe.SMoE(K, H, W, C, 1)
    y = h.render(smoe.Params.from_numpy(pool, "cuda"), oH, oW).cpu().numpy()
    y_ref, _ = O.render(O.Params.from_any(pool), H, W, oH, oW)
    assert_pixels(y, y_ref)
    acc = torch.full((C, oH, oW), 0.25, device="cuda")
    h.render(smoe.Params.from_numpy(pool, "cuda"), oH, oW, out=acc, accumulate=0.5)
    np.testing.assert_allclose(acc.cpu().numpy(), 0.25 + 0.5 * y, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("form", ["0", "1"])
@pytest.mark.parametrize("C,order,rbf", [(1, 0, False), (3, 0, True), (1, 1, False)])
def test_render_forms_heads_and_ragged(C, order, rbf, form, monkeypatch):
    """Grayscale, constant experts, the RBF head, ragged sizes and more than
    one record batch (> 128 kernels per block) in both forms."""
    monkeypatch.setenv("SMOE_RENDER4", form)
    H, W, K = 29, 43, 500
    pool = synth.aniso_pool(H, W, C, K, 410 + C, order=order, l_range=(1.5, 4.0), shear=1.0, margin_px=3)
    if rbf:
        pool.expert[:, :, 0] *= 0.2
    pool = conditioned(pool, H, W, 2 * H + 1, 2 * W - 3)
    h = smoe.SMoE(K, H, W, C, order, head="rbf" if rbf else "smoe")
    y = h.render(smoe.Params.from_numpy(pool, "cuda"), 2 * H + 1, 2 * W - 3).cpu().numpy()
    with O.head("rbf" if rbf else "smoe"):
        y_ref, _ = O.render(O.Params.from_any(pool), H, W, 2 * H + 1, 2 * W - 3)
    assert_pixels(y, y_ref)
