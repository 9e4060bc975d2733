"""Multi-rank tile-band fit on the GPU (paper_2510_05814_b200/dist.py): two
processes share the one visible B200 and exchange through gloo collectives
on CUDA tensors (NCCL refuses two ranks on one device; the driver's 8-GPU
runs use NCCL through the same code path): reduce-scatter of the per-band
gradients, all-reduce of the loss partials, Adam on each rank's kernel
shard, in-place all-gather of the parameters.  After k steps both ranks
must hold identical parameters, and both they and a single-process fit must
follow the oracle's fit within the trajectory tolerance (no outliers)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

H, W, C, K, STEPS = 96, 80, 3, 200, 5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    from paper_2510_05814_b200 import synth
    target = synth.image(H, W, C, 501)
    pool = synth.paper_init(target, K, 502, order=1)
    return target, pool


def _rank(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2510_05814_b200 import smoe
    from paper_2510_05814_b200.dist import BandedFit, padded
    torch.cuda.set_device(0)
    target, pool = _inputs()
    h = smoe.SMoE(K, H, W, C, 1)
    p = padded(smoe.Params.from_numpy(pool, "cuda:0"), world)
    fit = BandedFit(h, rank, world)
    tg = torch.as_tensor(target).cuda()
    sse = []
    for t in range(STEPS):
        sums = fit.step(p, tg, smoe.LR.paper(t, STEPS))
        sse.append(float(sums[0]))
    torch.cuda.synchronize()
    q.put((rank, fit.band, p.flat()[:K].cpu().numpy(), sse, (fit.k0, fit.k1)))
    dist.destroy_process_group()


def test_two_ranks_one_gpu_match_single_process():
    from paper_2510_05814_b200 import smoe
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=600) for _ in range(world)], key=lambda r: r[0])
    for pr in procs:
        pr.join(120)
        assert pr.exitcode == 0
    assert res[0][1] == (0, 3) and res[1][1] == (3, 6)          # 6 block rows split 3/3
    assert res[0][4] == (0, 100) and res[1][4] == (100, 200)      # kernel shards
    np.testing.assert_array_equal(res[0][2], res[1][2])          # all-gathered: identical
    # single-process reference
    target, pool = _inputs()
    h = smoe.SMoE(K, H, W, C, 1)
    p = smoe.Params.from_numpy(pool, "cuda:0")
    tg = torch.as_tensor(target).cuda()
    sse1 = []
    for t in range(STEPS):
        g, s = h.grad(p, tg)
        h.apply(p, g, smoe.LR.paper(t, STEPS))
        sse1.append(float(s[0]))
    np.testing.assert_allclose(res[0][3], sse1, rtol=1e-5)
    # both against the oracle fit (trajectory tolerance)
    import oracle as O
    from helpers import assert_params, oracle_fit_with_tolerance
    q, otrace, tol = oracle_fit_with_tolerance(O.Params.from_any(pool), target.astype(np.float64), STEPS,
                                               lambda t: O.LR(O.lr_mu_schedule(t, STEPS)))
    np.testing.assert_allclose(sse1, [tr[0] * H * W * C for tr in otrace], rtol=1e-5)
    assert_params(p.flat().cpu().numpy(), q.flat(), tol, what="single process")
    assert_params(res[0][2], q.flat(), tol, what="two ranks")


def test_band_host_target_copies_band_rows_only():
    """A banded smoe_grad with a HOST target stages only the band's rows; the
    result equals the device-target call (up to the order of the gradient
    atomics) for every band, including the clipped last one."""
    from paper_2510_05814_b200 import smoe
    target, pool = _inputs()
    p = smoe.Params.from_numpy(pool, "cuda:0")
    tg = torch.as_tensor(target).cuda()
    host = torch.as_tensor(target).pin_memory()
    for band in [(0, 2), (2, 5), (5, 6)]:
        h = smoe.SMoE(K, H, W, C, 1)
        h.set_band(*band)
        gd, sd = h.grad(p, tg)
        gh, sh = h.grad(p, host)
        gh2, sh2 = h.grad(p, host)          # second staging buffer
        torch.cuda.synchronize()
        tol = 1e-5 * float(gd.abs().max())
        for g, s in [(gh, sh), (gh2, sh2)]:
            assert torch.allclose(g, gd, rtol=1e-4, atol=tol)
            assert torch.allclose(s, sd, rtol=1e-6, atol=0)
        assert float(sd[0]) > 0
