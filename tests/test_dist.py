"""Multi-rank host logic on CPU (gloo, world size 2): tile-row band partition
and the gradient all-reduce of paper_2510_05814_b200/dist.py.  The per-band
gradients come from the oracle (the CUDA path is exercised by the GPU band
additivity test); what is checked here is that the band split plus the sum
over ranks reproduces the full-image gradient and keeps every rank's Adam
update identical."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_05814_b200.dist import allgather_params, allreduce_grads, band_rows, reduce_scatter_grads, shard_rows


def test_band_rows_partition():
    for ny in (1, 2, 5, 32, 85, 270, 339):
        for world in (1, 2, 3, 4, 8):
            bands = [band_rows(ny, r, world) for r in range(world)]
            assert bands[0][0] == 0 and bands[-1][1] == ny
            for (a0, a1), (b0, b1) in zip(bands, bands[1:]):
                assert a1 == b0
            sizes = [b - a for a, b in bands]
            assert max(sizes) - min(sizes) <= 1
    assert [b - a for a, b in (band_rows(270, r, 8) for r in range(8))] == [34] * 6 + [33] * 2
    with pytest.raises(ValueError):
        band_rows(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import oracle as O
    from paper_2510_05814_b200 import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H, W, C, K = 48, 40, 3, 30
    pool = synth.aniso_pool(H, W, C, K, 77, order=1)
    target = synth.image(H, W, C, 78).astype(np.float64)
    p = O.Params.from_any(pool)
    ny = (H + 15) // 16
    r0, r1 = band_rows(ny, rank, world)
    lg = O.loss_grad(p, target, rows=(r0 * 16, min(r1 * 16, H)))
    grad = torch.tensor(lg.grad, dtype=torch.float64)
    sums = torch.tensor([lg.sse, lg.sse_clamped, float(lg.uncovered)], dtype=torch.float64)
    allreduce_grads(grad, sums)
    opt = O.Adam(K, p.Pk)
    q2 = opt.step(p, grad.numpy(), O.LR())
    q.put((rank, grad.numpy(), sums.numpy(), q2.flat()))
    dist.destroy_process_group()


def test_gloo_world2_band_allreduce_matches_full():
    import oracle as O
    from paper_2510_05814_b200 import synth
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(60)
        assert pr.exitcode == 0
    res.sort(key=lambda r: r[0])
    H, W, C, K = 48, 40, 3, 30
    pool = synth.aniso_pool(H, W, C, K, 77, order=1)
    full = O.loss_grad(O.Params.from_any(pool), synth.image(H, W, C, 78).astype(np.float64))
    for _, g, s, _ in res:
        np.testing.assert_allclose(g, full.grad, rtol=1e-12, atol=1e-17)
        assert abs(s[0] - full.sse) < 1e-12
    # identical inputs -> identical replicated Adam updates on every rank
    np.testing.assert_array_equal(res[0][3], res[1][3])


def test_shard_rows_partition():
    for K in (1, 2, 7, 30, 1000, 1_000_001):
        for world in (1, 2, 3, 8):
            rows = [shard_rows(K, r, world) for r in range(world)]
            Ks = rows[0][2]
            assert Ks * world >= K and (Ks - 1) * world < K
            assert rows[0][0] == 0 and rows[-1][1] == K
            for (a0, a1, _), (b0, b1, _) in zip(rows, rows[1:]):
                assert a1 == b0 and a1 - a0 <= Ks


def _sharded_worker(rank, world, port, q):
    """Band gradient (oracle) -> reduce-scatter -> Adam on this rank's kernel
    shard (oracle Adam) -> in-place all-gather of the padded parameter
    arrays: the host logic of BandedFit with the CUDA calls replaced by the
    oracle."""
    import oracle as O
    from paper_2510_05814_b200 import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    H, W, C, K = 48, 40, 3, 31                       # K not divisible by world: padded shards
    pool = synth.aniso_pool(H, W, C, K, 77, order=1)
    target = synth.image(H, W, C, 78).astype(np.float64)
    p = O.Params.from_any(pool)
    ny = (H + 15) // 16
    r0, r1 = band_rows(ny, rank, world)
    k0, k1, Ks = shard_rows(K, rank, world)
    Kpad = Ks * world
    flat = np.zeros((Kpad, p.Pk))
    flat[:K] = p.flat()
    arrays = [torch.tensor(flat[:, a:b].copy()) for a, b in ((0, 2), (2, 5), (5, 6), (6, p.Pk))]
    opt = O.Adam(k1 - k0, p.Pk)
    for t in range(3):
        cur = np.concatenate([a.numpy() for a in arrays], 1)[:K]
        pc = O.Params.unflat(cur, C, 1)
        lg = O.loss_grad(pc, target, rows=(r0 * 16, min(r1 * 16, H)))
        gpad = torch.zeros((Kpad, p.Pk), dtype=torch.float64)
        gpad[:K] = torch.tensor(lg.grad)
        shard = torch.zeros((Ks, p.Pk), dtype=torch.float64)
        sums = torch.tensor([lg.sse, lg.sse_clamped, float(lg.uncovered), 0.0], dtype=torch.float64)
        reduce_scatter_grads(gpad, shard, sums)
        if sums[3] == 0 and k1 > k0:
            sp = O.Params.unflat(cur[k0:k1], C, 1)
            new = opt.step(sp, shard[:k1 - k0].numpy(), O.LR()).flat()
            for a, (lo, hi) in zip(arrays, ((0, 2), (2, 5), (5, 6), (6, p.Pk))):
                a[k0:k1] = torch.tensor(new[:, lo:hi])
        allgather_params(arrays, rank, world, Ks)
    q.put((rank, np.concatenate([a.numpy() for a in arrays], 1)[:K], float(sums[0])))
    dist.destroy_process_group()


def test_gloo_world2_sharded_adam_matches_replicated():
    """The reduce-scatter -> sharded Adam -> all-gather exchange reproduces
    the single-process full-image fit (3 steps) on every rank."""
    import oracle as O
    from paper_2510_05814_b200 import synth
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_sharded_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda r: r[0])
    for pr in procs:
        pr.join(60)
        assert pr.exitcode == 0
    H, W, C, K = 48, 40, 3, 31
    pool = synth.aniso_pool(H, W, C, K, 77, order=1)
    target = synth.image(H, W, C, 78).astype(np.float64)
    p = O.Params.from_any(pool)
    opt = O.Adam(K, p.Pk)
    for t in range(3):
        lg = O.loss_grad(p, target)
        p = opt.step(p, lg.grad, O.LR())
    np.testing.assert_array_equal(res[0][1], res[1][1])
    np.testing.assert_allclose(res[0][1], p.flat(), rtol=1e-12, atol=1e-14)
    assert abs(res[0][2] - lg.sse) < 1e-12 * lg.sse
