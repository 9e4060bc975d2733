#!/usr/bin/env python
"""bench.py -- Rasterized SMoE fit iterations/s (and render Mpix/s) on B200.

Metric (BASELINE.json): "SMoE fit iterations/s and render Mpix/s at 1/2/4/8
B200 (% of roofline)".  One bench step = one fit iteration of the whole hot
path (§8(a) a1-a8: preprocess, binning, forward, loss, backward, Adam) over
the configured synthetic workload; the render (a9) is timed separately, on
the fitted model, and reported under "render".  Default workload:
BASELINE.json config 3 (2040x1356 RGB DIV2K-shaped synthetic image, 100k
kernels, 2000-iteration fit + 4x native super-resolution render), the
largest configuration that fits one GPU (config 5 is the multi-GPU one).
N > 1 (torchrun): tile-row bands per rank, reduce-scatter of the gradients,
sharded Adam, all-gather of the parameters every step
(paper_2510_05814_b200/dist.py).

Timing: W warm-up steps; then K steps, each bracketed by CUDA events on the
launch stream with an L2 flush (256 MB write + 256 MB read) between steps outside the
events; barrier + synchronize on both sides; max over ranks.  The library's
own event pairs (smoe_profile_*) time every kernel inside the same region.

--impl reference: the CPU oracle (oracle/), as it stands, on the host, on a
bounded sample of the same workload per step (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Algorithmic FP32 lane-op counts of the raster (from SURVEY
# §8(d)): per tested (pixel, kernel) pair 7 (dx, dy, u, v x2, d^2 x2); per
# pair inside the ellipse (2 + C + 2 C o) forward + (12 + 2 C + 4 C o) backward.
def ops_per_unit(C, order):
    return 7, (2 + C + 2 * C * order) + (12 + 2 * C + 4 * C * order)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "10"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(5)
        except Exception:
            self.p.kill()
        self.f.flush()
        rows = [l.strip().split(", ") for l in open(self.f.name) if l.strip()]
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if len(r) >= 9]
        mx = [float(r[2]) for r in rows if len(r) >= 9]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for n, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def rank_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def cpu_info():
    """Host CPU model and core count (the cpu_baseline's context)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def cpu_oracle_sample(target, pool, rows):
    """Time the CPU oracle's loss+gradient on image rows [r0, r1) (dense over
    all kernels, fp64, one thread) plus its Adam step, pinned to one core
    (the equivalent of taskset -c <core>).  Returns (seconds for the rows,
    seconds for Adam, the core)."""
    import numpy as np
    import oracle as O
    op = O.Params.from_any(pool)
    t = target.astype(np.float64)
    old = os.sched_getaffinity(0)
    core = min(old)
    os.sched_setaffinity(0, {core})
    try:
        t0 = time.perf_counter()
        lg = O.loss_grad(op, t, rows=rows)
        t1 = time.perf_counter()
        opt = O.Adam(op.K, op.Pk)
        opt.step(op, lg.grad, O.LR())
        t2 = time.perf_counter()
    finally:
        os.sched_setaffinity(0, old)
    return t1 - t0, t2 - t1, core


def run_reference(args):
    rank, world, _ = rank_env()
    if rank != 0:
        return 0
    from paper_2510_05814_b200 import synth
    cfg = synth.CONFIGS[args.config]
    target, _, pool = synth.workload(args.config)
    H = cfg["H"]
    rows_per_step = 1
    times = []
    for i in range(args.warmup + args.steps):
        r0 = (i * 97) % (H - rows_per_step + 1)
        tg, ta, core = cpu_oracle_sample(target, pool, (r0, r0 + rows_per_step))
        if i >= args.warmup:
            times.append((tg, ta))
    tg = sum(t[0] for t in times) / len(times)
    ta = sum(t[1] for t in times) / len(times)
    sec_per_iter = tg * H / rows_per_step + ta
    value = 1.0 / sec_per_iter
    sample = (f"per step: dense fp64 loss+gradient of {rows_per_step} image row (of {H}) over all "
              f"{cfg['K']} kernels + one full Adam step; it/s = 1/(H/rows * t_rows + t_adam)")
    out = {
        "impl": "reference", "metric": "SMoE fit iterations/s", "value": value, "unit": "it/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sec_per_iter * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(args.config, world),
        "cpu_baseline": dict({"value": value, "unit": "it/s", "cores": 1, "kind": "oracle", "sample": sample,
                              "pinned_core": core}, **cpu_info()),
        "e2e": {"value": value, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))
    return 0


def run_mm(args):
    """MM-RSMoE: H hypotheses of the config's (noisy) image fitted
    concurrently on one GPU, fused by averaging (Eq. 11).  Reports hypothesis
    iterations/s over the timed fit and the PSNR of single vs fused models
    against the clean image."""
    import numpy as np
    import torch
    from paper_2510_05814_b200 import smoe, synth
    from paper_2510_05814_b200.multimodel import MultiModel, init_hypotheses
    cfg = synth.CONFIGS[args.config]
    C, H, W, K, order = cfg["C"], cfg["H"], cfg["W"], cfg["K"], cfg["order"]
    target, clean, _ = synth.workload(args.config)
    seg_info = None
    if args.seg > 0:
        t0 = time.perf_counter()
        labels, nseg = smoe.segment(np.clip(target, 0, 1), args.seg, 16)
        t1 = time.perf_counter()
        pools = [smoe.segment_init(target, labels, nseg, K, order, seed=1234 + cfg["cfg"] + 1 + h)
                 for h in range(args.mm)]
        t2 = time.perf_counter()
        seg_info = {"threshold": args.seg, "segments": nseg, "segment_s": t1 - t0, "init_s": (t2 - t1) / args.mm}
    else:
        pools = init_hypotheses(target, K, args.mm, 1234 + cfg["cfg"] + 1, order)
    mm = MultiModel(args.mm, K, H, W, C, order)
    prms = [smoe.Params.from_numpy(p, "cuda") for p in pools]
    tg = torch.as_tensor(target).cuda()
    T = args.warmup + args.steps
    for t in range(args.warmup):
        mm.step(prms, tg, smoe.LR.paper(t, T))
    for hd in mm.handles:
        hd.sync()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(args.warmup, T):
        mm.step(prms, tg, smoe.LR.paper(t, T))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    fused = mm.render(prms).cpu().numpy()
    psnr = lambda y: float(10 * np.log10(1.0 / np.mean((np.clip(y, 0, 1) - clean) ** 2)))
    singles = [psnr(mm.handles[i].render(prms[i]).cpu().numpy()) for i in range(args.mm)]
    out = {"metric": "MM-RSMoE hypothesis iterations/s", "value": args.mm * args.steps / (ms * 1e-3),
           "unit": "hypothesis-it/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
           "hypotheses": args.mm, "ms_per_step": ms / args.steps, "higher_is_better": True,
           "config": config_dict(args.config, 1), "data": "synthetic",
           "psnr_noisy_db": psnr(target), "psnr_single_db_mean": float(np.mean(singles)),
           "psnr_fused_db": psnr(fused), "l2": "not flushed (concurrent hypotheses)",
           "init": seg_info or "paper random init per hypothesis (seed + shift)"}
    print(json.dumps(out))
    return 0


def run_project(args):
    """Per-rank projection of the multi-GPU fit on ONE GPU:
    for N ranks, time rank r's share of a step -- smoe_grad on its band of
    block rows (band-local preprocess + binning + raster) and smoe_apply_ex
    on its kernel shard -- with CUDA events after warm-up, L2 flushed between
    calls, for the first, a middle and the last band.  The collectives
    (reduce-scatter of K x Pk fp32, all-reduce of 4 doubles, all-gather of
    the parameters) cannot run on one GPU: their time is modelled as ring
    transfers at 900 GB/s per direction plus 10 us latency each, and stated
    as a model, not a measurement."""
    import torch
    from paper_2510_05814_b200 import smoe, synth
    from paper_2510_05814_b200.dist import band_rows, shard_rows
    cfg = dict(synth.CONFIGS[args.config])
    C, H, W, K, order = cfg["C"], cfg["H"], cfg["W"], cfg["K"], cfg["order"]
    target, _, pool = synth.workload(args.config)
    dev = torch.device("cuda", 0)
    tgt = torch.as_tensor(target).to(dev)
    params = smoe.Params.from_numpy(pool, dev)
    flush = L2Flush(dev)
    ny = (H + 15) // 16
    E = 1 + 2 * order
    Pk = 6 + C * E
    out = {"metric": "per-rank step projection", "config": config_dict(args.config, 1), "ranks": {}}

    def timed(fn, n):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for i in range(n):
            flush()
            ev[i][0].record()
            fn()
            ev[i][1].record()
        torch.cuda.synchronize()
        return sorted(a.elapsed_time(b) for a, b in ev)[n // 2]

    for N in [int(x) for x in args.project.split(",")]:
        rows = {}
        k0, k1, Ks = shard_rows(K, 0, N)
        grad_sh = torch.zeros((k1 - k0, Pk), dtype=torch.float32, device=dev)
        for r in sorted({0, N // 2, N - 1}):
            b0, b1 = band_rows(ny, r, N)
            h = smoe.SMoE(K, H, W, C, order)
            if N > 1:
                h.set_band(b0, b1)
            g = torch.empty((K, Pk), dtype=torch.float32, device=dev)
            sums = torch.empty(4, dtype=torch.float64, device=dev)
            for _ in range(args.warmup):
                h.grad(params, tgt, g, sums)
            grad_ms = timed(lambda: h.grad(params, tgt, g, sums), args.steps)
            p2 = params.clone()
            apply_ms = timed(lambda: h.apply(p2, grad_sh, smoe.LR(0, 0, 0, 0, 0), k0, k1), args.steps)
            rows[f"rank{r}"] = {"band_rows": [b0, b1], "grad_ms": grad_ms, "apply_ms": apply_ms,
                                "pairs": h.sync().pairs}
            h.close()
        bytes_rs = K * Pk * 4
        bytes_ag = K * Pk * 4
        comm_ms = 0.0 if N == 1 else (2 * (N - 1) / N * (bytes_rs + bytes_ag) / 2 / 900e9 * 1e3 + 3 * 0.010)
        worst = max(v["grad_ms"] + v["apply_ms"] for v in rows.values())
        out["ranks"][N] = {"per_band": rows, "worst_rank_compute_ms": worst, "comm_model_ms": comm_ms,
                           "projected_ms_per_step": worst + comm_ms,
                           "projected_it_s": 1e3 / (worst + comm_ms)}
    print(json.dumps(out))
    return 0


def config_dict(name, world):
    from paper_2510_05814_b200 import synth
    c = synth.CONFIGS[name]
    return {"workload": f"config{c['cfg']}-{name}", "H": c["H"], "W": c["W"], "C": c["C"], "K": c["K"],
            "expert_order": c["order"], "fit_iterations": c["iters"],
            "parallelism": f"tile-row bands x{world}" if world > 1 else "single GPU",
            "l2": "flushed between timed steps (256 MB write, then 256 MB read: the step starts cold and clean)"}


class L2Flush:
    """Evict L2 between timed steps: write a 256 MB buffer (twice the 126 MB
    L2), then read another one, so the timed step starts with none of its
    data cached and without the flush's own dirty lines still waiting to be
    written back (which would otherwise land inside the timed region)."""

    def __init__(self, dev):
        import torch
        self.w = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
        self.r = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dev)
        self.s = torch.empty((), dtype=torch.float32, device=dev)

    def __call__(self):
        import torch
        self.w.zero_()
        torch.sum(self.r, dim=0, out=self.s)


def e2e_banded(fit, params, target, T_total, steps, dev):
    """e2e at N>1 through the public API (BandedFit.step with a pinned HOST
    target): each rank's smoe_grad copies only its band's pixel rows to the
    device (double-buffered copy stream), the gradient and loss partials are
    all-reduced, and every step's loss partials come back to pinned host
    memory (read two steps later).  Wall time per rank, max over ranks."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2510_05814_b200 import smoe
    host_t = torch.as_tensor(target).pin_memory()
    n = min(steps, 500)
    ring = torch.empty((4, 4), dtype=torch.float64).pin_memory()
    evs = [torch.cuda.Event() for _ in range(4)]
    lag, losses = 2, []
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for i in range(n):
        sums = fit.step(params, host_t, smoe.LR.paper(T_total, T_total))
        ring[i % 4].copy_(sums, non_blocking=True)
        evs[i % 4].record()
        if i >= lag:
            evs[(i - lag) % 4].synchronize()
            losses.append(float(ring[(i - lag) % 4][0]))
    torch.cuda.synchronize()
    for i in range(max(0, n - lag), n):
        losses.append(float(ring[i % 4][0]))
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    assert len(losses) == n and all(np.isfinite(losses))
    r0, r1 = fit.band
    return {"value": n / float(dt.item()), "unit": "it/s", "h2d_bytes_per_step": int(target.nbytes),
            "d2h_bytes_per_step": 32 * fit.world, "steps": n,
            "note": "each rank: pinned H2D of its band's target rows (double-buffered copy stream), gradient reduce-scatter + "
                    "loss all-reduce + sharded Adam + parameter all-gather, async D2H of the reduced loss partials; "
                    "bytes summed over ranks, time max over ranks"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)   # the config's 2000-iteration fit
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="div2k", choices=["tiny", "kodak", "div2k", "denoise", "8k"])
    ap.add_argument("--cpu-rows", type=int, default=0,
                    help="image rows of the cpu_baseline sample (0: about 15 s of oracle work, from the measured "
                         "~12 ns per (pixel, kernel) of the dense fp64 loss + gradient)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="N>1 process group; gloo (CUDA tensors) lets several ranks share one GPU in tests")
    ap.add_argument("--K", type=int, default=0, help="override the config's kernel count (density sweeps; not a bench line)")
    ap.add_argument("--backward-mode", type=int, default=-1, help="-1 auto (default), 0 pixel-parallel, 1 kernel-parallel")
    ap.add_argument("--no-profile", action="store_true", help="no per-kernel events in the timed region")
    ap.add_argument("--seg", type=float, default=0.0,
                    help="with --mm: segmentation-guided init (SURVEY f4) at this threshold (0-255 scale)")
    ap.add_argument("--mm", type=int, default=0,
                    help="MM-RSMoE (SURVEY f3): fit this many hypotheses concurrently and report the fused denoising")
    ap.add_argument("--box-modes", action="store_true",
                    help="after the fit: list pairs and time the gradient pass under each box mode (reading Q4)")
    ap.add_argument("--project", default="",
                    help="comma-separated rank counts: per-rank projection of the banded fit on one GPU")
    args = ap.parse_args()
    assert args.warmup >= 3, "at least 3 warm-up steps"
    if args.project:
        return run_project(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.mm:
        return run_mm(args)

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2510_05814_b200 import smoe, synth
    from paper_2510_05814_b200.dist import BandedFit, padded

    rank, world, local = rank_env()
    local = local % torch.cuda.device_count()       # ranks may share a GPU under --dist-backend gloo
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    cfg = dict(synth.CONFIGS[args.config])
    if args.K > 0:
        cfg["K"] = args.K
    C, H, W, K, order = cfg["C"], cfg["H"], cfg["W"], cfg["K"], cfg["order"]
    target, _, pool = synth.workload(args.config, args.K)
    dev = torch.device("cuda", local)
    tgt = torch.as_tensor(target).to(dev)
    params = smoe.Params.from_numpy(pool, dev)
    if world > 1:
        params = padded(params, world)       # in-place parameter all-gather needs Kpad rows
    h = smoe.SMoE(K, H, W, C, order, device=local, backward_mode=args.backward_mode)
    fit = BandedFit(h, rank, world) if world > 1 else None
    # the learning-rate schedule spans the config's fit; the timed
    # steps are its first ones, the rest of the fit runs untimed before the
    # render so the render is timed on the fitted model
    T_total = max(args.warmup + args.steps, cfg["iters"])

    def step(t):
        lr = smoe.LR.paper(t, T_total)
        if fit is None:
            h.step(params, tgt, lr, stats=False)
        else:
            fit.step(params, tgt, lr)

    flush = None if args.no_flush else L2Flush(dev)
    st0 = h.step(params.clone(), tgt, smoe.LR(0, 0, 0, 0, 0), stats=True)   # calibrate capacity
    if world > 1:
        h.grad(params, tgt)                  # calibrate the band's own lists
    h.reset_adam()
    for t in range(args.warmup):
        step(t)
    h.sync()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    launches0 = h.launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    for i in range(args.steps):
        if flush is not None:
            flush()
        ev[i][0].record()
        step(args.warmup + i)
        ev[i][1].record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = h.launch_count() - launches0
    clk = clocks.stop()
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    tms = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tms, op=dist.ReduceOp.MAX)
    total_ms = float(tms.item())

    # second timed region, same steps: CUDA event pairs (graph event nodes on
    # the launch stream) around the dominant kernel, for its roofline; kept
    # out of the headline region because event nodes cost ~10 us per step
    t_last = args.warmup + args.steps - 1
    ktimes, tested, hits, n_prof = {}, 0, 0, 0
    sort_cycles = cta_cycles = 0
    if not args.no_profile:
        n_prof = min(args.steps, 200)
        h.profile_begin(n_prof + 16, kernels=["k_raster<train>"])
        torch.cuda.synchronize()
        for i in range(n_prof):
            if flush is not None:
                flush()
            step(t_last)
        ktimes, _ = h.profile_end()

    st = h.sync()
    ms_step = total_ms / args.steps
    value = 1e3 / ms_step   # whole-image fit iterations per second (all ranks together)

    # per-kernel breakdown: a separate, shorter profiled pass (events around
    # every launch), reported for context only
    breakdown = None
    if not args.no_profile:
        nb = min(args.steps, 100)
        h.profile_begin(nb * 8 + 16, count_work=True)
        torch.cuda.synchronize()
        for i in range(nb):
            if flush is not None:
                flush()
            step(t_last)
        bt, (tested, hits) = h.profile_end()
        sort_cycles, cta_cycles = h.last_work[2], h.last_work[3]
        breakdown = {k: v[0] / nb for k, v in bt.items()}
        tested, hits = tested / nb, hits / nb        # per raster launch

    # the rest of the config's fit, untimed (the render below is timed on the
    # fitted model)
    for t in range(args.warmup + args.steps, T_total):
        step(t)
    st_fit = h.sync()

    # box modes (reading Q4) on the fitted pool: pairs listed and the train
    # raster's time per mode (pixels and gradients are mode-independent)
    box_modes = None
    if args.box_modes and world == 1:
        box_modes = {}
        gm = torch.empty((K, 6 + C * (1 + 2 * order)), dtype=torch.float32, device=dev)
        sm = torch.empty(4, dtype=torch.float64, device=dev)
        for mode in ("square", "aabb", "exact"):
            hm = smoe.SMoE(K, H, W, C, order, device=local, box_mode=mode)
            for _ in range(3):
                hm.grad(params, tgt, gm, sm)
            n = min(args.steps, 100)
            hm.profile_begin(8 * n + 16)
            for _ in range(n):
                if flush is not None:
                    flush()
                hm.grad(params, tgt, gm, sm)
            kt, _ = hm.profile_end()
            stm = hm.sync()
            box_modes[mode] = {"pairs": stm.pairs, "avg_kernels_per_block": stm.pairs / max(stm.n_tiles, 1),
                               "kernel_ms": {k2: v[0] / v[1] for k2, v in kt.items()},
                               "grad_ms": sum(v[0] for v in kt.values()) / n}
            hm.close()

    # roofline of the dominant kernel (raster: FP32 pipe)
    peaks, peak_kind = load_peaks()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    a_t, a_h = ops_per_unit(C, order)
    roof = None
    kernels = {}
    rast = ktimes.get("k_raster<train>")
    if breakdown:
        # per-kernel rooflines: the raster against the FP32
        # lanes and the MUFU (ex2: one per hit pair forward, one backward;
        # 16 MUFU lanes per SM per clock), binning and Adam against HBM
        # with their algorithmic bytes per launch
        E = 1 + 2 * order
        Pk, RSb = 6 + C * E, ((6 + C * E + 3) // 4) * 16
        V = 8 if Pk <= 8 else 16
        hbm = peaks.get("hbm_gbs", 6554.2)
        pairs = st.pairs
        two = "k_emit" in breakdown
        pre_bytes = K * (4 * Pk + 16 + RSb) + (0 if two else 4 * pairs)
        emit_bytes = K * (4 + 16) + 4 * pairs
        # fused records: with the two-stage binning the Adam
        # also writes the next step's tile box and record (no k_records launch)
        fused = two and "k_preprocess" not in breakdown
        Vu = 4 * ((Pk + 3) // 4)                 # raw-sum slots read + zeroed (the used float4 chunks)
        adam_bytes = K * (24 * Pk + 8 * Vu) + (K * (16 + RSb) if fused else 0)
        for name, b, what in (("k_preprocess", pre_bytes, f"read params {4 * Pk} B + write tile box 16 B + record "
                                                        f"{RSb} B per kernel" + ("" if two else ", + 4 B kernel id per "
                                                        "pair (count atomics are L2 traffic, not counted)")),
                              ("k_emit", emit_bytes, "read the spatial order 4 B + tile box 16 B per kernel, write "
                                                     "4 B kernel id per pair (one count atomic per CTA and block)"),
                              ("k_adam", adam_bytes, f"per kernel: params, m1, m2 read + write ({24 * Pk} B), raw "
                                                     f"sums read + zeroed ({8 * Vu} B)" +
                                                     (f", next step's tile box + record written ({16 + RSb} B)"
                                                      if fused else ""))):
            if name in breakdown and breakdown[name] > 0:
                gbs = b / (breakdown[name] * 1e-3) / 1e9
                kernels[name] = {"bound": "hbm", "bytes_per_launch": b, "avg_ms": breakdown[name],
                                 "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm, "bytes_note": what}
    if rast:
        r_ms, r_n = rast
        ops = a_t * tested + a_h * hits          # per launch (counted in the breakdown pass)
        achieved = ops / (r_ms / r_n * 1e-3) / 1e12
        peak = 148 * 128 * sm_mhz * 1e6 / 1e12
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_raster_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(f"{args.config}", {}).get("dram_bytes_per_launch")
            except Exception:
                traffic = None
        roof = {"bound": "alu", "kernel": "k_raster<train>", "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak, "traffic": traffic,
                "ops_note": f"FP32 lane-ops (FMA=1): {a_t}/tested pair + {a_h}/hit pair; peak = 148 SM x 128 "
                            f"lanes x {sm_mhz:.0f} MHz ({peak_kind} sm_max_mhz)",
                "tested_pairs_per_launch": tested, "hit_pairs_per_launch": hits,
                "avg_ms": r_ms / r_n, "share_of_step": (r_ms / r_n) / ms_step if world == 1 else None,
                "timed_region": f"second pass of {n_prof} steps with event pairs around the raster"}
        mufu_peak = 148 * 16 * sm_mhz * 1e6 / 1e12
        mufu = 2 * hits / (r_ms / r_n * 1e-3) / 1e12
        kernels["k_raster<train>"] = {
            "bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "mufu": {"achieved": mufu, "peak": mufu_peak, "unit": "Tex2/s", "frac": mufu / mufu_peak,
                     "note": "ex2 per hit pair: 1 forward + 1 backward; peak 16 MUFU lanes/SM/clk"},
            "sort_share": (sort_cycles / cta_cycles) if cta_cycles else None,
            "sort_note": "a4 in-raster bucket sort: SM cycles of the raster CTAs spent sorting / all their cycles"}

    # render (a9): plain reconstruction and the config's SR factor
    render = {}
    if rank == 0:
        sr = cfg.get("sr", 1)
        for s in sorted({1, sr}):
            oH, oW = H * s, W * s
            out = torch.empty((C, oH, oW), dtype=torch.float32, device=dev)
            h.render(params, oH, oW, out)
            torch.cuda.synchronize()
            reps = 20
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            rt = 0.0
            for _ in range(reps):
                if flush is not None:
                    flush()
                e0.record()
                h.render(params, oH, oW, out)
                e1.record()
                torch.cuda.synchronize()
                rt += e0.elapsed_time(e1)
            h.sync()
            # work counts of one render (device counters) for its roofline
            h.profile_begin(4, kernels=["k_raster<render>"], count_work=True)
            h.render(params, oH, oW, out)
            rk, (r_tested, r_hit) = h.profile_end()
            a_f = 2 + C + 2 * C * order
            peak = 148 * 128 * load_peaks()[0].get("sm_max_mhz", 1965.0) * 1e6 / 1e12
            rast_ms = rk.get("k_raster<render>", (rt / reps, 1))
            ach = (7 * r_tested + a_f * r_hit) / (rast_ms[0] / rast_ms[1] * 1e-3) / 1e12
            render[f"x{s}"] = {"mpix_s": oH * oW * reps / (rt * 1e-3) / 1e6, "ms": rt / reps, "out": [oH, oW],
                               "raster_roofline": {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                                                   "frac": ach / peak, "tested_pairs": r_tested, "hit_pairs": r_hit,
                                                   "ops_note": f"7/tested + {a_f}/hit FP32 lane-ops"}}

    # e2e through the public API: every step copies its target from pinned
    # host memory (the library double-buffers it on a copy stream, so the
    # H2D of step t+1 overlaps the compute of step t) and reads its loss/PSNR
    # back (smoe_stats_async into a pinned ring, consumed two steps later)
    e2e = None
    if not args.no_e2e and world > 1:
        e2e = e2e_banded(fit, params, target, T_total, args.steps, dev)
    if not args.no_e2e and world == 1:
        host_t = torch.as_tensor(target).pin_memory()
        n_e2e = min(args.steps, 500)
        ring = torch.empty(4 * 32, dtype=torch.uint8).pin_memory()       # 4 x smoe_raw_stats
        evs = [torch.cuda.Event() for _ in range(4)]
        lag, losses = 2, []
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(n_e2e):
            h.step(params, host_t, smoe.LR.paper(T_total, T_total), stats=False)
            h.stats_async(ring.data_ptr() + 32 * (i % 4))
            evs[i % 4].record()
            if i >= lag:
                evs[(i - lag) % 4].synchronize()
                losses.append(h.stats_from_raw(ring.data_ptr() + 32 * ((i - lag) % 4)).loss)
        torch.cuda.synchronize()
        for i in range(max(0, n_e2e - lag), n_e2e):
            losses.append(h.stats_from_raw(ring.data_ptr() + 32 * (i % 4)).loss)
        dt = time.perf_counter() - t0
        assert len(losses) == n_e2e and all(np.isfinite(losses))
        e2e = {"value": n_e2e / dt, "unit": "it/s", "h2d_bytes_per_step": int(target.nbytes),
               "d2h_bytes_per_step": 32, "steps": n_e2e,
               "note": "pinned H2D of the target each step (double-buffered copy stream) + async D2H of the step's loss"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        rows = args.cpu_rows or int(round(15.0 / (W * K * 1.2e-8)))
        rows = max(1, min(rows, H))
        r0 = (H - rows) // 2
        tg, ta, core = cpu_oracle_sample(target, pool, (r0, r0 + rows))
        cpu = dict({"value": 1.0 / (tg * H / rows + ta), "unit": "it/s", "cores": 1, "kind": "oracle",
                    "sample": f"dense fp64 loss+gradient on image rows {r0}-{r0 + rows} of {H} ({rows * W} px x "
                              f"{K} kernels, {tg:.1f} s) + full Adam ({ta:.3f} s), extrapolated to one iteration",
                    "pinned_core": core}, **cpu_info())

    if rank == 0:
        out = {
            "metric": "SMoE fit iterations/s", "value": value, "unit": "it/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(config_dict(args.config, world), **({"K": K, "K_override": True} if args.K else {})),
            "render": render, "roofline": roof, "kernel_rooflines": kernels, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk, **({"box_modes_on_fitted_pool": box_modes} if box_modes else {}),
            "kernel_ms_per_step": breakdown,
            "fit_stats": {"pairs": st.pairs, "avg_kernels_per_block": st.pairs / max(st.n_tiles, 1),
                          "loss": st.loss, "psnr_db": st.psnr_db, "initial_psnr_db": st0.psnr_db,
                          "fit_iterations_before_render": T_total,
                          "final_pairs": st_fit.pairs, "final_psnr_db": st_fit.psnr_db},
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
