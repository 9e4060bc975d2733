"""bench.py's N>1 path (tile-row bands, all-reduce, banded e2e) run under
torchrun with two ranks sharing the one visible B200 (gloo over CUDA tensors:
NCCL refuses two ranks on one device; the driver's multi-GPU runs use NCCL
through the same code).  Checks the JSON contract of the multi-rank line."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("config", ["tiny", "kodak"])
def test_bench_two_ranks_json_line(config):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--config", config, "--steps", "20", "--warmup", "3", "--no-cpu", "--dist-backend", "gloo"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 20 and d["warmup"] == 3
    assert d["config"]["parallelism"] == "tile-row bands x2"
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert d["gpu_launches"] > 0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] == 64
    assert d["fit_stats"]["loss"] == d["fit_stats"]["loss"]   # finite
