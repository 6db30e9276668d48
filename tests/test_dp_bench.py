"""GPU: the row-sharded data-parallel bench path (torchrun, 2 ranks). On the
one-GPU test box both ranks share cuda:0 and the dW all-reduce goes through
gloo; on an 8-GPU node the same code path runs over NCCL."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
def test_bench_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--size", "1024", "--no-sweep", "--no-e2e", "--no-cpu",
           "--dist-backend", "gloo", "--preroll", "0", "--config", "cfg2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env={**os.environ, "OMP_NUM_THREADS": "2"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["scaling"] == "weak"
    assert d["config"]["M_global"] == 2048
    # mask, forward, 2 dW row slabs (all-reduced one by one), dX: 5 launches per step
    assert d["gpu_launches"] == 5 * 3


@pytest.mark.gpu
def test_bench_cfg5_two_ranks_strong():
    """configs[4] mode (row-sharded strong scaling) at reduced size: 2 ranks on one
    GPU over gloo print ONE configs[4]-named line from rank 0."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), str(ROOT / "bench.py"), "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--config", "cfg5", "--m-global", "8192", "--kn", "1024",
           "--dist-backend", "gloo", "--preroll", "0"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env={**os.environ, "OMP_NUM_THREADS": "2"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["config"]["workload"].startswith("configs[4]")
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["M_global"] == 8192 and d["config"]["M_per_gpu"] == 4096
    assert d["gpu_launches"] == 4 * 3  # mask, forward, dW (one all-reduce, --dw-parts 1 default), dX
    assert d["comm"]["allreduce_ms"] > 0 and d["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.gpu
def test_bench_cfg5_single_gpu_reduced():
    """configs[4] at G=1 (the strong-scaling baseline), reduced size."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3", "--config", "cfg5",
           "--m-global", "16384", "--kn", "1024", "--preroll", "0"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["scaling"] == "strong" and d["n_gpus"] == 1 and d["config"]["M_global"] == 16384
