"""bench.py's N > 1 code path (the driver's scaling run launches it under
torchrun, one rank per GPU over NCCL), exercised functionally on one GPU:
two ranks over gloo sharing the device (SWMD_BENCH_BACKEND=gloo).  The
timings of such a run mean nothing; what is checked is that every rank gets
through the sharded solve, the gather, the c3 strong-scaling block and the
e2e path, and that rank 0 prints one contract line."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def _port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_rank_bench_line():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, SWMD_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(REPO, "bench.py"), "--gpus", "2", "--config", "c1", "--steps", "5",
           "--warmup", "3", "--no-c3"]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 5 and d["value"] > 0
    assert d["config"]["parallelism"] == "column shards x2"
