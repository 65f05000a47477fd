"""GPU: the multi-rank entry points under torchrun + NCCL (one rank: the pool gives one GPU).

Covers bench.py's distributed path (barrier, max-over-ranks all-reduce, per-rank batches) and
the sharded GA fit driver (per-generation NCCL all-gather); multi-rank host logic with real
rank counts is covered on CPU by tests/test_sharded.py (gloo, world 2 and 3)."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)


@pytest.mark.gpu
def test_bench_under_torchrun_nccl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    r = _torchrun(["bench.py", "--gpus", "1", "--steps", "3", "--warmup", "3", "--size", "1024",
                   "--dims", "4", "--batch", "32", "--no-fit", "--no-cpu-baseline"])
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["candidates_ok"] == 32
    assert line["roofline"]["frac"] > 0 and line["e2e"]["value"] > 0
    assert line["gpu_launches"] > 0


@pytest.mark.gpu
def test_sharded_fit_under_torchrun_nccl():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    r = _torchrun(["tools/sharded_fit.py", "512", "3", "16", "3"])
    assert r.returncode == 0, r.stderr[-3000:]
    assert "sharded fit n=512" in r.stdout
