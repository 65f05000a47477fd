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
                   "--dims", "4", "--batch", "32", "--no-fit", "--no-cpu-baseline", "--no-latency"])
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
    assert "bitwise equal to the unsharded prediction: True" in r.stdout


def _torchrun_n(n, args, env_extra, timeout=900):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(_port())] + args
    env = dict(os.environ, **env_extra)
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)


@pytest.mark.gpu
def test_bench_two_ranks_host_logic():
    """bench.py with world 2 (barriers, max-over-ranks time, rank-0 line; the strong-scaling
    value over the shared generation, the weak leg, the sharded GA fit): collectives on gloo and
    both ranks on the visible GPU (GPEMU_BENCH_DIST=gloo, test-only), since this pool gives one
    GPU; the ranks' candidate ranges are independent."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    r = _torchrun_n(2, ["bench.py", "--gpus", "2", "--steps", "3", "--warmup", "3", "--size", "768",
                        "--dims", "3", "--batch", "16", "--no-cpu-baseline", "--no-single"],
                    {"GPEMU_BENCH_DIST": "gloo"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 16 and line["config"]["batch_per_gpu"] == 8
    assert line["candidates_ok"] == 8
    assert abs(line["value"] - 16 * 3 / (line["ms_per_step"] * 3 / 1e3)) <= 1e-6 * line["value"]
    w = line["weak"]
    assert abs(w["value"] - 2 * 16 * 3 / (w["ms_per_step"] * 3 / 1e3)) <= 1e-6 * w["value"]
    assert line["e2e"]["value"] > 0
    assert line["fit"]["gpu_wall_s"] > 0 and line["fit"]["evals"] == 16 * 20
    r = _torchrun_n(2, ["bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "1",
                        "--size", "768", "--dims", "3", "--batch", "16"], {"GPEMU_BENCH_DIST": "gloo"})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["impl"] == "reference"
