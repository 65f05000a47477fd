#!/usr/bin/env python
"""Device time of one batch vs batch size B at a config (default C3: n=4096, d=10, p=1.95):
the per-GPU work of a GA generation of 100 sharded over N GPUs is ceil(100/N) candidates, so
this projects the strong-scaling curve bench.py measures under torchrun (N = 1, 2, 4, 8 ->
B = 100, 50, 25, 13). Same inputs as bench.py (random LHD, smooth_response, LHS thetas).

  python tools/batch_sweep.py [n] [d] [B ...]
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_1203_1269_b200.gpemu as g
    from bench import lhs_thetas, random_lhd, smooth_response
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    Bs = [int(b) for b in sys.argv[3:]] or [100, 50, 25, 13, 8, 4, 1]
    rng = np.random.default_rng(20120306)
    X = random_lhd(n, d, rng)
    y = smooth_response(X)
    th = lhs_thetas(d, 100, np.random.default_rng(20120306 + 1000))
    dev = torch.device("cuda", 0)
    ctx = g.Context(0)
    stream = torch.cuda.current_stream(dev)
    ctx.set_stream(stream.cuda_stream)
    be = g.Backend(ctx)
    data = g.new_dataset(X, y)
    out = {}
    for B in Bs:
        ev = g.ProfileEvaluator(data, 1.95, 0.0, be, max_batch=B)
        dth = torch.from_numpy(np.ascontiguousarray(th[:B])).to(dev)
        do = torch.empty(B * 8, dtype=torch.float64, device=dev)
        for _ in range(3):
            ev.eval_batch_device(dth.data_ptr(), B, do.data_ptr())
        reps = max(3, min(20, 400 // B))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(reps):
            ev.eval_batch_device(dth.data_ptr(), B, do.data_ptr())
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1) / reps
        out[B] = {"ms": ms, "evals_per_s": B / (ms / 1e3), "tflops": B * n ** 3 / 3 / (ms / 1e3) / 1e12}
        print(f"n={n} d={d} B={B}: {ms:.3f} ms/batch, {B / (ms / 1e3):.1f} evals/s, "
              f"{out[B]['tflops']:.2f} TF/s (step, n^3/3 per candidate)", flush=True)
        ev.close()
    if 100 in out:
        for N, B in ((2, 50), (4, 25), (8, 13)):
            if B in out:
                v = 100 / (out[B]["ms"] / 1e3)
                print(f"projected strong scaling N={N}: {v:.0f} evals/s, efficiency "
                      f"{v / (N * out[100]['evals_per_s']):.3f}")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
