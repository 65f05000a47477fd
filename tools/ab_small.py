"""Chain-bound timings for A/B runs (run from a tree's root): one B=1 evaluation at n=4096 and
n=1024 (the refine / model path) and one B=100 batch at n=1024 (a paper-protocol GA generation),
device-resident, median of repeated CUDA-event-timed calls."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g  # noqa: E402


def timed(n, d, B, reps=30):
    rng = np.random.default_rng(3)
    X = rng.random((n, d))
    y = np.sin(3 * X).sum(1)
    ctx = g.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)  # the events below see the kernels
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=B)
    th = torch.tensor(10 ** rng.uniform(-1.0, 0.5, size=(B, d)), device="cuda")
    out = torch.empty((B, 8), dtype=torch.float64, device="cuda")
    ts = []
    for i in range(reps + 3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ev.eval_batch_device(th.data_ptr(), B, out.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


tag = sys.argv[1] if len(sys.argv) > 1 else "."
print(tag, {f"n{n}_B{B}": round(timed(n, d, B), 3) for n, d, B in ((4096, 10, 1), (1024, 6, 1), (1024, 6, 100), (2048, 6, 64))})
