"""One C3 evaluation alone (B=1, n=4096, d=10): the chain-bound chol_dag instantiation, for ncu
(`ncu -k regex:chol_dag --launch-skip 3 -c 1 python tools/b1_profile.py`). Prints the
event-timed evaluation."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

rng = np.random.default_rng(3)
n, d = 4096, 10
X = rng.random((n, d))
y = np.sin(3 * X).sum(1)
ctx = g.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=1)
th = torch.tensor(10 ** rng.uniform(-1.0, 0.5, size=(1, d)), device="cuda")
out = torch.empty((1, 8), dtype=torch.float64, device="cuda")
ts = []
for i in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    ev.eval_batch_device(th.data_ptr(), 1, out.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"B=1 evaluation at n={n}: {min(ts[1:]):.3f} ms")
