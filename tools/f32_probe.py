"""Single-precision engine probe: the device float path vs the reference's float and double
instantiations on a few thetas (n d B p), plus C3-size timing of both device precisions."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g  # noqa: E402
from oracle.oracle import RefLib, ref_available  # noqa: E402

n, d, B = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (700, 3, 8)))
p = float(sys.argv[4]) if len(sys.argv) > 4 else 1.95
rng = np.random.default_rng(4)
X = rng.random((n, d))
y = np.sin(3 * X).sum(1) + 0.3 * X[:, 0]
th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
ctx = g.Context(0)
be = g.Backend(ctx)
evs = g.ProfileEvaluator(g.new_dataset(X, y), p, 0.0, be, max_batch=B, precision="single")
evd = g.ProfileEvaluator(g.new_dataset(X, y), p, 0.0, be, max_batch=B)
rs, rd = evs.eval_batch(th), evd.eval_batch(th)
print("device single neg2", rs["neg2"][:4], "jitter", rs["jitter"][:4])
print("device double neg2", rd["neg2"][:4])
if ref_available(True) and n <= 4096:
    ref = RefLib(fast=True)
    fs = ref.eval_batch(X, y, th, p, threads=0, precision="single")
    fd = ref.eval_batch(X, y, th, p, threads=0)
    rel = lambda a, b: np.abs(a - b) / np.abs(b)  # noqa: E731
    print("ref single vs ref double rel", rel(fs["neg2"], fd["neg2"]))
    print("dev single vs ref single rel", rel(rs["neg2"], fs["neg2"]))
    print("dev single vs ref double rel", rel(rs["neg2"], fd["neg2"]))
    print("dev double vs ref double rel", rel(rd["neg2"], fd["neg2"]))
    print("jitter ref single", fs["jitter"], "dev single", rs["jitter"])
for name, ev in (("single", evs), ("double", evd)):
    ev.eval_batch(th)
    torch.cuda.synchronize()
    t = time.time()
    for _ in range(3):
        ev.eval_batch(th)
    dt = (time.time() - t) / 3
    print(f"{name}: {B / dt:.1f} evals/s ({dt * 1e3:.2f} ms per batch of {B})")
