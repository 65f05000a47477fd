"""Jitter-ladder use of the float and double engines on bench.py's C3 batches (GA LHS thetas over
[1e-6, 12]^10): how many candidates need a jitter step and how many Cholesky launches a batch
takes in each precision."""
import sys

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_1203_1269_b200.gpemu as g  # noqa: E402


class A:
    n, d, p, batch, seed, steps, warmup = 4096, 10, 1.95, 100, 20120306, 2, 1


X, y, batches = bench.make_inputs(A, 0)
ctx = g.Context(0)
be = g.Backend(ctx)
for prec in ("double", "single"):
    ev = g.ProfileEvaluator(g.new_dataset(X, y), A.p, 0.0, be, max_batch=A.batch, precision=prec)
    for b in batches[:2]:
        ev.set_profiling(True)
        r = ev.eval_batch(b)
        _, launches = g.lib(), None
        ms, nl = ev.phase_ms(1)
        ev.set_profiling(False)
        steps = np.unique(r["jitter"], return_counts=True)
        print(f"{prec}: chol launches {nl}, chol {ms:.1f} ms, jitter steps {dict(zip(steps[0].tolist(), steps[1].tolist()))}")
    ev.close()
