"""C1 batch (n=200, d=2, p=2, B=100): wall time vs device phases, and how many candidates
climb the jitter ladder (each step relaunches assemble + DAG for the failed ones)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

rng = np.random.default_rng(0)
n, d, B = 200, 2, 100
X = rng.random((n, d))
y = np.sin(3 * X).sum(1)
ctx = g.Context(0)
ev = g.ProfileEvaluator(g.new_dataset(X, y), 2.0, 0.0, g.Backend(ctx), max_batch=B)
gg = rng.random((B, d))
th = 10.0 ** (-6 + (np.log10(12.0) + 6) * gg)
ev.eval_batch(th)
ev.set_profiling(True)
l0 = ctx.launch_count
t = time.perf_counter()
for _ in range(20):
    r = ev.eval_batch(th)
wall = (time.perf_counter() - t) / 20
print(f"wall {wall * 1e3:.3f} ms per batch; launches per batch {(ctx.launch_count - l0) / 20:.1f}; "
      f"device (ms, launches) assemble {ev.phase_ms(0)} chol {ev.phase_ms(1)} finalize {ev.phase_ms(2)} over 20 batches; jitter steps {np.unique(r['jitter'], return_counts=True)}")
