"""First-batch overhead of the ticket-order list schedule (built on the host once per batch
size): wall time of the first vs the second eval_batch at C3 and C4 shapes."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

for n, d, B in ((4096, 10, 100), (16384, 20, 100)):
    rng = np.random.default_rng(0)
    X = rng.random((n, d))
    y = np.sin(3 * X).sum(1)
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.9, 1e-8, g.Backend(g.Context(0)), max_batch=B)
    th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
    ts = []
    for _ in range(2):
        t = time.perf_counter()
        ev.eval_batch(th)
        ts.append(time.perf_counter() - t)
    print(f"n={n} B={B} order={os.environ.get('GPEMU_TICKET_ORDER', '1')}: first {ts[0]:.3f} s, second {ts[1]:.3f} s", flush=True)
    ev.close()
