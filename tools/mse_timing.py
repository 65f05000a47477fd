"""C5 predict + kriging MSE (n=8192, d=10, N=1M) wall time, repeated: the first call grows the
model's scratch (extension tiles) from the device pool, later calls reuse it."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

n, d, N = 8192, 10, 1_000_000
rng = np.random.default_rng(0)
X = np.empty((n, d))
for k in range(d):
    X[:, k] = (rng.permutation(n) + rng.random(n)) / n
y = (np.sin(3 * X + 0.37 * np.arange(d)) + 0.5 * X * X).sum(1)
m = g.model_at_theta(g.new_dataset(X, y), np.full(d, 2.0), 1.95, 0.0, g.Backend(g.Context(0)))
Xt = rng.random((N, d))
out = []
for i in range(3):
    t = time.perf_counter()
    g.predict(m, Xt, with_mse=True)
    out.append(time.perf_counter() - t)
print(sys.argv[1] if len(sys.argv) > 1 else ".", "predict+MSE wall (s):", [round(v, 3) for v in out], flush=True)
