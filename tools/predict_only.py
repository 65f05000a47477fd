"""One C5 predict (yhat only) for profiling: n=8192, d=10, N test points (default 200k)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g
n, d, N = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 10, 200000)))
rng = np.random.default_rng(0)
X = np.empty((n, d))
for k in range(d):
    X[:, k] = (rng.permutation(n) + rng.random(n)) / n
y = (np.sin(3 * X + 0.37 * np.arange(d)) + 0.5 * X * X).sum(1)
m = g.model_at_theta(g.new_dataset(X, y), np.full(d, 2.0), 1.95, 0.0, g.Backend(g.Context(0)))
yhat = g.predict(m, rng.random((N, d)))
print("ok", yhat[:3])
