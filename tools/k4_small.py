"""Short K1+K4 workload for ncu: one C3 batch assemble + C5-shaped predict/MSE on 65536 points."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g
rng = np.random.default_rng(0)
n, d = 8192, 10
X = np.empty((n, d))
for k in range(d):
    X[:, k] = (rng.permutation(n) + rng.random(n)) / n
y = (np.sin(3 * X + 0.37 * np.arange(d)) + 0.5 * X * X).sum(1)
ctx = g.Context(0)
m = g.model_at_theta(g.new_dataset(X, y), np.full(d, 2.0), 1.95, 0.0, g.Backend(ctx))
Xt = rng.random((65536, d))
yh = g.predict(m, Xt)
yh2, mse = g.predict(m, Xt, with_mse=True)
print("ok", yh[:2], mse[:2])
