"""C5 probe: model at a fixed theta on n=8192, d=10, then predict + MSE on N test points."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g
n, d, N = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 10, 1000000)))
rng = np.random.default_rng(0)
X = np.empty((n, d))
for k in range(d):
    X[:, k] = (rng.permutation(n) + rng.random(n)) / n
y = (np.sin(3 * X + 0.37 * np.arange(d)) + 0.5 * X * X).sum(1)
ctx = g.Context(0)
be = g.Backend(ctx)
t = time.time()
m = g.model_at_theta(g.new_dataset(X, y), np.full(d, 2.0), 1.95, 0.0, be)
print(f"model_at_theta n={n}: {time.time()-t:.2f} s (neg2 {m.neg2_log_lik:.6f})", flush=True)
Xt = rng.random((N, d))
for it in range(2):
    t = time.time(); yhat = g.predict(m, Xt); t1 = time.time() - t
    t = time.time(); yhat2, mse = g.predict(m, Xt, with_mse=True); t2 = time.time() - t
    print(f"N={N}: yhat {t1:.3f} s ({N/t1:.0f} pts/s); yhat+mse {t2:.3f} s ({N/t2:.0f} pts/s); "
          f"mse range [{mse.min():.3e}, {mse.max():.3e}] same-yhat={np.array_equal(yhat, yhat2)}", flush=True)
