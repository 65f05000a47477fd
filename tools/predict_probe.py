"""C5 probe: model at a fixed theta on n=8192, d=10, then predict (yhat) and predict+MSE on N
test points, `reps` times each; prints every wall time, the median, and SM clocks seen."""
import subprocess
import sys
import threading
import time

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

n, d, N = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 10, 1000000)))
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 5
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
clocks, stop = [], threading.Event()


def sample():
    while not stop.is_set():
        try:
            out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits",
                                  "-i", "0"], capture_output=True, text=True, timeout=5).stdout
            clocks.append(int(out.strip().splitlines()[0]))
        except Exception:
            pass
        time.sleep(0.2)


th = threading.Thread(target=sample, daemon=True)
th.start()
g.predict(m, Xt[:1000], with_mse=True)
ty, tm = [], []
for it in range(reps):
    t = time.perf_counter(); yhat = g.predict(m, Xt); ty.append(time.perf_counter() - t)
    t = time.perf_counter(); yhat2, mse = g.predict(m, Xt, with_mse=True); tm.append(time.perf_counter() - t)
stop.set()
print(f"N={N}: yhat s {[round(v, 3) for v in ty]} median {np.median(ty):.3f} ({N/np.median(ty):.0f} pts/s)")
print(f"N={N}: yhat+mse s {[round(v, 3) for v in tm]} median {np.median(tm):.3f} ({N/np.median(tm):.0f} pts/s)")
print(f"same-yhat={np.array_equal(yhat, yhat2)} mse range [{mse.min():.3e}, {mse.max():.3e}] "
      f"sm clocks MHz min/median/max {min(clocks, default=0)}/{int(np.median(clocks)) if clocks else 0}/{max(clocks, default=0)}")
