"""Host-side breakdown of one C5 predict call (n=8192, d=10, N=1M): wall time of the C-ABI
call vs the predict kernels' device time (ncu launch list), plus pageable vs pinned input."""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g
n, d, N = 8192, 10, 1_000_000
rng = np.random.default_rng(0)
X = np.empty((n, d))
for k in range(d):
    X[:, k] = (rng.permutation(n) + rng.random(n)) / n
y = (np.sin(3 * X + 0.37 * np.arange(d)) + 0.5 * X * X).sum(1)
m = g.model_at_theta(g.new_dataset(X, y), np.full(d, 2.0), 1.95, 0.0, g.Backend(g.Context(0)))
Xt = rng.random((N, d))
pinned = torch.from_numpy(Xt).pin_memory().numpy()
for label, arr in (("pageable", Xt), ("pinned", pinned), ("pageable", Xt)):
    t = time.perf_counter(); g.predict(m, arr); dt = time.perf_counter() - t
    print(f"{label}: predict wall {dt:.3f} s", flush=True)
t = time.perf_counter(); g.predict(m, Xt[:1000]); print(f"N=1000 wall {time.perf_counter()-t:.4f} s")
