"""A GA fit whose population does not fit in HBM: n (default 24000) design points, the plan sized
by fit_batch (free device memory), each generation evaluated in chunks. Prints the chosen
max_batch, the plan bytes and the wall time per generation."""
import sys
import time

import numpy as np

sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 10
gens = int(sys.argv[3]) if len(sys.argv) > 3 else 1
rng = np.random.default_rng(1)
X = np.empty((n, d))
for k in range(d):
    X[:, k] = (rng.permutation(n) + rng.random(n)) / n
y = (np.sin(3.0 * X + 0.37 * np.arange(d)) + 0.5 * X * X).sum(1)
ctx = g.Context(0)
be = g.Backend(ctx)
data = g.new_dataset(X, y)
cfg = g.FitConfig(ga=g.GaConfig(population=100, generations=gens), seed=0, p=1.95)
mb = g.fit_batch(data, cfg, be)
print(f"n={n} d={d}: max_batch {mb} of 100, plan {g.lib().gpemu_plan_bytes(n, d, mb, 0) / 1e9:.1f} GB "
      f"(a 100-slot plan would need {g.lib().gpemu_plan_bytes(n, d, 100, 0) / 1e9:.1f} GB)", flush=True)
t = time.time()
fr = g.fit_gp_detailed(data, cfg, be)
dt = time.time() - t
print(f"fit {100 * gens} evals in {dt:.1f} s ({100 * gens / dt:.2f} evals/s), neg2 {fr.model.neg2_log_lik:.6f}")
