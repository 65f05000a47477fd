import sys
import os

import numpy as np

# tickets are decoded here with the kernel's built-in column order: keep the list-schedule table off
os.environ["GPEMU_TICKET_ORDER"] = "0"
sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g
n, d, B = 4096, 10, 100
rng = np.random.default_rng(0)
X = rng.random((n, d)); y = np.sin(3 * X).sum(1)
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(g.Context(0)), max_batch=B)
th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
ev.eval_batch(th); ev.dag_profile(True); ev.eval_batch(th)
p = ev.dag_profile(False, read=True)
noff = p["n_off"].sum(); ndiag = p["n_diag"].sum()
print("n_off", noff, "n_diag", ndiag)
for k, v in p.items():
    if k == "trace": continue
    s = float(v.sum())
    print(f"{k:12s} total {s:.4g}  per-OFF-task-us {s / noff / 1.9e3:.3f}  per-DIAG-us {s / max(ndiag,1) / 1.9e3:.3f}")
