"""Per-phase cycle breakdown of the DAG engine on one C3 batch."""
import sys
import numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g
n, d, B = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 10, 100)))
rng = np.random.default_rng(0)
X = rng.random((n, d)); y = np.sin(3 * X).sum(1)
ctx = g.Context(0, "dag")
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=B)
th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
ev.eval_batch(th)
ev.dag_profile(True)
ev.eval_batch(th)
p = ev.dag_profile(False, read=True)
tot = p["total"].astype(float)
print(f"n={n} B={B}: ctas={int((tot>0).sum())} mean total cycles {tot[tot>0].mean():.3e} (max {tot.max():.3e})")
for k in g.ProfileEvaluator.DAG_PHASES:
    v = p[k].astype(float)
    if k in ("n_diag", "n_off", "slabs"):
        print(f"  {k:12s} sum {v.sum():.0f}  per-cta min/max {v.min():.0f}/{v.max():.0f}")
    elif k != "total":
        print(f"  {k:12s} {100*v.sum()/tot.sum():6.2f}%   per-task avg {v.sum()/max(1,(p['n_diag']+p['n_off']).sum()):.0f} cyc")
