import sys, numpy as np, ctypes as C
sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g
n, d, B = 4096, 10, 100
rng = np.random.default_rng(0)
X = rng.random((n, d)); y = np.sin(3 * X).sum(1)
ctx = g.Context(0)
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=B)
th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
ev.eval_batch(th)
ev.dag_profile(True)
ev.eval_batch(th)
out = np.zeros(148 * 24 + 256, dtype=np.uint64)
g._check(g.lib().gpemu_plan_dag_profile(ev.handle, 0, out.ctypes.data, out.size))
per = out[:148*24].reshape(148, 24)
tot = per[:, 15].astype(float).sum()
off = out[148*24:148*24+128].astype(float); dg = out[148*24+128:148*24+256].astype(float)
print("total CTA cycles %.3e; flag-wait OFF %.2f%% DIAG %.2f%%" % (tot, 100*off.sum()/tot, 100*dg.sum()/tot))
for j in range(32):
    print(j, "%.2f%% %.2f%%" % (100*off[j]/tot, 100*dg[j]/tot))
