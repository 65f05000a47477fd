import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g
n, d, B = 4096, 10, 100
rng = np.random.default_rng(0)
X = rng.random((n, d)); y = np.sin(3 * X).sum(1)
ctx = g.Context(0, "dag")
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=B)
th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
ev.eval_batch(th)
ev.set_profiling(True)
for _ in range(3): ev.eval_batch(th)
print("assemble ms/step %.3f  chol %.3f  finalize %.3f" % tuple(ev.phase_ms(k)[0] / 3 for k in range(3)))
