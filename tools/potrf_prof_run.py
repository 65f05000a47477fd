import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g
n, d = 4096, 10
rng = np.random.default_rng(3)
X = rng.random((n, d)); y = np.sin(3 * X).sum(1)
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(g.Context(0)), max_batch=1)
print(ev.eval_batch(10 ** rng.uniform(-1.0, 0.5, size=(1, d)))["neg2"])
