"""Bitwise A/B of two engine builds: the same C3-shaped batch through the working tree's library
and _ab/head's, comparing every record field exactly (run on the GPU box)."""
import subprocess
import sys

import numpy as np

CODE = r"""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_1203_1269_b200.gpemu as g
n, d, B = %d, %d, %d
rng = np.random.default_rng(1)
X = rng.random((n, d)); y = np.sin(3 * X).sum(1)
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(g.Context(0)), max_batch=B)
th = 10 ** rng.uniform(-1.5, 0.8, size=(B, d))
o = ev.eval_batch(th)
np.save(sys.argv[1], np.stack([o['neg2'], o['mu'], o['sigma2'], o['jitter'], o['log_det']]))
"""
shape = tuple(int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (4096, 10, 40)
for tree, out in ((".", "/tmp/ab_a.npy"), ("_ab/head", "/tmp/ab_b.npy")):
    subprocess.run([sys.executable, "-c", CODE % shape, out], cwd=tree, check=True)
a, b = np.load("/tmp/ab_a.npy"), np.load("/tmp/ab_b.npy")
same = np.array_equal(a.view(np.uint64), b.view(np.uint64))
print(f"shape {shape}: bitwise identical: {same}; max |rel diff| neg2 "
      f"{np.nanmax(np.abs(a[0] - b[0]) / np.abs(b[0])):.3e}")
