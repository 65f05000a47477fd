"""C4 on the reference's CPU path (n=16384, d=20, p=1.9, nugget 1e-8): plan construction and
one ParallelBackend evaluation on every host thread (time >= 1 eval, extrapolate).
Needs ~26 GB of host memory (the reference's |d|^p table is 21 GB)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import RefLib  # noqa: E402

ref = RefLib(fast=True)
rng = np.random.default_rng(4)
n, d = 16384, 20
X = rng.random((n, d))
y = np.sin(3 * X).sum(1)
th = 10 ** rng.uniform(-1.0, 0.5, size=(2, d))
neg2, sp, se = ref.eval_batch_timed(X, y, th, 1.9, nugget=1e-8, backend="parallel", threads=0)
res = {"n": n, "d": d, "p": 1.9, "nugget": 1e-8, "evals": 2, "plan_s": sp, "evals_s": se,
       "evals_per_s": 2 / se, "neg2": list(map(float, neg2))}
print(json.dumps(res))
json.dump(res, open(os.path.join(ROOT, "gpurun_out", "cpu_reference_c4.json"), "w"), indent=1)
