"""Full-size C4 golden (n=16384, d=20, p=1.9, nugget 1e-8): the reference's ProfileEvaluator
on two thetas, from BOTH reference builds (oracle/_ref strict and native-flag), so the GPU
test can gate on the reference's own self-discrepancy. The design is a seeded numpy LHD (the
test regenerates it; only thetas and outputs are stored): tests/golden/c4_full.npz.
Runtime: ~4 x 50 s on 16 host threads."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import RefLib, build  # noqa: E402

N, D, P, NUG, SEED = 16384, 20, 1.9, 1e-8, 16384


def design(n=N, d=D, seed=SEED):
    rng = np.random.default_rng(seed)
    X = np.empty((n, d))
    for k in range(d):
        X[:, k] = (rng.permutation(n) + rng.random(n)) / n
    y = (np.sin(3.0 * X + 0.37 * np.arange(d)) + 0.5 * X * X).sum(1)
    return X, y


def main():
    build()
    X, y = design()
    thetas = np.array([np.full(D, 2.0), 10 ** np.linspace(-1.5, 0.8, D)])
    res = {}
    for name, fast in (("strict", False), ("fast", True)):
        ref = RefLib(fast=fast)
        t = time.time()
        r = ref.eval_batch(X, y, thetas, P, NUG, threads=os.cpu_count())
        print(name, time.time() - t, r["neg2"], r["jitter"], flush=True)
        res[name] = r
    np.savez(os.path.join(ROOT, "tests", "golden", "c4_full.npz"), seed=SEED, n=N, d=D, p=P, nugget=NUG,
             thetas=thetas, **{f"{k}_{b}": res[b][k] for b in res for k in ("neg2", "mu", "sigma2", "jitter", "log_det")})


if __name__ == "__main__":
    main()
