#!/usr/bin/env python
"""Model build (model_at_theta: one B=1 evaluation + alpha) at config C5's n=8192, d=10 (or n
given), for ncu: the tile_trsv (alpha) and chol_dag launches. Prints the host-timed build.

  python tools/model_build_profile.py [n] [reps]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1203_1269_b200.gpemu as g  # noqa: E402
from bench import random_lhd, smooth_response  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    d = 10
    rng = np.random.default_rng(8192)
    X = random_lhd(n, d, rng)
    y = smooth_response(X)
    th = 10 ** rng.uniform(0.0, 0.6, d)
    be = g.Backend(g.Context(0))
    data = g.new_dataset(X, y)
    for r in range(reps):
        t = time.perf_counter()
        m = g.model_at_theta(data, th, 1.95, 0.0, be)
        dt = time.perf_counter() - t
        print(f"n={n} model_at_theta {1e3 * dt:.2f} ms (incl. plan creation), jitter {m.jitter_used}, "
              f"alpha residual {g.model_alpha_residual(m) if n <= 4096 else float('nan'):.2e}")
        m.close()


if __name__ == "__main__":
    main()
