"""maximin_lhd at the C4 design size (n=16384, d=20, budget 10000): the device path vs the
reference (oracle/_ref native build, one host thread -- the reference's design generation is
serial) on the GPU box; both designs are compared bitwise. usage: python tools/design_timing.py
[n d budget] [--no-ref]"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n, d, budget = (int(a) for a in args[:3]) if len(args) >= 3 else (16384, 20, 10000)
ctx = g.Context(0)
g.maximin_lhd(g.DesignSpec(256, d, 1, 100), ctx)  # warm-up (module load, pool)
t = time.perf_counter()
X, m = g.maximin_lhd(g.DesignSpec(n, d, 4, budget), ctx, return_min=True)
tg = time.perf_counter() - t
out = {"n": n, "d": d, "budget": budget, "gpu_s": tg, "min_sq_dist": m}
if "--no-ref" not in sys.argv:
    from oracle.oracle import RefLib
    t = time.perf_counter()
    R = RefLib(fast=True).maximin_lhd(n, d, 4, budget)
    out["ref_s"] = time.perf_counter() - t
    out["bitwise_equal"] = bool(np.array_equal(X, R))
print(json.dumps(out))
