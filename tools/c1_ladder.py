#!/usr/bin/env python
"""Config C1 (n=200, d=2, p=2, Goldstein-Price log on the reference's maximin design; the 100
GA-style thetas of tests/golden/c1.npz, every one of which climbs to jitter 1e-8): evals/s of
a 100-candidate batch with the speculative first ladder rung (one pass) and without it
(GPEMU_SPEC_LADDER=0: jitter 0, then a second pass at 1e-8), and the C1 GA fit (100 x 20).

  python tools/c1_ladder.py
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1203_1269_b200.gpemu as g  # noqa: E402


def rate(ev, th, reps=50):
    ev.eval_batch(th)
    ev.eval_batch(th)
    t = time.perf_counter()
    for _ in range(reps):
        r = ev.eval_batch(th)
    dt = (time.perf_counter() - t) / reps
    return len(th) / dt, dt, r


def main():
    z = np.load(os.path.join(ROOT, "tests", "golden", "c1.npz"))
    data = g.new_dataset(z["X"], z["y"])
    out = {}
    for mode in ("speculative", "two_pass"):
        if mode == "two_pass":
            os.environ["GPEMU_SPEC_LADDER"] = "0"
        ctx = g.Context(0)
        be = g.Backend(ctx)
        ev = g.ProfileEvaluator(data, 2.0, 0.0, be, max_batch=100)
        l0 = ctx.launch_count
        v, dt, r = rate(ev, z["thetas"])
        launches = (ctx.launch_count - l0) / 52
        cfg = g.FitConfig(ga=g.GaConfig(population=100, generations=20), seed=0, p=2.0)
        g.fit_gp_detailed(data, cfg, be)
        t = time.perf_counter()
        fr = g.fit_gp_detailed(data, cfg, be)
        fit_s = time.perf_counter() - t
        assert np.array_equal(np.array(fr.model.params.theta), z["fit_theta"])
        out[mode] = {"evals_per_s": v, "ms_per_batch": 1e3 * dt, "launches_per_batch": launches,
                     "jitter_steps": {str(k): int(c) for k, c in zip(*np.unique(r["jitter"], return_counts=True))},
                     "fit_100x20_s": fit_s}
        print(mode, json.dumps(out[mode]), flush=True)
        ev.close()
    os.environ.pop("GPEMU_SPEC_LADDER", None)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
