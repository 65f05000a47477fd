"""Measure every BASELINE.json config on one B200 (writes gpurun_out/configs.json).

C1 n=200  d=2  p=2    : one eval + GA fit (100x20) + predict on 1000 points
C2 n=2048 d=6  p=1.95 : batch of 64 thetas
C3 n=4096 d=10 p=1.95 : batch of 100 thetas (the bench.py headline) + full GA fit
C4 n=16384 d=20 p=1.9 : nugget 1e-8 (the "lower-bound nugget" fixed), batch of 100
C5 n=8192 d=10 p=1.95 : model at a fixed theta + predict and MSE on 1M points
Device time is CUDA-event time of the C-ABI phases; wall time includes host work.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1203_1269_b200.gpemu as g  # noqa: E402


def lhd(n, d, rng):
    X = np.empty((n, d))
    for k in range(d):
        X[:, k] = (rng.permutation(n) + rng.random(n)) / n
    return X


def smooth(X):
    return (np.sin(3.0 * X + 0.37 * np.arange(X.shape[1])) + 0.5 * X * X).sum(1)


def thetas(d, B, rng):
    gg = np.empty((B, d))
    for k in range(d):
        gg[:, k] = (rng.permutation(B) + rng.random(B)) / B
    return 10.0 ** (-6 + (np.log10(12.0) + 6) * gg)


def batch_rate(ev, th, reps=3):
    ev.eval_batch(th)
    ev.set_profiling(True)
    t = time.time()
    for _ in range(reps):
        r = ev.eval_batch(th)
    wall = (time.time() - t) / reps
    chol = ev.phase_ms(1)[0] / reps
    asm = ev.phase_ms(0)[0] / reps
    ev.set_profiling(False)
    return r, wall, chol, asm


def main():
    rng = np.random.default_rng(2012)
    ctx = g.Context(0)
    be = g.Backend(ctx)
    out = {}
    # C1
    X = lhd(200, 2, rng)
    y = np.log(1 + (X ** 2).sum(1))
    data = g.new_dataset(X, y)
    ev = g.ProfileEvaluator(data, 2.0, 0.0, be, max_batch=100)
    th = thetas(2, 100, rng)
    r, wall, chol, asm = batch_rate(ev, th)
    t = time.time()
    fr = g.fit_gp_detailed(data, g.FitConfig(ga=g.GaConfig(100, 20), seed=0, p=2.0), be, evaluator=ev)
    fit_s = time.time() - t
    Xt = lhd(1000, 2, rng)
    t = time.time()
    yh, mse = g.predict(fr.model, Xt, with_mse=True)
    pred_s = time.time() - t
    out["C1"] = dict(n=200, d=2, p=2.0, batch=100, evals_per_s=100 / wall, fit_100x20_s=fit_s,
                     predict_mse_1000_s=pred_s, jitter_used=sorted(set(r["jitter"].tolist())))
    ev.close()
    print("C1", out["C1"], flush=True)
    # C2
    X = lhd(2048, 6, rng)
    ev = g.ProfileEvaluator(g.new_dataset(X, smooth(X)), 1.95, 0.0, be, max_batch=64)
    r, wall, chol, asm = batch_rate(ev, thetas(6, 64, rng))
    out["C2"] = dict(n=2048, d=6, p=1.95, batch=64, evals_per_s=64 / wall, batch_ms=wall * 1e3,
                     chol_ms=chol, chol_tflops=64 * 2048 ** 3 / 3 / (chol / 1e3) / 1e12)
    ev.close()
    print("C2", out["C2"], flush=True)
    # C3
    X = lhd(4096, 10, rng)
    data = g.new_dataset(X, smooth(X))
    ev = g.ProfileEvaluator(data, 1.95, 0.0, be, max_batch=100)
    r, wall, chol, asm = batch_rate(ev, thetas(10, 100, rng))
    t = time.time()
    fr = g.fit_gp_detailed(data, g.FitConfig(ga=g.GaConfig(100, 20), seed=0, p=1.95), be, evaluator=ev)
    fit_s = time.time() - t
    out["C3"] = dict(n=4096, d=10, p=1.95, batch=100, evals_per_s=100 / wall, batch_ms=wall * 1e3,
                     chol_ms=chol, chol_tflops=100 * 4096 ** 3 / 3 / (chol / 1e3) / 1e12,
                     fit_100x20_s=fit_s)
    ev.close()
    print("C3", out["C3"], flush=True)
    # C5 (before C4 to keep memory low)
    X = lhd(8192, 10, rng)
    m = g.model_at_theta(g.new_dataset(X, smooth(X)), np.full(10, 2.0), 1.95, 0.0, be)
    Xt = rng.random((1_000_000, 10))
    g.predict(m, Xt[:1000], with_mse=True)
    t = time.time()
    yh = g.predict(m, Xt)
    y_s = time.time() - t
    t = time.time()
    yh2, mse = g.predict(m, Xt, with_mse=True)  # first call: also grows the model's scratch
    ym_first = time.time() - t
    t = time.time()
    yh2, mse = g.predict(m, Xt, with_mse=True)
    ym_s = time.time() - t
    out["C5"] = dict(n=8192, d=10, N=1_000_000, predict_s=y_s, predict_mse_s=ym_s,
                     predict_mse_first_call_s=ym_first,
                     points_per_s=1e6 / y_s, points_with_mse_per_s=1e6 / ym_s)
    m.close()
    print("C5", out["C5"], flush=True)
    # C4
    X = lhd(16384, 20, rng)
    ev = g.ProfileEvaluator(g.new_dataset(X, smooth(X)), 1.9, 1e-8, be, max_batch=100)
    r, wall, chol, asm = batch_rate(ev, thetas(20, 100, rng), reps=1)
    out["C4"] = dict(n=16384, d=20, p=1.9, nugget=1e-8, batch=100, evals_per_s=100 / wall,
                     batch_ms=wall * 1e3, chol_ms=chol,
                     chol_tflops=100 * 16384 ** 3 / 3 / (chol / 1e3) / 1e12,
                     device_gb=ev.device_bytes() / 1e9,
                     status_counts={int(k): int(v) for k, v in zip(*np.unique(r["status"], return_counts=True))})
    ev.close()
    print("C4", out["C4"], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "configs.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
