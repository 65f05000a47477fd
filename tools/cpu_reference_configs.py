"""The reference's own CPU path on the GPU box's host, per BASELINE config (SURVEY 8(d) "How the
CPU reference is timed"): ParallelBackend on every host thread and the unblocked "reference"
backend on one thread, deviance evals/s over a theta batch (plan construction reported
separately), and C5 kriging predictions/s. Uses oracle/_ref (the reference compiled from its own
headers with its build flags). Prints one JSON object; writes gpurun_out/cpu_reference.json."""
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import RefLib  # noqa: E402

ref = RefLib(fast=True)
cpu = next((ln.split(":", 1)[1].strip() for ln in open("/proc/cpuinfo") if ln.startswith("model name")),
           platform.processor())
out = {"host": {"nproc": os.cpu_count(), "cpu_model": cpu}, "lib": "oracle/_ref/libgpemu_ref_fast.so"}


def case(name, n, d, p, B_par, B_ref, seed):
    rng = np.random.default_rng(seed)
    X = rng.random((n, d))
    y = np.sin(3 * X).sum(1)
    th = 10 ** rng.uniform(-1.0, 0.5, size=(max(B_par, B_ref), d))
    res = {"n": n, "d": d, "p": p}
    _, sp, se = ref.eval_batch_timed(X, y, th[:B_par], p, backend="parallel", threads=0)
    res["parallel_all_threads"] = {"evals": B_par, "evals_per_s": B_par / se, "plan_s": sp}
    if B_ref:
        _, sp1, se1 = ref.eval_batch_timed(X, y, th[:B_ref], p, backend="reference", threads=1)
        res["reference_1_thread"] = {"evals": B_ref, "evals_per_s": B_ref / se1, "plan_s": sp1}
    out[name] = res
    print(name, json.dumps(res), flush=True)


case("C1", 200, 2, 2.0, 100, 100, 1)
case("C2", 2048, 6, 1.95, 16, 2, 2)
case("C3", 4096, 10, 1.95, 8, 0, 3)

# C5: model at a fixed theta (n=8192, d=10), then ŷ for test points (reference predict path)
rng = np.random.default_rng(5)
n, d = 8192, 10
X = rng.random((n, d))
y = np.sin(3 * X).sum(1)
theta = np.full(d, 2.0)
t0 = time.perf_counter()
ref.model_predict(X, y, theta, 1.95, 0.0, None, threads=0)
t1 = time.perf_counter()
N = 20000
Xt = rng.random((N, d))
ref.model_predict(X, y, theta, 1.95, 0.0, Xt, threads=0)
t2 = time.perf_counter()
pred_s = (t2 - t1) - (t1 - t0)
out["C5"] = {"n": n, "d": d, "model_s": t1 - t0, "test_points": N, "predict_s": pred_s,
             "points_per_s": N / pred_s, "note": "predict time = (model + N points) - (model alone)"}
print("C5", json.dumps(out["C5"]), flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "cpu_reference.json"), "w"), indent=1)
