"""Stress of the DAG engine's synchronisation (named barriers, slab-wise release, flag snapshot,
slab-0 prefetch, ladder relaunches): random designs and theta batches -- many candidates
failing pivots at various columns -- evaluated (a) twice in a 100-candidate launch, (b) in
8-candidate and single-candidate launches (the chain-bound instantiation), all of which must
agree bitwise; plus the deadlock word. usage: python tools/stress_dag.py [seconds] [n1,n2,...]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
sizes = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [130, 257, 600, 1000, 1500, 2100]
ctx = g.Context(0)
be = g.Backend(ctx)
rng = np.random.default_rng(12345)
t_end = time.time() + budget
cases = mism = 0
while time.time() < t_end:
    n = int(rng.choice(sizes))
    d = int(rng.integers(1, 7))
    p = float(rng.choice([1.0, 1.5, 1.95, 2.0]))
    X = rng.random((n, d))
    y = np.sin(3 * X).sum(1) + 0.1 * rng.standard_normal(n)
    th = 10 ** rng.uniform(-5.0, 1.5, size=(100, d))
    ev = g.ProfileEvaluator(g.new_dataset(X, y), p, 0.0, be, max_batch=100)
    a = ev.eval_batch(th)
    b = ev.eval_batch(th)
    lo = int(rng.integers(0, 92))
    c = ev.eval_batch(th[lo:lo + 8])
    i = int(rng.integers(0, 100))
    e = ev.eval_batch(th[i:i + 1])
    ok = True
    for k in ("neg2", "mu", "sigma2", "jitter", "log_det"):
        ok &= np.array_equal(a[k], b[k], equal_nan=True)
        ok &= np.array_equal(a[k][lo:lo + 8], c[k], equal_nan=True)
        ok &= np.array_equal(a[k][i:i + 1], e[k], equal_nan=True)
    cases += 1
    if not ok:
        mism += 1
        print(f"MISMATCH n={n} d={d} p={p} lo={lo} i={i}", flush=True)
    ev.close()
    if cases % 10 == 0:
        print(f"{cases} cases, {mism} mismatches, jitter>0 share {np.mean(a['jitter'] > 0):.2f}", flush=True)
print(f"done: {cases} cases, {mism} mismatches")
sys.exit(1 if mism else 0)
