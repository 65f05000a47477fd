#!/usr/bin/env python
"""Regenerates tests/golden/c2.npz with the full config-C2 batch: 64 GA-style thetas (the
previous fixture held the first 16). Same fields and recipe as tools/make_golden.py's C2 block:
the reference itself (oracle/_ref strict build, ParallelBackend) for the records, its native
build's ReferenceBackend vs ParallelBackend for `self_disc`, and the oracle's long-double truth
and 1-ulp sensitivity of the same double R. The 80-bit checks are split over host processes.

  python tools/make_golden_c2_full.py [--procs 8]
"""
import argparse
import ctypes as C
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from oracle.oracle import Oracle, RefLib, build  # noqa: E402
from make_golden import ga_thetas, self_disc  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c2.npz")


def _sens(args):
    X, y, th, jit = args
    return Oracle().eval_sensitivity(X, y, th, 1.95, jit, reps=2)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--procs", type=int, default=os.cpu_count())
    a = ap.parse_args()
    build()
    ref, fast = RefLib(), RefLib(fast=True)
    X = ref.maximin_lhd(2048, 6, 7, 10000)
    y = np.array([ref.lib.ref_hartman6(np.ascontiguousarray(x).ctypes.data_as(C.POINTER(C.c_double)))
                  for x in X])
    th = ga_thetas(ref, 6, 64)
    ev = ref.eval_batch(X, y, th, 1.95, threads=a.procs)
    print("records done", flush=True)
    disc = self_disc(fast, X, y, th, 1.95)
    print("self-discrepancy done", flush=True)
    chunks = np.array_split(np.arange(len(th)), a.procs)
    with ProcessPoolExecutor(a.procs) as pool:
        parts = list(pool.map(_sens, [(X, y, th[c], ev["jitter"][c]) for c in chunks]))
    truth = np.concatenate([p[0] for p in parts])
    sens = np.concatenate([p[1] for p in parts])
    np.savez(OUT, X=X, y=y, p=1.95, thetas=th, neg2=ev["neg2"], mu=ev["mu"], sigma2=ev["sigma2"],
             jitter=ev["jitter"], log_det=ev["log_det"], self_disc=disc, truth=truth, sens=sens)
    print("c2 done:", len(th), "thetas", flush=True)


if __name__ == "__main__":
    main()
