"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref, built from
/root/reference/proj/include by oracle/Makefile). Run here (needs /root/reference at build
time only); the fixtures are committed and travel to the GPU box.

  kat.npz   known answers of the reference's own tests (test_correlation.cpp, test_backend.cpp,
            SPEC.md n=2 profile example) evaluated by the reference
  c1.npz    config C1 (n=200, d=2, p=2, goldstein_price_log): 100 GA-style thetas, the fit
            (GA 100x20) and 1000 test-point predictions
  c1p195.npz  same design, p=1.95 (self-discrepancy stress: near-singular thetas)
  c2.npz    config C2 design (n=2048, d=6, p=1.95, hartman6) with 16 thetas (the committed
            fixture holds all 64: tools/make_golden_c2_full.py)
Each eval set also stores `self_disc` (the reference's native build: ReferenceBackend vs
ParallelBackend), `truth` (long-double deviance of the same double R) and `sens` (max relative
change of that long-double deviance under random 1-ulp perturbations of R: the conditioning
floor any FP64 assembly of R inherits).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, RefLib, build  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")


def ga_thetas(ref, d, count, seed=0):
    lo = np.full(d, np.log10(1e-6))
    hi = np.full(d, np.log10(12.0))
    s = ref.lib.ref_derive_seed2(ref.lib.ref_derive_seed2(seed, 0x9A5EED), 0x1E17)
    return 10.0 ** ref.lhs_population(lo, hi, count, s)


def self_disc(fast, X, y, th, p):
    a = fast.eval_batch(X, y, th, p, backend="reference")
    b = fast.eval_batch(X, y, th, p, backend="parallel")
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(np.isfinite(a["neg2"]), np.abs(a["neg2"] - b["neg2"]) / np.abs(a["neg2"]), 0.0)


def main(only_extra=False):
    build()
    ref, fast = RefLib(), RefLib(fast=True)
    orc = Oracle()
    os.makedirs(OUT, exist_ok=True)

    # ---- known answers ------------------------------------------------------
    kat = {}
    kat["r_unit"] = ref.build_corr(np.array([[0.0], [1.0]]), [2.0], 1.95)[0, 1]
    kat["r_gauss"] = ref.corr_vector([0.5], np.array([[0.0]]), [1.0], 2.0)[0]
    L, ld, jt = ref.factorize(np.array([[1.0, 0.5], [0.5, 1.0]]), "reference")
    kat["L22"], kat["logdet22"], kat["jit22"] = L, ld, jt
    kat["u22"] = ref.solve(L, np.array([1.0, 1.0]))
    kat["x22"] = ref.solve(L, ref.solve(L, np.array([1.0, 1.0])), upper=True)
    Xc = np.array([[0.3, 0.3], [0.3, 0.3], [0.7, 0.1]])
    Rc = ref.build_corr(Xc, [2.0, 2.0], 1.95)
    Lc, ldc, jtc = ref.factorize(Rc, "parallel")
    kat["Xc"], kat["Rc"], kat["Lc"], kat["ldc"], kat["jitc"] = Xc, Rc, Lc, ldc, jtc
    r = ref.eval_batch(np.array([[0.0], [1.0]]), np.array([0.0, 1.0]), np.array([[2.0]]), 1.95)
    kat["spec_neg2"], kat["spec_mu"], kat["spec_sigma2"] = r["neg2"][0], r["mu"][0], r["sigma2"][0]
    mp = ref.model_predict(np.array([[0.0], [1.0]]), np.array([0.0, 1.0]), [2.0], 1.95, 0.0,
                           np.array([[0.5]]))
    kat["spec_pred"] = mp["yhat"][0]
    np.savez(os.path.join(OUT, "kat.npz"), **kat)

    # ---- C1 ------------------------------------------------------------------
    for name, p in (("c1", 2.0), ("c1p195", 1.95)):
        X = ref.maximin_lhd(200, 2, 7, 10000)
        y = np.array([ref.lib.ref_goldstein_price_log(np.ascontiguousarray(x).ctypes.data_as(
            __import__("ctypes").POINTER(__import__("ctypes").c_double))) for x in X])
        th = ga_thetas(ref, 2, 100)
        ev = ref.eval_batch(X, y, th, p)
        disc = self_disc(fast, X, y, th, p)
        truth, sens = orc.eval_sensitivity(X, y, th, p, ev["jitter"], reps=3)
        fit = ref.fit(X, y, p=p, population=100, generations=20, seed=0)
        opt = ref.eval_batch(X, y, fit["theta"][None, :], p)
        fit_truth = orc.eval_truth(X, y, fit["theta"][None, :], p, opt["jitter"])[0]
        Xt = ref.maximin_lhd(1000, 2, 11, 10000)
        mp = ref.model_predict(X, y, fit["theta"], p, 0.0, Xt)
        # reference self-discrepancy of the predictions (native build, reference vs parallel)
        ya = fast.model_predict(X, y, fit["theta"], p, 0.0, Xt, backend="reference")["yhat"]
        yb = fast.model_predict(X, y, fit["theta"], p, 0.0, Xt, backend="parallel")["yhat"]
        yscale = max(np.abs(mp["yhat"]).max(), np.abs(y).max())
        yhat_self_disc = np.abs(ya - yb).max() / yscale
        np.savez(os.path.join(OUT, f"{name}.npz"), X=X, y=y, p=p, thetas=th,
                 neg2=ev["neg2"], mu=ev["mu"], sigma2=ev["sigma2"], jitter=ev["jitter"],
                 log_det=ev["log_det"], self_disc=disc, truth=truth, sens=sens, fit_theta=fit["theta"],
                 fit_neg2=fit["neg2"], fit_truth=fit_truth,
                 fit_mu=fit["mu"], fit_sigma2=fit["sigma2"], fit_jitter_max=fit["jitter_max"],
                 fit_alpha=fit["alpha"], trace_best=fit["trace_best"],
                 trace_genes=fit["trace_genes"], Xt=Xt, yhat=mp["yhat"],
                 yhat_self_disc=yhat_self_disc)
        print(name, "done", flush=True)

    # ---- C2 ------------------------------------------------------------------
    X = ref.maximin_lhd(2048, 6, 7, 10000)
    C = __import__("ctypes")
    y = np.array([ref.lib.ref_hartman6(np.ascontiguousarray(x).ctypes.data_as(C.POINTER(C.c_double)))
                  for x in X])
    th = ga_thetas(ref, 6, 64)[:16]
    ev = ref.eval_batch(X, y, th, 1.95, threads=8)
    disc = self_disc(fast, X, y, th, 1.95)
    truth, sens = orc.eval_sensitivity(X, y, th, 1.95, ev["jitter"], reps=2)
    np.savez(os.path.join(OUT, "c2.npz"), X=X, y=y, p=1.95, thetas=th, neg2=ev["neg2"], mu=ev["mu"],
             sigma2=ev["sigma2"], jitter=ev["jitter"], log_det=ev["log_det"], self_disc=disc,
             truth=truth, sens=sens)
    print("c2 done")

    # ---- extra shapes: d=20 + nugget (C4-like), exponential kernel p=1, d=1 ------------
    for name, n, d, p, nugget, B in (("x_d20_nugget", 600, 20, 1.9, 1e-8, 16),
                                      ("x_p1", 500, 3, 1.0, 0.0, 16),
                                      ("x_d1", 300, 1, 1.5, 0.01, 16)):
        rng = np.random.default_rng(n * 31 + d)
        X = ref.maximin_lhd(n, d, 17, 2000)
        y = np.sin(3.0 * X + 0.37 * np.arange(d)).sum(1) + 0.5 * (X * X).sum(1)
        th = ga_thetas(ref, d, 64, seed=n)[:B]
        ev = ref.eval_batch(X, y, th, p, nugget)
        a = fast.eval_batch(X, y, th, p, nugget, backend="reference")
        b = fast.eval_batch(X, y, th, p, nugget, backend="parallel")
        with np.errstate(invalid="ignore", divide="ignore"):
            disc = np.where(np.isfinite(a["neg2"]), np.abs(a["neg2"] - b["neg2"]) / np.abs(a["neg2"]), 0.0)
        truth, sens = orc.eval_sensitivity(X, y, th, p, ev["jitter"], nugget=nugget, reps=2)
        np.savez(os.path.join(OUT, f"{name}.npz"), X=X, y=y, p=p, nugget=nugget, thetas=th,
                 neg2=ev["neg2"], mu=ev["mu"], sigma2=ev["sigma2"], jitter=ev["jitter"],
                 log_det=ev["log_det"], self_disc=disc, truth=truth, sens=sens)
        print(name, "done", flush=True)


if __name__ == "__main__":
    main()
