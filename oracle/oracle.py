"""ctypes front end for the CPU checker libraries.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py. The product package
(paper_1203_1269_b200) never imports this module.

Two libraries, same calling conventions:
  * ``Oracle``  -> oracle/liborc.so, the C restatement (gpemu_oracle.c);
  * ``RefLib``  -> oracle/_ref/libgpemu_ref{,_fast}.so, the unmodified reference
    headers behind a C shim (ref_shim.cpp). Present when built in a container
    that has /root/reference; the .so files travel to the GPU box.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_dp = C.POINTER(C.c_double)
_sz = C.c_size_t
_u64 = C.c_uint64

LADDER = (0.0, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4)  # backend.hpp:77


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def build(quiet: bool = True) -> None:
    """Build liborc.so (always possible) and _ref/ (when /root/reference exists)."""
    targets = ["liborc.so"]
    if os.path.isdir("/root/reference/proj/include"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class _GaConfig(C.Structure):
    _fields_ = [("population", C.c_int), ("generations", C.c_int),
                ("crossover_rate", C.c_double), ("mutation_sigma", C.c_double),
                ("mutation_prob", C.c_double), ("elitism", C.c_int), ("seed", _u64)]


class _FitResult(C.Structure):
    _fields_ = [("neg2_log_lik", C.c_double), ("mu_hat", C.c_double), ("sigma2_hat", C.c_double),
                ("jitter_max", C.c_double), ("log_det", C.c_double), ("jitter_used", C.c_double)]


class Oracle:
    """The C restatement of the reference path (test infrastructure)."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "liborc.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        self.lib = L
        L.orc_derive_seed2.restype = _u64
        L.orc_derive_seed2.argtypes = [_u64, _u64]
        L.orc_derive_seed3.restype = _u64
        L.orc_derive_seed3.argtypes = [_u64, _u64, _u64]
        L.orc_maximin_lhd.argtypes = [_sz, _sz, _u64, _sz, _dp]
        L.orc_goldstein_price_log.restype = C.c_double
        L.orc_goldstein_price_log.argtypes = [_dp]
        L.orc_hartman6.restype = C.c_double
        L.orc_hartman6.argtypes = [_dp]
        L.orc_lhs_population.argtypes = [_dp, _dp, _sz, C.c_int, _u64, _dp]
        L.orc_corr_table.argtypes = [_dp, _sz, _sz, C.c_double, _dp]
        L.orc_build_from_table.argtypes = [_dp, _sz, _sz, _dp, C.c_double, _dp]
        L.orc_build_corr.argtypes = [_dp, _sz, _sz, _dp, C.c_double, C.c_double, _dp]
        L.orc_corr_vector.argtypes = [_dp, _dp, _sz, _sz, _dp, C.c_double, _dp]
        L.orc_factorize.argtypes = [_dp, _sz, C.c_int, _dp, _dp, _dp]
        L.orc_solve_lower.argtypes = [_dp, _sz, _dp, _dp]
        L.orc_solve_upper.argtypes = [_dp, _sz, _dp, _dp]
        L.orc_profile_eval_batch.argtypes = [_dp, _dp, _sz, _sz, C.c_double, C.c_double, _dp, _sz,
                                             C.c_int, _dp, _dp, _dp, _dp, _dp]
        L.orc_fit.argtypes = [_dp, _dp, _sz, _sz, C.c_double, C.c_double, _dp, _dp,
                              C.POINTER(_GaConfig), _u64, C.c_int, _dp, C.POINTER(_FitResult),
                              _dp, _dp, _dp, _dp]
        L.orc_predict.argtypes = [_dp, _sz, _sz, _dp, C.c_double, C.c_double, _dp, _dp, _sz, _dp]
        L.orc_kriging_mse.argtypes = [_dp, _sz, _sz, _dp, C.c_double, C.c_double, _dp, _dp, _sz, _dp]
        L.orc_profile_eval_ld.argtypes = [_dp, _dp, _sz, _sz, C.c_double, C.c_double, _dp, _sz,
                                          _dp, _dp]
        L.orc_profile_sensitivity.argtypes = [_dp, _dp, _sz, _sz, C.c_double, C.c_double, _dp,
                                              _sz, _dp, C.c_int, _u64, _dp, _dp]
        L.orc_refine_fit.argtypes = [_dp, _dp, _sz, _sz, C.c_double, C.c_double, _dp, _dp, _dp,
                                     C.c_double, C.c_int, C.c_int, _dp, _dp, C.POINTER(C.c_int)]
        L.orc_sspe.restype = C.c_double
        L.orc_sspe.argtypes = [_dp, _dp, _sz]

    # -- rng / designs ------------------------------------------------------
    def derive_seed(self, base, *rest):
        if len(rest) == 1:
            return self.lib.orc_derive_seed2(base, rest[0])
        if len(rest) == 2:
            return self.lib.orc_derive_seed3(base, rest[0], rest[1])
        raise ValueError("derive_seed arity")

    def maximin_lhd(self, n, d, seed, budget=10000):
        X = np.empty((n, d))
        if self.lib.orc_maximin_lhd(n, d, seed, budget, _ptr(X)) != 0:
            raise ValueError("maximin_lhd: bad spec")
        return X

    def goldstein_price_log(self, X):
        X = _f64(X)
        return np.array([self.lib.orc_goldstein_price_log(_ptr(X[i])) for i in range(len(X))])

    def hartman6(self, X):
        X = _f64(X)
        return np.array([self.lib.orc_hartman6(_ptr(X[i])) for i in range(len(X))])

    def lhs_population(self, lo, hi, count, seed):
        lo, hi = _f64(lo), _f64(hi)
        pop = np.empty((count, len(lo)))
        self.lib.orc_lhs_population(_ptr(lo), _ptr(hi), len(lo), count, seed, _ptr(pop))
        return pop

    # -- correlation --------------------------------------------------------
    def build_corr(self, X, theta, p, nugget=0.0):
        X, theta = _f64(X), _f64(theta)
        n, d = X.shape
        R = np.empty((n, n))
        if self.lib.orc_build_corr(_ptr(X), n, d, _ptr(theta), p, nugget, _ptr(R)) != 0:
            raise FloatingPointError("non-finite correlation value")
        return R

    def plan_build(self, X, theta, p, nugget=0.0):
        X, theta = _f64(X), _f64(theta)
        n, d = X.shape
        T = np.empty(max(n * (n - 1) // 2 * d, 1))
        self.lib.orc_corr_table(_ptr(X), n, d, p, _ptr(T))
        R = np.empty((n, n))
        if self.lib.orc_build_from_table(_ptr(T), n, d, _ptr(theta), nugget, _ptr(R)) != 0:
            raise FloatingPointError("non-finite correlation value")
        return R

    def corr_vector(self, xstar, X, theta, p):
        X, theta, xstar = _f64(X), _f64(theta), _f64(xstar)
        n, d = X.shape
        r = np.empty(n)
        self.lib.orc_corr_vector(_ptr(xstar), _ptr(X), n, d, _ptr(theta), p, _ptr(r))
        return r

    # -- backend ------------------------------------------------------------
    def factorize(self, R, kind=1):
        """Returns (L, log_det, jitter) or None when the ladder is exhausted."""
        R = _f64(R)
        n = R.shape[0]
        L = np.empty((n, n))
        ld, jt = C.c_double(), C.c_double()
        if self.lib.orc_factorize(_ptr(R), n, kind, _ptr(L), C.byref(ld), C.byref(jt)) != 0:
            return None
        return L, ld.value, jt.value

    def solve_lower(self, L, b):
        L, b = _f64(L), _f64(b)
        x = np.empty_like(b)
        self.lib.orc_solve_lower(_ptr(L), L.shape[0], _ptr(b), _ptr(x))
        return x

    def solve_upper(self, L, b):
        L, b = _f64(L), _f64(b)
        x = np.empty_like(b)
        self.lib.orc_solve_upper(_ptr(L), L.shape[0], _ptr(b), _ptr(x))
        return x

    # -- likelihood ---------------------------------------------------------
    def eval_batch(self, X, y, thetas, p, nugget=0.0, kind=1):
        """ProfileEvaluator::eval over each row of thetas -> dict of arrays."""
        X, y, thetas = _f64(X), _f64(y), _f64(np.atleast_2d(thetas))
        n, d = X.shape
        B = thetas.shape[0]
        out = {k: np.empty(B) for k in ("neg2", "mu", "sigma2", "jitter", "log_det")}
        rc = self.lib.orc_profile_eval_batch(_ptr(X), _ptr(y), n, d, p, nugget, _ptr(thetas), B, kind,
                                             _ptr(out["neg2"]), _ptr(out["mu"]), _ptr(out["sigma2"]),
                                             _ptr(out["jitter"]), _ptr(out["log_det"]))
        if rc != 0:
            raise MemoryError("oracle eval_batch allocation failed")
        return out

    def eval_truth(self, X, y, thetas, p, jitters, nugget=0.0):
        """Long-double deviance of the reference's double R + jitter (accuracy yardstick)."""
        X, y, thetas = _f64(X), _f64(y), _f64(np.atleast_2d(thetas))
        n, d = X.shape
        B = thetas.shape[0]
        jit = _f64(np.broadcast_to(jitters, (B,)))
        out = np.empty(B)
        if self.lib.orc_profile_eval_ld(_ptr(X), _ptr(y), n, d, p, nugget, _ptr(thetas), B,
                                        _ptr(jit), _ptr(out)) != 0:
            raise MemoryError("oracle eval_truth allocation failed")
        return out

    def eval_sensitivity(self, X, y, thetas, p, jitters, nugget=0.0, reps=3, seed=1):
        """(truth, sensitivity): long-double deviance and its max relative change under
        `reps` random 1-ulp perturbations of R (conditioning of each candidate)."""
        X, y, thetas = _f64(X), _f64(y), _f64(np.atleast_2d(thetas))
        n, d = X.shape
        B = thetas.shape[0]
        jit = _f64(np.broadcast_to(jitters, (B,)))
        truth, sens = np.empty(B), np.empty(B)
        if self.lib.orc_profile_sensitivity(_ptr(X), _ptr(y), n, d, p, nugget, _ptr(thetas), B,
                                            _ptr(jit), reps, seed, _ptr(truth), _ptr(sens)) != 0:
            raise MemoryError("oracle eval_sensitivity allocation failed")
        return truth, sens

    def fit(self, X, y, p=1.95, nugget=0.0, lo=1e-6, hi=12.0, population=100, generations=20,
            seed=0, kind=1, want_L=False, crossover_rate=0.9, mutation_sigma=0.15,
            mutation_prob=0.0, elitism=1):
        X, y = _f64(X), _f64(y)
        n, d = X.shape
        lo = _f64(np.broadcast_to(lo, (d,)))
        hi = _f64(np.broadcast_to(hi, (d,)))
        ga = _GaConfig(population, generations, crossover_rate, mutation_sigma, mutation_prob,
                       elitism, 0)
        theta = np.empty(d)
        res = _FitResult()
        alpha = np.empty(n)
        L = np.empty((n, n)) if want_L else None
        tb = np.empty(generations)
        tg = np.empty((generations, d))
        rc = self.lib.orc_fit(_ptr(X), _ptr(y), n, d, p, nugget, _ptr(lo), _ptr(hi), C.byref(ga),
                              seed, kind, _ptr(theta), C.byref(res), _ptr(alpha), _ptr(L),
                              _ptr(tb), _ptr(tg))
        if rc != 0:
            raise RuntimeError(f"oracle fit failed rc={rc}")
        return dict(theta=theta, neg2=res.neg2_log_lik, mu=res.mu_hat, sigma2=res.sigma2_hat,
                    jitter_max=res.jitter_max, jitter_used=res.jitter_used, log_det=res.log_det,
                    alpha=alpha, L=L, trace_best=tb, trace_genes=tg)

    def refine_fit(self, X, y, theta_fit, neg2_fit, p=1.95, nugget=0.0, lo=1e-6, hi=12.0,
                   budget=20, kind=1):
        """bench.hpp:302-383 golden-section polish -> (theta, neg2, evals used)."""
        X, y, th = _f64(X), _f64(y), _f64(theta_fit)
        n, d = X.shape
        lo = _f64(np.broadcast_to(lo, (d,)))
        hi = _f64(np.broadcast_to(hi, (d,)))
        out, nv, used = np.empty(d), C.c_double(), C.c_int()
        rc = self.lib.orc_refine_fit(_ptr(X), _ptr(y), n, d, p, nugget, _ptr(lo), _ptr(hi), _ptr(th),
                                     neg2_fit, budget, kind, _ptr(out), C.byref(nv), C.byref(used))
        if rc != 0:
            raise MemoryError("oracle refine_fit failed")
        return out, nv.value, used.value

    # -- predictor ----------------------------------------------------------
    def predict(self, X, theta, p, mu, alpha, Xtest):
        X, theta, alpha, Xtest = _f64(X), _f64(theta), _f64(alpha), _f64(Xtest)
        n, d = X.shape
        N = Xtest.shape[0]
        yhat = np.empty(N)
        if self.lib.orc_predict(_ptr(X), n, d, _ptr(theta), p, mu, _ptr(alpha), _ptr(Xtest), N,
                                _ptr(yhat)) != 0:
            raise FloatingPointError("non-finite correlation value")
        return yhat

    def kriging_mse(self, X, theta, p, sigma2, L, Xtest):
        X, theta, L, Xtest = _f64(X), _f64(theta), _f64(L), _f64(Xtest)
        n, d = X.shape
        N = Xtest.shape[0]
        mse = np.empty(N)
        self.lib.orc_kriging_mse(_ptr(X), n, d, _ptr(theta), p, sigma2, _ptr(L), _ptr(Xtest), N,
                                 _ptr(mse))
        return mse


class RefLib:
    """The reference's own headers behind ref_shim.cpp (oracle/_ref)."""

    def __init__(self, fast: bool = False, path: str | None = None):
        name = "libgpemu_ref_fast.so" if fast else "libgpemu_ref.so"
        path = path or os.path.join(HERE, "_ref", name)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = C.CDLL(path)
        self.lib = L
        cs = C.c_char_p
        L.ref_last_error.restype = cs
        L.ref_derive_seed2.restype = _u64
        L.ref_derive_seed2.argtypes = [_u64, _u64]
        L.ref_derive_seed3.restype = _u64
        L.ref_derive_seed3.argtypes = [_u64, _u64, _u64]
        L.ref_rng_draws.argtypes = [_u64, C.c_int, _u64, _sz, _dp]
        L.ref_maximin_lhd.argtypes = [_sz, _sz, _u64, _sz, _dp]
        L.ref_goldstein_price_log.restype = C.c_double
        L.ref_goldstein_price_log.argtypes = [_dp]
        L.ref_hartman6.restype = C.c_double
        L.ref_hartman6.argtypes = [_dp]
        L.ref_lhs_population.argtypes = [_dp, _dp, _sz, C.c_int, _u64, _dp]
        L.ref_build_corr.argtypes = [_dp, _sz, _sz, _dp, C.c_double, C.c_double, _dp]
        L.ref_plan_build.argtypes = [_dp, _sz, _sz, _dp, C.c_double, C.c_double, C.c_uint, _dp]
        L.ref_corr_vector.argtypes = [_dp, _dp, _sz, _sz, _dp, C.c_double, _dp]
        L.ref_factorize.argtypes = [_dp, _sz, cs, C.c_uint, _dp, _dp, _dp]
        L.ref_solve.argtypes = [_dp, _sz, _dp, C.c_int, _dp]
        L.ref_eval_batch.argtypes = [_dp, _dp, _sz, _sz, C.c_double, C.c_double, _dp, _sz, cs,
                                     C.c_uint, _dp, _dp, _dp, _dp, _dp]
        L.ref_eval_batch_timed.argtypes = [_dp, _dp, _sz, _sz, C.c_double, C.c_double, _dp, _sz,
                                           cs, C.c_uint, _dp, _dp, _dp]
        L.ref_fit.argtypes = [_dp, _dp, _sz, _sz, C.c_double, C.c_double, _dp, _dp, C.c_int,
                              C.c_int, _u64, cs, C.c_uint, _dp, _dp, _dp, _dp, _dp]
        L.ref_fit_refine.argtypes = [_dp, _dp, _sz, _sz, C.c_double, C.c_double, _dp, _dp, C.c_int,
                                     C.c_int, _u64, C.c_int, C.c_uint, _dp, _dp, _dp]
        L.ref_model_predict.argtypes = [_dp, _dp, _sz, _sz, _dp, C.c_double, C.c_double, cs,
                                        C.c_uint, _dp, _sz, _dp, _dp, _dp]
        # single precision (the reference's float instantiation)
        L.ref_eval_batch_f32.argtypes = L.ref_eval_batch.argtypes
        L.ref_eval_batch_timed_f32.argtypes = L.ref_eval_batch_timed.argtypes
        L.ref_fit_f32.argtypes = [_dp, _dp, _sz, _sz, C.c_double, C.c_double, _dp, _dp, C.c_int,
                                  C.c_int, _u64, cs, C.c_uint, _dp, _dp, _dp, _dp]
        L.ref_model_predict_f32.argtypes = L.ref_model_predict.argtypes

    def _check(self, rc):
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            raise {1: ValueError, 2: ArithmeticError, 3: RuntimeError, 4: KeyError}.get(rc, RuntimeError)(msg)

    def rng_draws(self, seed, kind, count, arg=0):
        out = np.empty(count)
        self.lib.ref_rng_draws(seed, kind, arg, count, _ptr(out))
        return out

    def maximin_lhd(self, n, d, seed, budget=10000):
        X = np.empty((n, d))
        self._check(self.lib.ref_maximin_lhd(n, d, seed, budget, _ptr(X)))
        return X

    def lhs_population(self, lo, hi, count, seed):
        lo, hi = _f64(lo), _f64(hi)
        pop = np.empty((count, len(lo)))
        self.lib.ref_lhs_population(_ptr(lo), _ptr(hi), len(lo), count, seed, _ptr(pop))
        return pop

    def build_corr(self, X, theta, p, nugget=0.0):
        X, theta = _f64(X), _f64(theta)
        n, d = X.shape
        R = np.empty((n, n))
        self._check(self.lib.ref_build_corr(_ptr(X), n, d, _ptr(theta), p, nugget, _ptr(R)))
        return R

    def plan_build(self, X, theta, p, nugget=0.0, threads=1):
        X, theta = _f64(X), _f64(theta)
        n, d = X.shape
        R = np.empty((n, n))
        self._check(self.lib.ref_plan_build(_ptr(X), n, d, _ptr(theta), p, nugget, threads, _ptr(R)))
        return R

    def corr_vector(self, xstar, X, theta, p):
        X, theta, xstar = _f64(X), _f64(theta), _f64(xstar)
        n, d = X.shape
        r = np.empty(n)
        self._check(self.lib.ref_corr_vector(_ptr(xstar), _ptr(X), n, d, _ptr(theta), p, _ptr(r)))
        return r

    def factorize(self, R, backend="parallel", threads=1):
        R = _f64(R)
        n = R.shape[0]
        L = np.empty((n, n))
        ld, jt = C.c_double(), C.c_double()
        rc = self.lib.ref_factorize(_ptr(R), n, backend.encode(), threads, _ptr(L), C.byref(ld),
                                    C.byref(jt))
        if rc == 2:
            return None
        self._check(rc)
        return L, ld.value, jt.value

    def solve(self, L, b, upper=False):
        L, b = _f64(L), _f64(b)
        x = np.empty_like(b)
        self._check(self.lib.ref_solve(_ptr(L), L.shape[0], _ptr(b), int(upper), _ptr(x)))
        return x

    def eval_batch(self, X, y, thetas, p, nugget=0.0, backend="parallel", threads=1,
                   precision="double"):
        X, y, thetas = _f64(X), _f64(y), _f64(np.atleast_2d(thetas))
        n, d = X.shape
        B = thetas.shape[0]
        out = {k: np.empty(B) for k in ("neg2", "mu", "sigma2", "jitter", "log_det")}
        fn = self.lib.ref_eval_batch_f32 if precision == "single" else self.lib.ref_eval_batch
        self._check(fn(_ptr(X), _ptr(y), n, d, p, nugget, _ptr(thetas), B,
                                            backend.encode(), threads, _ptr(out["neg2"]),
                                            _ptr(out["mu"]), _ptr(out["sigma2"]),
                                            _ptr(out["jitter"]), _ptr(out["log_det"])))
        return out

    def eval_batch_timed(self, X, y, thetas, p, nugget=0.0, backend="parallel", threads=0,
                         precision="double"):
        """-> (neg2, seconds_plan, seconds_evals); threads=0 = hardware_concurrency."""
        X, y, thetas = _f64(X), _f64(y), _f64(np.atleast_2d(thetas))
        n, d = X.shape
        B = thetas.shape[0]
        neg2 = np.empty(B)
        sp, se = C.c_double(), C.c_double()
        fn = self.lib.ref_eval_batch_timed_f32 if precision == "single" else self.lib.ref_eval_batch_timed
        self._check(fn(_ptr(X), _ptr(y), n, d, p, nugget, _ptr(thetas), B,
                                                  backend.encode(), threads, _ptr(neg2),
                                                  C.byref(sp), C.byref(se)))
        return neg2, sp.value, se.value

    def fit(self, X, y, p=1.95, nugget=0.0, lo=1e-6, hi=12.0, population=100, generations=20,
            seed=0, backend="parallel", threads=1):
        X, y = _f64(X), _f64(y)
        n, d = X.shape
        lo = _f64(np.broadcast_to(lo, (d,)))
        hi = _f64(np.broadcast_to(hi, (d,)))
        theta = np.empty(d)
        sc = np.empty(4)
        alpha = np.empty(n)
        tb = np.empty(generations)
        tg = np.empty((generations, d))
        self._check(self.lib.ref_fit(_ptr(X), _ptr(y), n, d, p, nugget, _ptr(lo), _ptr(hi),
                                     population, generations, seed, backend.encode(), threads,
                                     _ptr(theta), _ptr(sc), _ptr(alpha), _ptr(tb), _ptr(tg)))
        return dict(theta=theta, neg2=sc[0], mu=sc[1], sigma2=sc[2], jitter_max=sc[3], alpha=alpha,
                    trace_best=tb, trace_genes=tg)

    def fit_refine(self, X, y, p=1.95, nugget=0.0, lo=1e-6, hi=12.0, population=100,
                   generations=20, seed=0, budget=20, threads=1):
        """fit_gp_detailed + bench.hpp refine_fit -> (theta_fit, neg2_fit, theta_ref, neg2_ref, extra)."""
        X, y = _f64(X), _f64(y)
        n, d = X.shape
        lo = _f64(np.broadcast_to(lo, (d,)))
        hi = _f64(np.broadcast_to(hi, (d,)))
        tf, tr, sc = np.empty(d), np.empty(d), np.empty(3)
        self._check(self.lib.ref_fit_refine(_ptr(X), _ptr(y), n, d, p, nugget, _ptr(lo), _ptr(hi),
                                            population, generations, seed, budget, threads, _ptr(tf),
                                            _ptr(tr), _ptr(sc)))
        return tf, sc[0], tr, sc[1], int(sc[2])

    def fit_f32(self, X, y, p=1.95, nugget=0.0, lo=1e-6, hi=12.0, population=100, generations=20,
                seed=0, backend="parallel", threads=1):
        """fit_gp_detailed<float> (FitConfig::precision = single)."""
        X, y = _f64(X), _f64(y)
        n, d = X.shape
        lo = _f64(np.broadcast_to(lo, (d,)))
        hi = _f64(np.broadcast_to(hi, (d,)))
        theta, sc, alpha, tb = np.empty(d), np.empty(4), np.empty(n), np.empty(generations)
        self._check(self.lib.ref_fit_f32(_ptr(X), _ptr(y), n, d, p, nugget, _ptr(lo), _ptr(hi),
                                         population, generations, seed, backend.encode(), threads,
                                         _ptr(theta), _ptr(sc), _ptr(alpha), _ptr(tb)))
        return dict(theta=theta, neg2=sc[0], mu=sc[1], sigma2=sc[2], jitter_max=sc[3], alpha=alpha,
                    trace_best=tb)

    def model_predict(self, X, y, theta, p, nugget, Xtest, backend="parallel", threads=1,
                      precision="double"):
        X, y, theta = _f64(X), _f64(y), _f64(theta)
        n, d = X.shape
        Xtest = _f64(Xtest) if Xtest is not None else np.empty((0, d))
        N = Xtest.shape[0]
        yhat = np.empty(N)
        sc = np.empty(4)
        alpha = np.empty(n)
        fn = self.lib.ref_model_predict_f32 if precision == "single" else self.lib.ref_model_predict
        self._check(fn(_ptr(X), _ptr(y), n, d, _ptr(theta), p, nugget,
                                               backend.encode(), threads, _ptr(Xtest), N,
                                               _ptr(yhat), _ptr(sc), _ptr(alpha)))
        return dict(yhat=yhat, neg2=sc[0], mu=sc[1], sigma2=sc[2], jitter=sc[3], alpha=alpha)


def ref_available(fast: bool = False) -> bool:
    name = "libgpemu_ref_fast.so" if fast else "libgpemu_ref.so"
    return os.path.exists(os.path.join(HERE, "_ref", name))
