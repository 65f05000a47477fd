"""Python mirror of the reference ``gpemu`` API on top of the B200 C-ABI.

Same names, argument meaning and error behaviour as the reference headers
(paths relative to /root/reference/proj/include/gpemu/):

  errors.hpp       Error, ValidationError, NotPositiveDefiniteError, FitError, ConfigError
  core.hpp         Dataset / new_dataset, Hyperparameters, FitConfig
  optimizer.hpp    GaConfig, GaTrace
  correlation.hpp  build_corr_matrix, corr_vector, CorrelationPlan, CorrelationMatrix
  backend.hpp      Backend ("accelerated"), CorrelationFactor, Ledger, make_backend, kJitterLadder
  likelihood.hpp   ProfileEvaluator (eval + eval_batch), ProfileEval, model_at_theta,
                   fit_gp_detailed, fit_gp, GpModel, FitResult
  predictor.hpp    predict (+ predict_mse), sspe

Every numeric result comes from libgpemu_b200.so (sm_100a kernels); there is
no CPU fallback, and loading fails loudly when the library is missing.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libgpemu_b200.so")

kJitterLadder = (0.0, 1e-8, 1e-7, 1e-6, 1e-5, 1e-4)  # backend.hpp:77
kUnitCubeTolerance = 1e-12                            # core.hpp:45


# ---------------------------------------------------------------- errors.hpp
class Error(RuntimeError):
    """Base class for all errors (errors.hpp:9-13)."""


class ValidationError(Error):
    pass


class NotPositiveDefiniteError(Error):
    pass


class FitError(Error):
    pass


class ConfigError(Error):
    pass


class DeviceError(Error):
    """CUDA / device failure (mapped from GPEMU_CUDA)."""


_STATUS_EXC = {1: ValidationError, 2: NotPositiveDefiniteError, 3: FitError, 4: ConfigError,
               5: Error, 6: DeviceError, 7: Error}

# ---------------------------------------------------------------- library
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_sz = C.c_size_t
_vp = C.c_void_p

EXPORTED_SYMBOLS = (
    "gpemu_last_error", "gpemu_version", "gpemu_ctx_create", "gpemu_ctx_destroy",
    "gpemu_ctx_set_stream", "gpemu_ctx_set_engine", "gpemu_ctx_launch_count", "gpemu_build_corr",
    "gpemu_corr_vector", "gpemu_factorize", "gpemu_solve_lower", "gpemu_solve_upper",
    "gpemu_plan_create", "gpemu_plan_destroy", "gpemu_plan_device_bytes", "gpemu_eval_batch",
    "gpemu_eval_batch_device", "gpemu_plan_last_factor", "gpemu_fit", "gpemu_model_at_theta",
    "gpemu_model_destroy", "gpemu_predict", "gpemu_plan_set_profiling", "gpemu_plan_phase_ms",
    "gpemu_plan_dag_profile", "gpemu_try_cholesky", "gpemu_ga_create", "gpemu_ga_destroy",
    "gpemu_ga_thetas", "gpemu_ga_tell", "gpemu_ga_status", "gpemu_refine_fit",
    "gpemu_plan_create_ex", "gpemu_plan_precision", "gpemu_refine_fit_ex", "gpemu_model_scalars",
    "gpemu_ctx_mem_info", "gpemu_plan_bytes", "gpemu_ticket_order", "gpemu_ctx_num_sms",
    "gpemu_eval_batch_multi", "gpemu_fit_multi", "gpemu_model_factor", "gpemu_model_import",
    "gpemu_model_alpha", "gpemu_maximin_lhd",
)


class _GaConfigC(C.Structure):
    _fields_ = [("population", C.c_int), ("generations", C.c_int), ("crossover_rate", C.c_double),
                ("mutation_sigma", C.c_double), ("mutation_prob", C.c_double),
                ("elitism", C.c_int)]


class _FitResultC(C.Structure):
    _fields_ = [("neg2_log_lik", C.c_double), ("mu_hat", C.c_double), ("sigma2_hat", C.c_double),
                ("jitter_max", C.c_double), ("r_builds", C.c_uint64),
                ("factorizations", C.c_uint64), ("triangular_solves", C.c_uint64)]


_LIB = None


def lib():
    """Load libgpemu_b200.so (build it first with paper_1203_1269_b200.build)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1203_1269_b200.build` "
                          "(the B200 engine has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.gpemu_last_error.restype = C.c_char_p
    L.gpemu_version.restype = C.c_char_p
    L.gpemu_ctx_create.argtypes = [C.c_int, C.POINTER(_vp)]
    L.gpemu_ctx_destroy.argtypes = [_vp]
    L.gpemu_ctx_set_stream.argtypes = [_vp, _vp]
    L.gpemu_ctx_set_engine.argtypes = [_vp, C.c_int]
    L.gpemu_ctx_launch_count.argtypes = [_vp]
    L.gpemu_ctx_launch_count.restype = C.c_uint64
    L.gpemu_ctx_num_sms.argtypes = [_vp]
    L.gpemu_build_corr.argtypes = [_vp, _dp, _sz, _sz, _dp, C.c_double, C.c_double, _dp]
    L.gpemu_corr_vector.argtypes = [_vp, _dp, _dp, _sz, _sz, _dp, C.c_double, _dp]
    L.gpemu_factorize.argtypes = [_vp, _dp, _sz, _dp, _dp, _dp]
    L.gpemu_try_cholesky.argtypes = [_vp, _dp, _sz]
    L.gpemu_ga_create.argtypes = [_sz, _dp, _dp, C.POINTER(_GaConfigC), C.c_uint64, C.POINTER(_vp)]
    L.gpemu_ga_destroy.argtypes = [_vp]
    L.gpemu_ga_thetas.argtypes = [_vp, _dp]
    L.gpemu_ga_tell.argtypes = [_vp, _dp]
    L.gpemu_ga_status.argtypes = [_vp, _ip, _ip, _dp, _dp, _ip, _ip, _dp, _dp]
    L.gpemu_solve_lower.argtypes = [_vp, _dp, _sz, _dp, _dp]
    L.gpemu_solve_upper.argtypes = [_vp, _dp, _sz, _dp, _dp]
    L.gpemu_plan_create.argtypes = [_vp, _dp, _dp, _sz, _sz, C.c_double, C.c_double, _sz,
                                    C.POINTER(_vp)]
    L.gpemu_plan_create_ex.argtypes = [_vp, _dp, _dp, _sz, _sz, C.c_double, C.c_double, _sz,
                                       C.c_int, C.POINTER(_vp)]
    L.gpemu_plan_precision.argtypes = [_vp]
    L.gpemu_plan_destroy.argtypes = [_vp]
    L.gpemu_plan_device_bytes.argtypes = [_vp]
    L.gpemu_plan_device_bytes.restype = _sz
    L.gpemu_eval_batch.argtypes = [_vp, _dp, _sz, _dp, _dp, _dp, _dp, _dp, _ip]
    L.gpemu_eval_batch_device.argtypes = [_vp, _vp, _sz, _vp]
    L.gpemu_plan_last_factor.argtypes = [_vp, _sz, _dp, _dp, _dp]
    L.gpemu_plan_set_profiling.argtypes = [_vp, C.c_int]
    L.gpemu_plan_phase_ms.argtypes = [_vp, C.c_int, _dp, _ip]
    L.gpemu_plan_dag_profile.argtypes = [_vp, C.c_int, C.c_void_p, _sz]
    L.gpemu_ticket_order.argtypes = [C.c_int, C.c_int, C.c_int, C.c_void_p, _sz]
    L.gpemu_fit.argtypes = [_vp, _dp, _dp, C.POINTER(_GaConfigC), C.c_uint64,
                            C.POINTER(_FitResultC), _dp, _dp, _dp, _dp, C.POINTER(_vp)]
    L.gpemu_fit_multi.argtypes = [C.POINTER(_vp), C.c_int, _dp, _dp, C.POINTER(_GaConfigC),
                                  C.c_uint64, C.POINTER(_FitResultC), _dp, _dp, _dp, _dp,
                                  C.POINTER(_vp)]
    L.gpemu_eval_batch_multi.argtypes = [C.POINTER(_vp), C.c_int, _dp, _sz, _dp, _dp, _dp, _dp,
                                         _dp, _ip]
    L.gpemu_model_at_theta.argtypes = [_vp, _dp, C.POINTER(_vp), _dp, _dp]
    L.gpemu_refine_fit.argtypes = [_vp, _dp, _dp, _dp, C.c_double, C.c_int, _dp, _dp,
                                   C.POINTER(C.c_int), C.POINTER(_vp), _dp, _dp]
    L.gpemu_model_scalars.argtypes = [_vp, _dp]
    L.gpemu_model_factor.argtypes = [_vp, _dp, _dp]
    L.gpemu_model_alpha.argtypes = [_vp, _dp]
    L.gpemu_model_import.argtypes = [_vp, _dp, _sz, _sz, _dp, C.c_double, _dp, C.c_double, _dp,
                                     _dp, C.POINTER(_vp)]
    L.gpemu_ctx_mem_info.argtypes = [_vp, C.POINTER(_sz), C.POINTER(_sz)]
    L.gpemu_plan_bytes.argtypes = [_sz, _sz, _sz, C.c_int]
    L.gpemu_plan_bytes.restype = _sz
    L.gpemu_refine_fit_ex.argtypes = [_vp, _vp, _dp, _dp, _dp, C.c_double, C.c_int, _dp, _dp,
                                      C.POINTER(C.c_int), C.POINTER(_vp), _dp, _dp]
    L.gpemu_model_destroy.argtypes = [_vp]
    L.gpemu_predict.argtypes = [_vp, _dp, _sz, _dp, _dp]
    L.gpemu_maximin_lhd.argtypes = [_vp, _sz, _sz, C.c_uint64, _sz, _dp, _dp]
    _LIB = L
    return L


def _check(rc: int):
    if rc != 0:
        msg = lib().gpemu_last_error().decode()
        raise _STATUS_EXC.get(rc, Error)(msg)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


# ---------------------------------------------------------------- context
class Context:
    """One device + one stream (C-ABI gpemu_ctx)."""

    def __init__(self, device: int = 0, engine: str = "dag"):
        h = _vp()
        _check(lib().gpemu_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device
        self.set_engine(engine)

    def set_engine(self, engine: str):
        _check(lib().gpemu_ctx_set_engine(self.handle, {"dag": 0, "simple": 1}[engine]))
        self.engine = engine

    def set_stream(self, stream_ptr: Optional[int]):
        _check(lib().gpemu_ctx_set_stream(self.handle, _vp(stream_ptr or 0)))

    @property
    def launch_count(self) -> int:
        return int(lib().gpemu_ctx_launch_count(self.handle))

    @property
    def num_sms(self) -> int:
        return int(lib().gpemu_ctx_num_sms(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            lib().gpemu_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_DEFAULT_CTX: Optional[Context] = None


def default_context() -> Context:
    global _DEFAULT_CTX
    if _DEFAULT_CTX is None:
        _DEFAULT_CTX = Context(0)
    return _DEFAULT_CTX


# ---------------------------------------------------------------- core.hpp
class Dataset:
    """Design points on the unit cube plus responses (core.hpp:24-41)."""

    def __init__(self, inputs: np.ndarray, outputs: np.ndarray):
        self._inputs = inputs
        self._outputs = outputs

    def n(self) -> int:
        return self._inputs.shape[0]

    def d(self) -> int:
        return self._inputs.shape[1]

    def inputs(self) -> np.ndarray:
        return self._inputs

    def outputs(self) -> np.ndarray:
        return self._outputs


def new_dataset(inputs, outputs) -> Dataset:
    """core.hpp:47-66 validation rules."""
    X = _f64(inputs)
    y = _f64(outputs).reshape(-1)
    if X.ndim != 2 or X.shape[0] < 2:
        raise ValidationError("new_dataset: need at least 2 design points")
    if X.shape[1] < 1:
        raise ValidationError("new_dataset: need at least 1 input dimension")
    if y.shape[0] != X.shape[0]:
        raise ValidationError(f"new_dataset: dimension mismatch: {X.shape[0]} input rows vs "
                              f"{y.shape[0]} outputs")
    if not np.all(np.isfinite(X)):
        raise ValidationError("new_dataset: non-finite input coordinate")
    bad = (X < -kUnitCubeTolerance) | (X > 1.0 + kUnitCubeTolerance)
    if bad.any():
        i = int(np.argwhere(bad)[0][0])
        raise ValidationError(f"new_dataset: coordinate outside the unit cube at row {i}")
    if not np.all(np.isfinite(y)):
        raise ValidationError("new_dataset: non-finite output")
    X.setflags(write=False)
    y.setflags(write=False)
    return Dataset(X, y)


@dataclass
class Hyperparameters:
    """core.hpp:71-84."""
    theta: Sequence[float]
    p: float = 1.95
    nugget: float = 0.0

    def validate(self, expected_d: int):
        th = np.asarray(self.theta, dtype=np.float64)
        if th.shape != (expected_d,):
            raise ValidationError("Hyperparameters: theta length does not match input dimension")
        if not np.all(np.isfinite(th)) or not np.all(th >= 0.0):
            raise ValidationError("Hyperparameters: theta entries must be finite and nonnegative")
        if not (self.p > 0.0) or not (self.p <= 2.0):
            raise ValidationError("Hyperparameters: p must be in (0, 2]")
        if not (self.nugget >= 0.0) or not math.isfinite(self.nugget):
            raise ValidationError("Hyperparameters: nugget must be finite and nonnegative")


@dataclass
class GaConfig:
    """optimizer.hpp:20-39."""
    population: int = 100
    generations: int = 20
    crossover_rate: float = 0.9
    mutation_sigma: float = 0.15
    mutation_prob: float = 0.0
    elitism: int = 1
    seed: int = 0

    def budget(self) -> int:
        return self.population * self.generations


PRECISIONS = {"double": 0, "single": 1, "float": 1}


def parse_precision(s: str) -> str:
    """core.hpp:92-96: 'single' | 'float' | 'double', else ConfigError."""
    if s in ("single", "float"):
        return "single"
    if s == "double":
        return "double"
    raise ConfigError(f"unknown precision '{s}' (expected single|double)")


@dataclass
class FitConfig:
    """core.hpp:100-124. precision 'single' runs the reference's float instantiation on the
    device's FP32 engine (float R / factor / solves, log|R| and dots in double)."""
    backend: str = "accelerated"
    precision: str = "double"
    ga: GaConfig = field(default_factory=GaConfig)
    theta_bounds: List[tuple] = field(default_factory=list)
    seed: int = 0
    p: float = 1.95
    nugget: float = 0.0
    kDefaultThetaLower = 1e-6
    kDefaultThetaUpper = 12.0

    def bounds_for(self, d: int):
        b = list(self.theta_bounds)
        if not b:
            b = [(self.kDefaultThetaLower, self.kDefaultThetaUpper)] * d
        if len(b) == 1 and d > 1:
            b = b * d
        if len(b) != d:
            raise ValidationError("FitConfig: theta_bounds length does not match input dimension")
        for lo, hi in b:
            if not (lo > 0.0) or not (lo < hi):
                raise ValidationError("FitConfig: theta bounds require 0 < lower < upper")
        return b


# ---------------------------------------------------------------- correlation.hpp
@dataclass
class CorrelationMatrix:
    values: np.ndarray
    nugget: float = 0.0

    def n(self) -> int:
        return self.values.shape[0]


def build_corr_matrix(X, params: Hyperparameters, ctx: Optional[Context] = None) -> CorrelationMatrix:
    """correlation.hpp:99-146 on the device."""
    ctx = ctx or default_context()
    X = _f64(X)
    n, d = X.shape
    params.validate(d)
    th = _f64(params.theta)
    R = np.empty((n, n))
    _check(lib().gpemu_build_corr(ctx.handle, _p(X), n, d, _p(th), float(params.p),
                                  float(params.nugget), _p(R)))
    return CorrelationMatrix(R, float(params.nugget))


def corr_vector(x_star, X, params: Hyperparameters, ctx: Optional[Context] = None) -> np.ndarray:
    """correlation.hpp:67-91 on the device (no nugget)."""
    ctx = ctx or default_context()
    X = _f64(X)
    n, d = X.shape
    params.validate(d)
    xs = _f64(x_star).reshape(-1)
    if xs.shape[0] != d:
        raise ValidationError("corr_vector: test point dimension mismatch")
    th = _f64(params.theta)
    r = np.empty(n)
    _check(lib().gpemu_corr_vector(ctx.handle, _p(xs), _p(X), n, d, _p(th), float(params.p), _p(r)))
    return r


class CorrelationPlan:
    """correlation.hpp:153-229: per-design plan; build_into fills R for a theta."""

    def __init__(self, X, p: float, ctx: Optional[Context] = None):
        self._X = _f64(X)
        self._p = float(p)
        self._ctx = ctx or default_context()

    def n(self) -> int:
        return self._X.shape[0]

    def d(self) -> int:
        return self._X.shape[1]

    def build_into(self, R: CorrelationMatrix, theta, nugget: float):
        th = _f64(theta)
        if th.shape[0] != self.d():
            raise ValidationError("CorrelationPlan: theta length mismatch")
        out = build_corr_matrix(self._X, Hyperparameters(th, self._p, nugget), self._ctx)
        R.values = out.values
        R.nugget = float(nugget)


# ---------------------------------------------------------------- backend.hpp
@dataclass
class LedgerCounts:
    r_builds: int = 0
    factorizations: int = 0
    triangular_solves: int = 0


class Ledger:
    """backend.hpp:26-49 (counts the reference's cost model, not device kernels)."""

    def __init__(self):
        self._c = LedgerCounts()

    def add_r_build(self, k=1):
        self._c.r_builds += k

    def add_factorization(self, k=1):
        self._c.factorizations += k

    def add_triangular_solves(self, k):
        self._c.triangular_solves += k

    def snapshot(self) -> LedgerCounts:
        return LedgerCounts(self._c.r_builds, self._c.factorizations, self._c.triangular_solves)


@dataclass
class CorrelationFactor:
    """backend.hpp:54-70: lower (strict upper zero), log_det, jitter_used."""
    lower: np.ndarray
    log_det: float = 0.0
    jitter_used: float = 0.0

    def n(self) -> int:
        return self.lower.shape[0]

    def dense_lower(self) -> np.ndarray:
        return np.tril(self.lower)


class Backend:
    """The "accelerated" backend (BackendKind::kAccelerated, backend.hpp:72, :321-351)."""

    kind = "accelerated"

    def __init__(self, ctx: Optional[Context] = None, engine: str = "dag"):
        self.ctx = ctx or Context(0, engine)
        self._ledger = Ledger()

    def name(self) -> str:
        return "accelerated"

    def ledger(self) -> Ledger:
        return self._ledger

    def factorize(self, R: CorrelationMatrix) -> CorrelationFactor:
        """factorize_into (backend.hpp:102-120): ladder on the device."""
        self._ledger.add_factorization()
        A = _f64(R.values)
        n = A.shape[0]
        L = np.empty((n, n))
        ld, jt = C.c_double(), C.c_double()
        _check(lib().gpemu_factorize(self.ctx.handle, _p(A), n, _p(L), C.byref(ld), C.byref(jt)))
        return CorrelationFactor(L, ld.value, jt.value)

    def solve_lower(self, f: CorrelationFactor, b) -> np.ndarray:
        self._ledger.add_triangular_solves(1)
        L, b = _f64(f.lower), _f64(b)
        x = np.empty_like(b)
        _check(lib().gpemu_solve_lower(self.ctx.handle, _p(L), L.shape[0], _p(b), _p(x)))
        return x

    def solve_upper(self, f: CorrelationFactor, b) -> np.ndarray:
        self._ledger.add_triangular_solves(1)
        L, b = _f64(f.lower), _f64(b)
        x = np.empty_like(b)
        _check(lib().gpemu_solve_upper(self.ctx.handle, _p(L), L.shape[0], _p(b), _p(x)))
        return x

    def solve_full(self, f: CorrelationFactor, b) -> np.ndarray:
        return self.solve_upper(f, self.solve_lower(f, b))

    # the reference's in-place forms (backend.hpp:102, :129, :143)
    def factorize_into(self, R: CorrelationMatrix, out: CorrelationFactor) -> None:
        f = self.factorize(R)
        out.lower, out.log_det, out.jitter_used = f.lower, f.log_det, f.jitter_used

    def solve_lower_into(self, f: CorrelationFactor, b, x: np.ndarray) -> None:
        x[...] = self.solve_lower(f, b)

    def solve_upper_into(self, f: CorrelationFactor, b, x: np.ndarray) -> None:
        x[...] = self.solve_upper(f, b)


_REGISTRY = {"accelerated": lambda threads=0: Backend()}


def backend_registry() -> dict:
    """backend.hpp:324-331. This package registers only "accelerated"; the reference's
    "reference" / "parallel" CPU backends are the oracle (oracle/), not part of the product."""
    return _REGISTRY


def make_backend(id: str, threads: int = 0) -> Backend:
    """backend.hpp:340-351. Only "accelerated" lives here; the CPU backends are the reference's."""
    if id not in _REGISTRY:
        raise ConfigError(f"unknown backend '{id}'; available: " + " ".join(sorted(_REGISTRY)))
    return _REGISTRY[id](threads)


def register_backend(id: str, factory):
    _REGISTRY[id] = factory


# ---------------------------------------------------------------- likelihood.hpp
@dataclass
class ProfileEval:
    """likelihood.hpp:21-27."""
    theta: List[float]
    neg2_log_lik: float = math.inf
    mu_hat: float = 0.0
    sigma2_hat: float = 0.0
    jitter_used: float = 0.0


def _dot_accumulate(a, b) -> float:
    """matrix.hpp:64-69: sequential double dot."""
    s = 0.0
    for x, z in zip(np.asarray(a, dtype=np.float64).tolist(), np.asarray(b, dtype=np.float64).tolist()):
        s += x * z
    return s


def mu_hat(backend: Backend, f: CorrelationFactor, y) -> float:
    """likelihood.hpp:32-44: (v.u)/(v.v), u = L^-1 y, v = L^-1 1 (two solves)."""
    y = _f64(y)
    if y.shape[0] != f.n():
        raise ValidationError("mu_hat: output length mismatch")
    u = backend.solve_lower(f, y)
    v = backend.solve_lower(f, np.ones_like(y))
    vtv = _dot_accumulate(v, v)
    if not vtv > 0.0:
        raise Error("mu_hat: degenerate denominator (broken factor)")
    return _dot_accumulate(v, u) / vtv


def sigma2_hat(backend: Backend, f: CorrelationFactor, y, mu: float) -> float:
    """likelihood.hpp:47-57: (y - mu)' R^-1 (y - mu) / n via one solve."""
    y = _f64(y)
    if y.shape[0] != f.n():
        raise ValidationError("sigma2_hat: output length mismatch")
    w = backend.solve_lower(f, y - mu)
    s = _dot_accumulate(w, w) / y.shape[0]
    return 0.0 if s < 0.0 else s


def sigma2_hat_from_parts(utu: float, vtu: float, vtv: float, mu: float, n: int) -> float:
    """likelihood.hpp:63-66: w'w = u'u - 2 mu v'u + mu^2 v'v, floored at 0."""
    s = (utu - 2.0 * mu * vtu + mu * mu * vtv) / float(n)
    return 0.0 if s < 0.0 else s


class ProfileEvaluator:
    """likelihood.hpp:74-158 bound to a device plan. eval_batch is the B200 hot path."""

    def __init__(self, data: Dataset, p: float, nugget: float, backend: Backend,
                 max_batch: int = 128, precision: str = "double"):
        self.backend = backend
        self._n, self._d = data.n(), data.d()
        self._data = data
        self.precision = parse_precision(precision)
        Hyperparameters([1.0] * self._d, p, nugget).validate(self._d)
        h = _vp()
        X, y = _f64(data.inputs()), _f64(data.outputs())
        _check(lib().gpemu_plan_create_ex(backend.ctx.handle, _p(X), _p(y), self._n, self._d,
                                          float(p), float(nugget), int(max_batch),
                                          PRECISIONS[self.precision], C.byref(h)))
        self.handle = h
        self.p, self.nugget, self.max_batch = float(p), float(nugget), int(max_batch)
        self._jitter_max = 0.0
        self._last = None

    def n(self):
        return self._n

    def d(self):
        return self._d

    def jitter_max(self) -> float:
        return self._jitter_max

    def device_bytes(self) -> int:
        return int(lib().gpemu_plan_device_bytes(self.handle))

    def set_profiling(self, enable: bool):
        _check(lib().gpemu_plan_set_profiling(self.handle, int(enable)))

    def phase_ms(self, phase: int):
        """(total device ms, launches) of phase 0 assemble / 1 cholesky / 2 finalize."""
        t, c = C.c_double(), C.c_int()
        _check(lib().gpemu_plan_phase_ms(self.handle, phase, C.byref(t), C.byref(c)))
        return t.value, c.value

    DAG_PHASES = ("ticket", "gemm", "acc_store", "potrf", "diag_store", "border", "off_wait",
                  "trsm", "off_store", "task_end", "prod_flags", "prod_empty", "n_diag", "n_off",
                  "slabs", "total", "full_wait", "diag_full_wait", "diag_gemm", "potrf_pivot",
                  "potrf_bd_wait", "potrf_panel", "potrf_bp_wait", "potrf_update")

    def dag_profile(self, enable: bool = True, read: bool = False):
        """Diagnostics: arm / read the DAG engine's per-CTA phase cycle counters."""
        sms = self.backend.ctx.num_sms  # the C side lays the counters out per CTA (one per SM)
        out = np.zeros(sms * 24 + 256 + 65536 * 4, dtype=np.uint64) if read else None
        _check(lib().gpemu_plan_dag_profile(self.handle, int(enable),
                                            None if out is None else out.ctypes.data, 0 if out is None else out.size))
        if out is None:
            return None
        m = out[:sms * 24].reshape(-1, 24)
        res = {k: m[:, i] for i, k in enumerate(self.DAG_PHASES)}
        res["flag_wait_by_j"] = out[sms * 24:sms * 24 + 256]  # producer flag waits: [0,128) OFF, [128,256) DIAG, by j
        res["trace"] = out[sms * 24 + 256:].reshape(-1, 4)  # per ticket: start, gemm end, publish, end (ns)
        return res

    def eval_batch_device(self, theta_ptr: int, B: int, out_ptr: int):
        """Device-resident batch: theta_ptr -> B x d doubles, out_ptr -> B x 8 records."""
        _check(lib().gpemu_eval_batch_device(self.handle, _vp(theta_ptr), B, _vp(out_ptr)))

    def eval_batch(self, thetas) -> dict:
        """B independent ProfileEvaluator::eval calls in one device batch."""
        T = _f64(np.atleast_2d(thetas))
        B = T.shape[0]
        if T.shape[1] != self._d:
            raise ValidationError("CorrelationPlan: theta length mismatch")
        out = {k: np.empty(B) for k in ("neg2", "mu", "sigma2", "jitter", "log_det")}
        st = np.empty(B, dtype=np.int32)
        for s0 in range(0, B, self.max_batch):
            s1 = min(B, s0 + self.max_batch)
            sub = np.ascontiguousarray(T[s0:s1])
            views = {k: v[s0:s1] for k, v in out.items()}
            _check(lib().gpemu_eval_batch(self.handle, _p(sub), s1 - s0, _p(views["neg2"]),
                                          _p(views["mu"]), _p(views["sigma2"]), _p(views["jitter"]),
                                          _p(views["log_det"]), st[s0:s1].ctypes.data_as(_ip)))
        out["status"] = st
        ok = st != 1
        if ok.any():
            self._jitter_max = max(self._jitter_max, float(out["jitter"][ok].max()))
        led = self.backend.ledger()
        led.add_r_build(B)
        led.add_factorization(B)
        led.add_triangular_solves(2 * B)
        self._last = (T, B)
        return out

    def eval(self, theta) -> ProfileEval:
        r = self.eval_batch(np.asarray(theta, dtype=np.float64)[None, :])
        return ProfileEval(list(np.asarray(theta, dtype=np.float64)), float(r["neg2"][0]),
                           float(r["mu"][0]), float(r["sigma2"][0]), float(r["jitter"][0]))

    def last_factor(self, slot: int = 0) -> CorrelationFactor:
        L = np.empty((self._n, self._n))
        ld, jt = C.c_double(), C.c_double()
        _check(lib().gpemu_plan_last_factor(self.handle, slot, _p(L), C.byref(ld), C.byref(jt)))
        return CorrelationFactor(L, ld.value, jt.value)

    def close(self):
        if getattr(self, "handle", None):
            lib().gpemu_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def neg2_log_profile(theta, data: Dataset, cfg: FitConfig, backend: Backend) -> ProfileEval:
    """likelihood.hpp:161-166: one evaluation, so a one-slot plan."""
    ev = ProfileEvaluator(data, cfg.p, cfg.nugget, backend, max_batch=1,
                          precision=cfg.precision)
    try:
        return ev.eval(theta)
    finally:
        ev.close()


class GpModel:
    """likelihood.hpp:171-182 with a device-resident factor (C-ABI gpemu_model)."""

    def __init__(self, handle, dataset, params, mu_hat, sigma2_hat, neg2, alpha, ctx):
        self.handle = handle
        self.dataset = dataset
        self.params = params
        self.mu_hat = mu_hat
        self.sigma2_hat = sigma2_hat
        self.neg2_log_lik = neg2
        self.alpha = alpha
        self.ctx = ctx

    @property
    def jitter_used(self) -> float:
        """factor.jitter_used of the model's factorization (backend.hpp:54-70)."""
        sc = np.empty(4)
        _check(lib().gpemu_model_scalars(self.handle, _p(sc)))
        return float(sc[3])

    def close(self):
        if getattr(self, "handle", None):
            lib().gpemu_model_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class GaGenerationRecord:
    best_value: float
    best_point: List[float]
    evaluations: int


@dataclass
class GaTrace:
    generations: List[GaGenerationRecord]


@dataclass
class FitResult:
    model: GpModel
    trace: GaTrace
    jitter_max: float
    ledger: LedgerCounts


class GeneticOptimizer:
    """The reference GA (optimizer.hpp:93-187) as a host state machine (C-ABI gpemu_ga_*;
    no device needed). thetas() -> the current generation (theta space), tell(fitness)."""

    def __init__(self, d: int, bounds, ga: GaConfig, seed: int):
        lo = _f64([b[0] for b in bounds])
        hi = _f64([b[1] for b in bounds])
        c = _GaConfigC(ga.population, ga.generations, ga.crossover_rate, ga.mutation_sigma,
                       ga.mutation_prob, ga.elitism)
        h = _vp()
        _check(lib().gpemu_ga_create(d, _p(lo), _p(hi), C.byref(c), C.c_uint64(seed), C.byref(h)))
        self.handle, self.d, self.P, self.G = h, d, ga.population, ga.generations

    def thetas(self) -> np.ndarray:
        out = np.empty((self.P, self.d))
        _check(lib().gpemu_ga_thetas(self.handle, _p(out)))
        return out

    def tell(self, fitness):
        f = _f64(fitness)
        assert f.shape == (self.P,)
        _check(lib().gpemu_ga_tell(self.handle, _p(f)))

    def status(self) -> dict:
        gen, done, sg, ss = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        bv = C.c_double()
        bt = np.zeros(self.d)
        tb = np.zeros(self.G)
        tg = np.zeros((self.G, self.d))
        _check(lib().gpemu_ga_status(self.handle, C.byref(gen), C.byref(done), C.byref(bv), _p(bt),
                                     C.byref(sg), C.byref(ss), _p(tb), _p(tg)))
        return dict(generation=gen.value, done=bool(done.value), best_value=bv.value,
                    best_theta=bt, stash_generation=sg.value, stash_slot=ss.value,
                    trace_best=tb[:gen.value], trace_genes=tg[:gen.value])

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                lib().gpemu_ga_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def fit_batch(data: Dataset, cfg: FitConfig, backend: Backend, reserve: float = 0.9) -> int:
    """Candidate slots for a fit: the whole GA population when its plan fits in `reserve` of the
    free device memory, else as many as fit (the generation is then evaluated in chunks, with
    the same candidates and the same theta-hat)."""
    prec = PRECISIONS[parse_precision(cfg.precision)]
    P = cfg.ga.population
    free, tot = C.c_size_t(), C.c_size_t()
    _check(lib().gpemu_ctx_mem_info(backend.ctx.handle, C.byref(free), C.byref(tot)))
    budget = reserve * free.value
    n, d = data.n(), data.d()
    if lib().gpemu_plan_bytes(n, d, P, prec) <= budget:
        return P
    lo, hi = 1, P
    while lo < hi:  # largest max_batch whose plan fits
        mid = (lo + hi + 1) // 2
        if lib().gpemu_plan_bytes(n, d, mid, prec) <= budget:
            lo = mid
        else:
            hi = mid - 1
    return lo


def fit_gp_detailed(data: Dataset, cfg: FitConfig, backend: Backend,
                    evaluator: Optional[ProfileEvaluator] = None) -> FitResult:
    """likelihood.hpp:243-303: one device batch per GA generation. `evaluator` may be a list
    of ProfileEvaluators of the same data on several devices: each generation is then split
    into contiguous candidate ranges, one per evaluator, run concurrently (gpemu_fit_multi);
    theta-hat and the trace are bitwise the one-device fit's."""
    d = data.d()
    bounds = cfg.bounds_for(d)
    own = evaluator is None
    ev = evaluator or ProfileEvaluator(data, cfg.p, cfg.nugget, backend,
                                       max_batch=fit_batch(data, cfg, backend),
                                       precision=cfg.precision)
    evs = list(ev) if isinstance(ev, (list, tuple)) else [ev]
    try:
        lo = _f64([b[0] for b in bounds])
        hi = _f64([b[1] for b in bounds])
        ga = _GaConfigC(cfg.ga.population, cfg.ga.generations, cfg.ga.crossover_rate,
                        cfg.ga.mutation_sigma, cfg.ga.mutation_prob, cfg.ga.elitism)
        res = _FitResultC()
        theta = np.empty(d)
        alpha = np.empty(data.n())
        tb = np.empty(cfg.ga.generations)
        tg = np.empty((cfg.ga.generations, d))
        mh = _vp()
        hs = (_vp * len(evs))(*[e.handle for e in evs])
        _check(lib().gpemu_fit_multi(hs, len(evs), _p(lo), _p(hi), C.byref(ga),
                                     C.c_uint64(cfg.seed), C.byref(res), _p(theta), _p(alpha),
                                     _p(tb), _p(tg), C.byref(mh)))
        led = backend.ledger()
        B = cfg.ga.budget()
        led.add_r_build(B)
        led.add_factorization(B)
        led.add_triangular_solves(2 * B + 2)
        model = GpModel(mh, data, Hyperparameters(list(theta), cfg.p, cfg.nugget), res.mu_hat,
                        res.sigma2_hat, res.neg2_log_lik, alpha, backend.ctx)
        model._contexts = [e.backend.ctx for e in evs]  # the model lives on one of them
        trace = GaTrace([GaGenerationRecord(float(tb[g]), list(tg[g]),
                                            (g + 1) * cfg.ga.population)
                         for g in range(cfg.ga.generations)])
        return FitResult(model, trace, res.jitter_max, led.snapshot())
    finally:
        if own:
            ev.close()


def eval_batch_multi(evaluators: Sequence[ProfileEvaluator], thetas) -> dict:
    """B independent evaluations sharded over several evaluators of the same data (one per
    device; contiguous ranges of ceil(B/G), concurrent host threads, gpemu_eval_batch_multi).
    Records come back in slot order, bitwise those of one evaluator."""
    T = _f64(np.atleast_2d(thetas))
    B = T.shape[0]
    out = {k: np.empty(B) for k in ("neg2", "mu", "sigma2", "jitter", "log_det")}
    st = np.empty(B, dtype=np.int32)
    hs = (_vp * len(evaluators))(*[e.handle for e in evaluators])
    _check(lib().gpemu_eval_batch_multi(hs, len(evaluators), _p(T), B, _p(out["neg2"]),
                                        _p(out["mu"]), _p(out["sigma2"]), _p(out["jitter"]),
                                        _p(out["log_det"]), st.ctypes.data_as(_ip)))
    out["status"] = st
    return out


def refine_fit(fit: FitResult, data: Dataset, cfg: FitConfig, backend: Backend,
               budget: int = 20) -> int:
    """bench.hpp:302-383 detail::refine_fit on the device: golden-section polish of the
    fitted theta with exactly `budget` extra evaluations; the model in `fit` is replaced when
    the polish improves -2logL. Returns the number of extra evaluations (budget, +1 when the
    model was rebuilt), as the reference's extra_evals."""
    d = data.d()
    bounds = cfg.bounds_for(d)
    lo = _f64([b[0] for b in bounds])
    hi = _f64([b[1] for b in bounds])
    # the polish evaluates in double whatever the run precision (bench.hpp:300-301); the model
    # is rebuilt in the run's precision (bench.hpp:363-382)
    # 8 slots let the polish evaluate each coordinate's golden-section decision tree in one
    # batch (same theta / -2logL / count as one-at-a-time, see gpemu_refine_fit_ex)
    free, tot = C.c_size_t(), C.c_size_t()
    _check(lib().gpemu_ctx_mem_info(backend.ctx.handle, C.byref(free), C.byref(tot)))
    mb = 8 if lib().gpemu_plan_bytes(data.n(), d, 8, 0) <= 0.9 * free.value else 1
    ev = ProfileEvaluator(data, cfg.p, cfg.nugget, backend, max_batch=mb)
    rb = ev if parse_precision(cfg.precision) == "double" else ProfileEvaluator(
        data, cfg.p, cfg.nugget, backend, max_batch=1, precision=cfg.precision)
    try:
        th = np.empty(d)
        sc = np.empty(4)
        alpha = np.empty(data.n())
        nv, used, mh = C.c_double(), C.c_int(), _vp()
        _check(lib().gpemu_refine_fit_ex(ev.handle, rb.handle, _p(lo), _p(hi),
                                         _p(_f64(fit.model.params.theta)),
                                         float(fit.model.neg2_log_lik), int(budget), _p(th),
                                         C.byref(nv), C.byref(used), C.byref(mh), _p(sc), _p(alpha)))
        extra = used.value
        if mh.value:
            extra += 1
            fit.model.close()
            fit.model = GpModel(mh, data, Hyperparameters(list(th), cfg.p, cfg.nugget),
                                float(sc[1]), float(sc[2]), float(sc[0]), alpha, backend.ctx)
        led = backend.ledger()
        led.add_r_build(extra)
        led.add_factorization(extra)
        led.add_triangular_solves(2 * extra + (2 if mh.value else 0))
        return extra
    finally:
        ev.close()
        if rb is not ev:
            rb.close()


def fit_gp(data: Dataset, cfg: FitConfig, backend: Backend) -> GpModel:
    return fit_gp_detailed(data, cfg, backend).model


def model_at_theta(data: Dataset, theta, p: float, nugget: float, backend: Backend,
                   precision: str = "double") -> GpModel:
    """likelihood.hpp:216-237 (precision 'single': the float instantiation)."""
    ev = ProfileEvaluator(data, p, nugget, backend, max_batch=1, precision=precision)
    try:
        th = _f64(theta)
        sc = np.empty(4)
        alpha = np.empty(data.n())
        mh = _vp()
        _check(lib().gpemu_model_at_theta(ev.handle, _p(th), C.byref(mh), _p(sc), _p(alpha)))
        led = backend.ledger()
        led.add_r_build()
        led.add_factorization()
        led.add_triangular_solves(4)
        return GpModel(mh, data, Hyperparameters(list(th), p, nugget), float(sc[1]), float(sc[2]),
                       float(sc[0]), alpha, backend.ctx)
    finally:
        ev.close()


# ---------------------------------------------------------------- predictor.hpp
def predict(model: GpModel, test_inputs, with_mse: bool = False):
    """predictor.hpp:20-50 (yhat); with_mse also returns the kriging MSE."""
    Xt = _f64(test_inputs)
    if Xt.ndim != 2 or Xt.shape[1] != model.dataset.d():
        raise ValidationError("predict: test input dimension mismatch")
    N = Xt.shape[0]
    yhat = np.empty(N)
    mse = np.empty(N) if with_mse else None
    _check(lib().gpemu_predict(model.handle, _p(Xt), N, _p(yhat), _p(mse)))
    return (yhat, mse) if with_mse else yhat


def model_alpha_residual(model: GpModel) -> float:
    """likelihood.hpp:191-213: ||(R + jitter I) alpha - (y - 1 mu)||_inf / ||y||_inf with R rebuilt
    from the stored hyperparameters (the GpModel contract keeps it <= 1e-6 in double)."""
    X = model.dataset.inputs()
    R = build_corr_matrix(X, model.params, model.ctx).values.copy()
    R[np.diag_indices_from(R)] += model.jitter_used
    y = model.dataset.outputs()
    row = R @ _f64(model.alpha)
    worst = float(np.max(np.abs(row - (y - model.mu_hat))))
    ymax = float(np.max(np.abs(y)))
    return worst / ymax if ymax > 0.0 else worst


@dataclass
class PredictionSet:
    """predictor.hpp:64-69."""
    test_inputs: np.ndarray
    predictions: np.ndarray
    sspe: float = 0.0


def predict_set(model: GpModel, test_inputs, truth=None) -> PredictionSet:
    """predictor.hpp:71-79: predictions plus, when truth is given, their SSPE."""
    Xt = _f64(test_inputs)
    out = PredictionSet(Xt, predict(model, Xt))
    if truth is not None and len(truth):
        out.sspe = sspe(out.predictions, truth)
    return out


def sspe(predictions, truth) -> float:
    """predictor.hpp:53-61."""
    a, b = _f64(predictions), _f64(truth)
    if a.shape != b.shape:
        raise ValidationError("sspe: length mismatch")
    e = b - a
    return float(np.dot(e, e))


# ---------------------------------------------------------------- experiment.hpp
@dataclass
class DesignSpec:
    """experiment.hpp:19-30."""
    n: int = 0
    d: int = 0
    seed: int = 0
    exchange_budget: int = 10000

    def validate(self):
        if self.n < 2:
            raise ValidationError("DesignSpec: n must be at least 2")
        if self.d < 1:
            raise ValidationError("DesignSpec: d must be at least 1")


def maximin_lhd(spec: DesignSpec, ctx: Optional[Context] = None, return_min: bool = False):
    """experiment.hpp:142-172: a random LHD and exchange_budget column-entry swaps, each kept only
    when it strictly raises the minimum pairwise distance. The random draws run on the host with
    the reference's RNG; the tracker and the swap scoring run on the device (kernels_design.cu).
    Returns the n x d design (bitwise the reference's) and, with return_min, its minimum squared
    pairwise distance (NaN when no exchange ran)."""
    spec.validate()
    ctx = ctx or default_context()
    x = np.empty((spec.n, spec.d))
    m = C.c_double(0.0)
    _check(lib().gpemu_maximin_lhd(ctx.handle, spec.n, spec.d, C.c_uint64(spec.seed & (2**64 - 1)),
                                   spec.exchange_budget, _p(x), C.byref(m)))
    return (x, m.value) if return_min else x
