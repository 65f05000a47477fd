"""B200-native GP profile-deviance engine (arXiv 1203.1269 hot path).

The product is libgpemu_b200.so (sm_100a kernels + C-ABI, include/gpemu_b200.h);
`gpemu` mirrors the reference's gpemu API on top of it.
"""
from . import gpemu  # noqa: F401
from .gpemu import (Backend, ConfigError, Context, CorrelationFactor, CorrelationMatrix,  # noqa: F401
                    CorrelationPlan, Dataset, Error, FitConfig, FitError, GaConfig,
                    Hyperparameters, NotPositiveDefiniteError, ProfileEvaluator, ValidationError,
                    build_corr_matrix, corr_vector, fit_gp, fit_gp_detailed, make_backend,
                    model_at_theta, new_dataset, predict, sspe)

__all__ = [n for n in dir() if not n.startswith("_")]
