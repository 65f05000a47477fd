"""GPU maximin Latin-hypercube design (experiment.hpp:142-172; kernels_design.cu) against the
reference itself: the design is compared BITWISE with the compiled reference (oracle/_ref, strict
and native builds), with the oracle restatement, and with the C1 golden's design, which the
reference generated (tools/make_golden.py)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def g():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_1203_1269_b200 import gpemu
    return gpemu


def min_sq_dist(X):
    """Minimum squared pairwise distance with the reference's summation order (sequential over k,
    every product and sum rounded separately, as numpy's elementwise ops are)."""
    n, d = X.shape
    s = np.zeros((n, n))
    for k in range(d):
        diff = X[:, k][:, None] - X[:, k][None, :]
        s = s + diff * diff
    s[np.diag_indices(n)] = np.inf
    return s.min()


def test_design_golden_c1(g, ctx):
    z = np.load(os.path.join(GOLD, "c1.npz"))
    X = g.maximin_lhd(g.DesignSpec(200, 2, 7, 10000), ctx)
    assert np.array_equal(X, z["X"])


SPECS = [(3, 1, 1, 50), (10, 3, 5, 1000), (200, 2, 7, 10000), (500, 6, 11, 5000),
         (1000, 10, 3, 3000), (64, 20, 13, 2000), (2, 4, 9, 100), (300, 3, 2, 0),
         (2500, 6, 21, 4000), (129, 1, 4, 3000)]


@pytest.mark.parametrize("spec", SPECS)
def test_design_bitwise_vs_reference(g, ctx, orc, ref, ref_fast, spec):
    n, d, seed, budget = spec
    X, m = g.maximin_lhd(g.DesignSpec(n, d, seed, budget), ctx, return_min=True)
    R = ref.maximin_lhd(n, d, seed, budget)
    assert np.array_equal(X, R), "design differs from the reference (strict build)"
    assert np.array_equal(X, ref_fast.maximin_lhd(n, d, seed, budget)), "differs from the native build"
    assert np.array_equal(X, orc.maximin_lhd(n, d, seed, budget))
    # Latin property: one point per stratum in every column
    for k in range(d):
        assert np.array_equal(np.sort(np.floor(X[:, k] * n)), np.arange(n))
    if budget > 0 and n > 2:
        assert m == min_sq_dist(X)
    else:
        assert np.isnan(m)


def test_design_large_vs_reference(g, ctx, ref):
    """n = 4096, d = 10 (the C3 design size): 16.8M pairs in the tracker, 2000 swaps."""
    n, d, seed, budget = 4096, 10, 17, 2000
    X = g.maximin_lhd(g.DesignSpec(n, d, seed, budget), ctx)
    assert np.array_equal(X, ref.maximin_lhd(n, d, seed, budget))


def test_design_validation(g, ctx):
    with pytest.raises(g.ValidationError):
        g.maximin_lhd(g.DesignSpec(1, 2, 0, 10), ctx)
    with pytest.raises(g.ValidationError):
        g.maximin_lhd(g.DesignSpec(5, 0, 0, 10), ctx)
