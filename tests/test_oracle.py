"""CPU: pin the oracle (C restatement, oracle/gpemu_oracle.c) to the reference.

Known answers are the reference tests' own (file:line cited); golden fixtures were
produced by the UNMODIFIED reference (tools/make_golden.py -> oracle/_ref).
"""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def rel_diff(a, b):  # test_helpers.hpp:14-17
    den = max(abs(a), abs(b))
    return 0.0 if den == 0 else abs(a - b) / den


def test_known_answers_correlation(orc):
    # test_correlation.cpp:22-29 coincident points correlate perfectly
    R = orc.build_corr(np.array([[0.2, 0.7], [0.2, 0.7]]), [3.0, 5.0], 1.95)
    assert np.all(R == 1.0)
    # :31-37 zero decay -> all ones
    assert np.all(orc.build_corr(np.array([[0.1], [0.4], [0.9]]), [0.0], 1.95) == 1.0)
    # :39-44 exp(-2)
    assert rel_diff(orc.build_corr(np.array([[0.0], [1.0]]), [2.0], 1.95)[0, 1], 0.1353352832366127) < 1e-15
    # :60-65 gaussian special case
    assert rel_diff(orc.corr_vector([0.5], np.array([[0.0]]), [1.0], 2.0)[0], 0.7788007830714049) < 1e-15


def test_known_answers_backend(orc):
    L, ld, jt = orc.factorize(np.array([[1.0, 0.5], [0.5, 1.0]]), kind=0)
    # test_backend.cpp:48-56
    assert L[0, 0] == 1.0 and L[1, 0] == 0.5
    assert rel_diff(L[1, 1], 0.8660254037844386) < 1e-15
    assert rel_diff(ld, -0.2876820724517809) < 1e-12 and jt == 0.0
    # :96-101 and :116-121
    u = orc.solve_lower(L, np.array([1.0, 1.0]))
    assert u[0] == 1.0 and rel_diff(u[1], 0.5773502691896258) < 1e-15
    x = orc.solve_upper(L, u)
    assert rel_diff(x[0], 2 / 3) < 1e-12 and rel_diff(x[1], 2 / 3) < 1e-12
    # :81-87 ladder exhaustion
    assert orc.factorize(np.array([[1.0, 2.0], [2.0, 1.0]])) is None
    # :58-79 coincident points force the ladder
    Xc = np.array([[0.3, 0.3], [0.3, 0.3], [0.7, 0.1]])
    f = orc.factorize(orc.build_corr(Xc, [2.0, 2.0], 1.95))
    assert f[2] > 0.0 and f[2] in (1e-8, 1e-7, 1e-6, 1e-5, 1e-4)


def test_spec_profile_example(orc):
    # SPEC.md:245 / SURVEY 8(c): X=[[0],[1]], y=[0,1], theta=2, p=1.95
    r = orc.eval_batch(np.array([[0.0], [1.0]]), np.array([0.0, 1.0]), np.array([[2.0]]), 1.95)
    assert rel_diff(r["neg2"][0], -1.113952892208059) < 1e-13
    assert r["mu"][0] == 0.5 and rel_diff(r["sigma2"][0], 0.28912941068741643) < 1e-14


def test_oracle_matches_reference_kat_fixture(orc):
    z = np.load(os.path.join(GOLD, "kat.npz"))
    assert orc.build_corr(np.array([[0.0], [1.0]]), [2.0], 1.95)[0, 1] == z["r_unit"]
    L, ld, jt = orc.factorize(np.array([[1.0, 0.5], [0.5, 1.0]]), kind=0)
    assert np.array_equal(np.tril(L), np.tril(z["L22"])) and ld == z["logdet22"]
    Lc, ldc, jtc = orc.factorize(z["Rc"])
    assert np.array_equal(np.tril(Lc), np.tril(z["Lc"])) and ldc == z["ldc"] and jtc == z["jitc"]
    r = orc.eval_batch(np.array([[0.0], [1.0]]), np.array([0.0, 1.0]), np.array([[2.0]]), 1.95)
    assert r["neg2"][0] == z["spec_neg2"] and r["sigma2"][0] == z["spec_sigma2"]


@pytest.mark.parametrize("name", ["c1", "c1p195"])
def test_oracle_bitwise_on_c1_goldens(orc, name):
    z = np.load(os.path.join(GOLD, f"{name}.npz"))
    X, y, p = z["X"], z["y"], float(z["p"])
    # design generation (experiment.hpp:142-172) and simulator are bitwise the reference's
    assert np.array_equal(orc.maximin_lhd(200, 2, 7, 10000), X)
    assert np.array_equal(orc.goldstein_price_log(X), y)
    r = orc.eval_batch(X, y, z["thetas"], p)
    for k in ("neg2", "mu", "sigma2", "jitter", "log_det"):
        assert np.array_equal(r[k], z[k]), k


def test_oracle_fit_and_predict_c1(orc):
    z = np.load(os.path.join(GOLD, "c1.npz"))
    X, y = z["X"], z["y"]
    f = orc.fit(X, y, p=2.0, population=100, generations=20, seed=0)
    assert np.array_equal(f["theta"], z["fit_theta"])
    assert f["neg2"] == z["fit_neg2"] and f["mu"] == z["fit_mu"]
    assert np.array_equal(f["trace_best"], z["trace_best"])
    assert np.array_equal(f["trace_genes"], z["trace_genes"])
    assert np.array_equal(f["alpha"], z["fit_alpha"])
    yhat = orc.predict(X, f["theta"], 2.0, f["mu"], f["alpha"], z["Xt"])
    assert np.array_equal(yhat, z["yhat"])


def test_oracle_c2_subset(orc):
    z = np.load(os.path.join(GOLD, "c2.npz"))
    r = orc.eval_batch(z["X"], z["y"], z["thetas"][:2], 1.95)
    for k in ("neg2", "mu", "sigma2", "jitter", "log_det"):
        assert np.array_equal(r[k], z[k][:2]), k


def test_oracle_vs_reference_random(orc, ref):
    rng = np.random.default_rng(5)
    for n, d in ((9, 2), (40, 3), (70, 1)):
        X = rng.random((n, d))
        y = np.sin(3 * X).sum(1)
        th = rng.uniform(0.3, 5.0, size=(5, d))
        a = orc.eval_batch(X, y, th, 1.95)
        b = ref.eval_batch(X, y, th, 1.95)
        assert np.array_equal(a["neg2"], b["neg2"])
        assert np.array_equal(orc.build_corr(X, th[0], 1.7), ref.build_corr(X, th[0], 1.7))
        assert np.array_equal(orc.plan_build(X, th[0], 1.7, 0.01), ref.plan_build(X, th[0], 1.7, 0.01))


def test_rng_streams_match_reference(orc, ref):
    import ctypes as C
    r = ref.rng_draws(12345, 1, 1000)
    from oracle.oracle import _GaConfig  # noqa: F401
    st = (C.c_uint64 * 313)()
    orc.lib.orc_rng_init.argtypes = [C.c_void_p, C.c_uint64]
    orc.lib.orc_rng_uniform01.restype = C.c_double
    orc.lib.orc_rng_uniform01.argtypes = [C.c_void_p]
    orc.lib.orc_rng_init(C.addressof(st), 12345)
    mine = np.array([orc.lib.orc_rng_uniform01(C.addressof(st)) for _ in range(1000)])
    assert np.array_equal(mine, r)
    assert orc.derive_seed(7, 0x1D64) == ref.lib.ref_derive_seed2(7, 0x1D64)


def test_mse_restatement_properties(orc):
    # MSE has no reference: check the restatement's defining properties.
    z = np.load(os.path.join(GOLD, "c1p195.npz"))
    X, y = z["X"][:60], z["y"][:60]
    th = np.array([3.0, 2.0])
    R = orc.build_corr(X, th, 1.95)
    L, ld, jt = orc.factorize(R)
    sigma2 = 1.7
    # interpolation: MSE at a training point is ~0
    m = orc.kriging_mse(X, th, 1.95, sigma2, L, X[:5])
    assert np.all(m < 1e-8 * sigma2)
    # explicit-inverse form (oracles.hpp style) at random points
    Xt = np.random.default_rng(1).random((7, 2))
    m = orc.kriging_mse(X, th, 1.95, sigma2, L, Xt)
    Ri = np.linalg.inv(R)
    one = np.ones(len(X))
    for j in range(len(Xt)):
        r = orc.corr_vector(Xt[j], X, th, 1.95)
        want = sigma2 * (1 - r @ Ri @ r + (1 - one @ Ri @ r) ** 2 / (one @ Ri @ one))
        assert abs(m[j] - max(want, 0.0)) < 1e-6 * sigma2


@pytest.mark.parametrize("name", ["x_d20_nugget", "x_p1", "x_d1"])
def test_oracle_bitwise_on_extra_goldens(orc, name):
    z = np.load(os.path.join(GOLD, f"{name}.npz"))
    r = orc.eval_batch(z["X"], z["y"], z["thetas"], float(z["p"]), float(z["nugget"]))
    for k in ("neg2", "mu", "sigma2", "jitter", "log_det"):
        assert np.array_equal(r[k], z[k]), k


def test_oracle_refine_fit_golden(orc):
    """bench.hpp:302-383 refine_fit: the oracle's GA fit and golden-section polish reproduce the
    reference's theta / -2logL bitwise (tests/golden/refine.npz, tools/make_golden_refine.py)."""
    z = np.load(os.path.join(GOLD, "refine.npz"))
    for k in range(int(z["ncases"])):
        X, y, p = z[f"X_{k}"], z[f"y_{k}"], float(z[f"p_{k}"])
        P, G, seed = (int(v) for v in z[f"ga_{k}"])
        f = orc.fit(X, y, p=p, population=P, generations=G, seed=seed)
        assert np.array_equal(f["theta"], z[f"theta_fit_{k}"]) and f["neg2"] == z[f"neg2_fit_{k}"]
        th, nv, used = orc.refine_fit(X, y, f["theta"], f["neg2"], p=p)
        assert used == 20 and int(z[f"extra_{k}"]) == 21
        assert np.array_equal(th, z[f"theta_ref_{k}"]), k
        assert nv == z[f"neg2_ref_{k}"], k
