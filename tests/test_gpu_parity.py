"""GPU parity: the sm_100a path (through the C-ABI) against the oracle and the
reference-generated golden fixtures.

Gates:
  * R, corr_vector: elementwise relative <= 1e-14 (libdevice exp/log vs glibc: not bitwise)
  * per candidate -2logL: |gpu-ref|/|ref| <= max(1e-9, 10 * reference self-discrepancy,
    3 * reference error vs the long-double truth, 10 * sensitivity to 1-ulp perturbations of R);
    self-discrepancy = the reference's own `reference` vs `parallel` backends in its native
    build; truth = oracle eval_truth (80-bit) of the same double R; sensitivity = oracle
    eval_sensitivity (80-bit, random 1-ulp relative perturbations of R's off-diagonal). The jitter step and the +inf status must be EQUAL, and the device's
    median error vs truth must not exceed twice the reference's.
  * GA argmin theta-hat and the per-generation trace: bitwise equal
  * predictions: max|yhat-ref| / max(|yhat|, |y|_inf) <= max(1e-8, 10 * reference self-disc.)
  * simple engine on identical R: bitwise equal to ReferenceBackend
"""
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


def rel(a, b):
    a, b = np.atleast_1d(np.asarray(a, dtype=float)), np.atleast_1d(np.asarray(b, dtype=float))
    den = np.maximum(np.abs(a), np.abs(b))
    den[den == 0] = 1.0
    return float(np.max(np.abs(a - b) / den)) if a.size else 0.0


def gate_neg2(got, z):
    """Per candidate: |gpu-ref|/|ref| <= max(1e-9, 10*self_disc, 3*|ref-truth|/|truth|,
    10*sens), and in aggregate the device is at least as close to the long-double truth as
    the reference."""
    want, self_disc, truth, sens = z["neg2"], z["self_disc"], z["truth"], z["sens"]
    fin = np.isfinite(want)
    assert np.array_equal(np.isinf(got), np.isinf(want)), "+inf status differs"
    r = np.abs(got[fin] - want[fin]) / np.abs(want[fin])
    ref_err = np.abs(want[fin] - truth[fin]) / np.abs(truth[fin])
    dev_err = np.abs(got[fin] - truth[fin]) / np.abs(truth[fin])
    tol = np.maximum(np.maximum(1e-9, 10.0 * self_disc[fin]),
                     np.maximum(3.0 * ref_err, 10.0 * sens[fin]))
    bad = np.nonzero(r > tol)[0]
    assert bad.size == 0, f"{bad.size} candidates over gate; worst rel {r.max():.3e}"
    assert np.median(dev_err) <= 2.0 * np.median(ref_err) + 1e-15, (np.median(dev_err), np.median(ref_err))
    return float(r.max()) if r.size else 0.0


# ---------------------------------------------------------------- correlation
def test_corr_known_answers(g, ctx):
    R = g.build_corr_matrix([[0.2, 0.7], [0.2, 0.7]], g.Hyperparameters([3.0, 5.0]), ctx).values
    assert np.all(R == 1.0)
    R = g.build_corr_matrix([[0.1], [0.4], [0.9]], g.Hyperparameters([0.0]), ctx).values
    assert np.all(R == 1.0)
    R = g.build_corr_matrix([[0.0], [1.0]], g.Hyperparameters([2.0]), ctx).values
    assert rel(R[0, 1], 0.1353352832366127) < 1e-15
    r = g.corr_vector([0.5], [[0.0]], g.Hyperparameters([1.0], 2.0), ctx)
    assert rel(r[0], 0.7788007830714049) < 1e-15
    with pytest.raises(g.ValidationError):
        g.corr_vector([0.5], [[0.1, 0.3], [0.6, 0.9]], g.Hyperparameters([1.0, 1.0]), ctx)


def test_corr_matches_oracle(g, ctx, orc):
    rng = np.random.default_rng(7781)
    for it in range(10):
        n, d = 2 + int(rng.integers(60)), 1 + int(rng.integers(5))
        X = rng.random((n, d))
        th = rng.uniform(0.0, 8.0, d)
        nug = 0.05 if it % 3 == 0 else 0.0
        R = g.build_corr_matrix(X, g.Hyperparameters(th, 1.95, nug), ctx).values
        assert rel(R, orc.build_corr(X, th, 1.95, nug)) < 1e-14
        assert np.array_equal(R, R.T)
        assert np.all(np.diag(R) == 1.0 + nug)
        # corr_vector equals a matrix row minus the nugget, bitwise (test_correlation.cpp:142-162)
        v = g.corr_vector(X[1], X, g.Hyperparameters(th, 1.95, nug), ctx)
        row = R[1].copy()
        row[1] -= nug
        assert np.array_equal(v, row)


# ---------------------------------------------------------------- backend
@pytest.mark.parametrize("engine", ["simple", "dag"])
def test_factorize_known_answers(g, engine):
    be = g.Backend(g.Context(0, engine))
    f = be.factorize(g.CorrelationMatrix(np.eye(2)))
    assert f.lower[0, 0] == 1.0 and f.lower[1, 1] == 1.0 and f.lower[1, 0] == 0.0
    assert f.log_det == 0.0 and f.jitter_used == 0.0
    f = be.factorize(g.CorrelationMatrix(np.array([[1.0, 0.5], [0.5, 1.0]])))
    assert f.lower[0, 0] == 1.0 and f.lower[1, 0] == 0.5
    assert rel(f.lower[1, 1], 0.8660254037844386) < 1e-15
    assert rel(f.log_det, -0.2876820724517809) < 1e-12
    u = be.solve_lower(f, [1.0, 1.0])
    assert u[0] == 1.0 and rel(u[1], 0.5773502691896258) < 1e-15
    x = be.solve_full(f, [1.0, 1.0])
    assert rel(x, [2 / 3, 2 / 3]) < 1e-12
    with pytest.raises(g.NotPositiveDefiniteError):
        be.factorize(g.CorrelationMatrix(np.array([[1.0, 2.0], [2.0, 1.0]])))
    Xc = np.array([[0.3, 0.3], [0.3, 0.3], [0.7, 0.1]])
    R = g.build_corr_matrix(Xc, g.Hyperparameters([2.0, 2.0]), be.ctx)
    f = be.factorize(R)
    assert f.jitter_used in (1e-8, 1e-7, 1e-6, 1e-5, 1e-4)
    LLt = f.lower @ f.lower.T
    assert np.max(np.abs(np.tril(LLt - R.values - f.jitter_used * np.eye(3)))) <= 1e-8 * 3


def test_simple_engine_bitwise_reference_cholesky(g, orc):
    be = g.Backend(g.Context(0, "simple"))
    rng = np.random.default_rng(222)
    for n in (5, 40, 100, 300):
        X = rng.random((n, 2))
        R = orc.build_corr(X, rng.uniform(0.3, 5.0, 2) * 10, 1.95)
        f = be.factorize(g.CorrelationMatrix(R))
        L, ld, jt = orc.factorize(R, kind=0)
        assert np.array_equal(f.lower, np.tril(L)) and f.log_det == ld and f.jitter_used == jt


@pytest.mark.parametrize("n", [7, 64, 130, 257, 300, 640])
def test_dag_factorize_reconstruction(g, orc, n):
    be = g.Backend(g.Context(0, "dag"))
    rng = np.random.default_rng(n)
    X = rng.random((n, 3))
    R = orc.build_corr(X, rng.uniform(0.3, 5.0, 3), 1.95)
    f = be.factorize(g.CorrelationMatrix(R))
    L, ld, jt = orc.factorize(R)
    assert f.jitter_used == jt
    assert abs(f.log_det - ld) <= 1e-10 * max(1.0, abs(ld))
    # reconstruction bound (test_backend.cpp:155-174)
    err = np.max(np.abs(np.tril(f.lower @ f.lower.T - R - jt * np.eye(n))))
    assert err <= 1e-8 * n
    # solve round-trip (test_backend.cpp:176-196)
    x = rng.uniform(-1, 1, n)
    b = f.lower @ (f.lower.T @ x)
    assert rel(be.solve_full(f, b), x) < 1e-6


# ---------------------------------------------------------------- deviance
@pytest.mark.parametrize("engine", ["simple", "dag"])
@pytest.mark.parametrize("name", ["c1", "c1p195"])
def test_eval_batch_c1_goldens(g, name, engine):
    z = np.load(os.path.join(GOLD, f"{name}.npz"))
    be = g.Backend(g.Context(0, engine))
    ev = g.ProfileEvaluator(g.new_dataset(z["X"], z["y"]), float(z["p"]), 0.0, be, max_batch=100)
    r = ev.eval_batch(z["thetas"])
    assert np.array_equal(r["jitter"], z["jitter"])
    gate_neg2(r["neg2"], z)
    fin = np.isfinite(z["neg2"])
    # log|R| is part of -2logL (gated above); near-singular thetas move it at ~1e-8
    assert rel(r["log_det"][fin], z["log_det"][fin]) < 1e-7
    ev.close()


def test_eval_batch_c2_golden(g, ctx):
    """Config C2: the full 64-candidate batch (n=2048, d=6, p=1.95) in one device batch."""
    z = np.load(os.path.join(GOLD, "c2.npz"))
    assert z["thetas"].shape == (64, 6)
    ev = g.ProfileEvaluator(g.new_dataset(z["X"], z["y"]), 1.95, 0.0, g.Backend(ctx), max_batch=64)
    r = ev.eval_batch(z["thetas"])
    assert np.array_equal(r["jitter"], z["jitter"])
    gate_neg2(r["neg2"], z)
    ev.close()


def test_batch_invariance(g, ctx):
    """Same theta in any slot / batch size -> bitwise identical record."""
    z = np.load(os.path.join(GOLD, "c1p195.npz"))
    ev = g.ProfileEvaluator(g.new_dataset(z["X"], z["y"]), 1.95, 0.0, g.Backend(ctx), max_batch=100)
    a = ev.eval_batch(z["thetas"])
    perm = np.random.default_rng(3).permutation(100)
    b = ev.eval_batch(z["thetas"][perm])
    c = ev.eval_batch(z["thetas"][17:21])
    for k in ("neg2", "mu", "sigma2", "jitter", "log_det"):
        assert np.array_equal(a[k][perm], b[k]), k
        assert np.array_equal(a[k][17:21], c[k]), k
    single = ev.eval(z["thetas"][42])
    assert single.neg2_log_lik == a["neg2"][42]
    ev.close()


def test_ladder_mixed_batch(g, ctx, orc):
    """Coincident design points: some thetas need jitter, the ladder reruns only those."""
    X = np.array([[0.3, 0.3], [0.3, 0.3], [0.7, 0.1], [0.2, 0.9], [0.55, 0.45]])
    y = np.array([1.0, 1.0, -0.5, 0.25, 0.75])
    th = np.array([[2.0, 2.0], [0.5, 7.0], [11.0, 0.1], [1e-6, 1e-6]])
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=4)
    r = ev.eval_batch(th)
    o = orc.eval_batch(X, y, th, 1.95)
    assert np.array_equal(r["jitter"], o["jitter"])
    assert np.array_equal(np.isinf(r["neg2"]), np.isinf(o["neg2"]))
    assert rel(r["neg2"], o["neg2"]) < 1e-6
    ev.close()


def test_large_n_property_checks(g, ctx, orc):
    """n=2048 / d=6 at B=4: factor reconstruction and deviance recomputed from the factor."""
    import torch
    z = np.load(os.path.join(GOLD, "c2.npz"))
    ev = g.ProfileEvaluator(g.new_dataset(z["X"], z["y"]), 1.95, 0.0, g.Backend(ctx), max_batch=4)
    r = ev.eval_batch(z["thetas"][:4])
    for s in range(4):
        f = ev.last_factor(s)
        Lt = torch.from_numpy(f.lower).cuda()
        R = torch.from_numpy(g.build_corr_matrix(z["X"], g.Hyperparameters(z["thetas"][s], 1.95),
                                                 ctx).values).cuda()
        err = torch.max(torch.abs(torch.tril(Lt @ Lt.T - R))).item()
        assert err <= 1e-8 * 2048
        assert abs(f.log_det - 2 * np.sum(np.log(np.diag(f.lower)))) <= 1e-9 * abs(f.log_det)
        # deviance from the factor by an independent route (torch triangular solves)
        y = torch.from_numpy(z["y"]).cuda()[:, None]
        one = torch.ones_like(y)
        u = torch.linalg.solve_triangular(Lt, y, upper=False)
        v = torch.linalg.solve_triangular(Lt, one, upper=False)
        utu, vtu, vtv = (u * u).sum().item(), (v * u).sum().item(), (v * v).sum().item()
        mu = vtu / vtv
        s2 = max(0.0, (utu - 2 * mu * vtu + mu * mu * vtv) / 2048)
        neg2 = f.log_det + 2048 * np.log(max(2048 * s2, np.finfo(float).tiny))
        assert abs(neg2 - r["neg2"][s]) <= 1e-9 * abs(neg2) + 1e-12
    ev.close()


# ---------------------------------------------------------------- fit + predict
def test_fit_c1_argmin_bitwise(g, ctx, orc):
    z = np.load(os.path.join(GOLD, "c1.npz"))
    data = g.new_dataset(z["X"], z["y"])
    cfg = g.FitConfig(ga=g.GaConfig(population=100, generations=20), seed=0, p=2.0)
    be = g.Backend(ctx)
    fr = g.fit_gp_detailed(data, cfg, be)
    assert np.array_equal(np.array(fr.model.params.theta), z["fit_theta"])
    assert np.array_equal(np.array([r.best_point for r in fr.trace.generations]), z["trace_genes"])
    # at the optimum, the same conditioning-aware gate as per candidate: <= max(1e-9, 3 x the
    # reference's own error vs the long-double truth, 10 x the 1-ulp sensitivity of -2logL)
    ref_err = abs(z["fit_neg2"] - z["fit_truth"]) / abs(z["fit_truth"])
    _, sens = orc.eval_sensitivity(z["X"], z["y"], z["fit_theta"][None, :], 2.0,
                                   [z["fit_jitter_max"]], reps=3)
    tol = max(1e-9, 3 * ref_err, 10 * sens[0])
    assert abs(fr.model.neg2_log_lik - z["fit_neg2"]) <= tol * abs(z["fit_neg2"])
    assert fr.jitter_max == z["fit_jitter_max"]
    led = fr.ledger  # SPEC.md:499 cost model: 2000 / 2000 / 4002
    assert (led.r_builds, led.factorizations, led.triangular_solves) == (2000, 2000, 4002)
    yhat, mse = g.predict(fr.model, z["Xt"], with_mse=True)
    scale = max(np.abs(z["yhat"]).max(), np.abs(z["y"]).max())
    tol = max(1e-8, 10 * float(z["yhat_self_disc"]))
    assert np.max(np.abs(yhat - z["yhat"])) / scale <= tol
    assert np.all(mse >= 0.0)


def test_refine_fit_bitwise(g, ctx):
    """bench.hpp:302-383: device GA fit + golden-section polish reproduce the reference's
    fitted and polished theta bitwise (tests/golden/refine.npz); -2logL within 1e-9."""
    z = np.load(os.path.join(GOLD, "refine.npz"))
    be = g.Backend(ctx)
    for k in range(int(z["ncases"])):
        X, y, p = z[f"X_{k}"], z[f"y_{k}"], float(z[f"p_{k}"])
        P, G, seed = (int(v) for v in z[f"ga_{k}"])
        data = g.new_dataset(X, y)
        cfg = g.FitConfig(ga=g.GaConfig(population=P, generations=G), seed=seed, p=p)
        fr = g.fit_gp_detailed(data, cfg, be)
        assert np.array_equal(np.array(fr.model.params.theta), z[f"theta_fit_{k}"]), k
        extra = g.refine_fit(fr, data, cfg, be)
        assert extra == int(z[f"extra_{k}"])
        assert np.array_equal(np.array(fr.model.params.theta), z[f"theta_ref_{k}"]), k
        assert rel(fr.model.neg2_log_lik, z[f"neg2_ref_{k}"]) <= 1e-9
        yhat = g.predict(fr.model, X[:10])  # the rebuilt model interpolates
        assert np.max(np.abs(yhat - y[:10])) <= 1e-6 * np.abs(y).max()


@pytest.mark.parametrize("name", ["c2fit", "c3fit"])
def test_fit_large_argmin_bitwise(g, ctx, name):
    """Full GA (100x20) at C2 / C3 sizes: theta-hat and the per-generation best genes are
    bitwise the reference's (tests/golden/<name>.npz, tools/make_golden_fit.py)."""
    path = os.path.join(GOLD, name + ".npz")
    if not os.path.exists(path):
        pytest.skip(name + " golden not generated")
    z = np.load(path)
    data = g.new_dataset(z["X"], z["y"])
    cfg = g.FitConfig(ga=g.GaConfig(population=100, generations=20), seed=0, p=float(z["p"]))
    fr = g.fit_gp_detailed(data, cfg, g.Backend(ctx))
    assert np.array_equal(np.array(fr.model.params.theta), z["theta"])
    assert np.array_equal(np.array([r.best_point for r in fr.trace.generations]), z["trace_genes"])
    assert rel(np.array([r.best_value for r in fr.trace.generations]), z["trace_best"]) <= 1e-9
    assert rel(fr.model.neg2_log_lik, z["neg2"]) <= 1e-9
    assert fr.jitter_max == z["jitter_max"]


def test_predict_and_mse_vs_oracle(g, ctx, orc):
    z = np.load(os.path.join(GOLD, "c1p195.npz"))
    X, y = z["X"], z["y"]
    th = np.array([3.0, 2.0])
    m = g.model_at_theta(g.new_dataset(X, y), th, 1.95, 0.0, g.Backend(ctx))
    mp = orc.eval_batch(X, y, th[None, :], 1.95)
    assert rel(m.neg2_log_lik, mp["neg2"][0]) < 1e-9
    R = orc.build_corr(X, th, 1.95)
    L, ld, jt = orc.factorize(R)
    alpha = orc.solve_upper(L, orc.solve_lower(L, y - mp["mu"][0]))
    Xt = z["Xt"][:200]
    yo = orc.predict(X, th, 1.95, mp["mu"][0], alpha, Xt)
    yhat, mse = g.predict(m, Xt, with_mse=True)
    scale = max(np.abs(yo).max(), np.abs(y).max())
    assert np.max(np.abs(yhat - yo)) / scale <= 1e-8
    mo = orc.kriging_mse(X, th, 1.95, mp["sigma2"][0], L, Xt)
    assert np.max(np.abs(mse - mo)) <= 1e-8 * mp["sigma2"][0]
    # interpolation: yhat at training points reproduces y, MSE ~ 0
    yt, mt = g.predict(m, X[:20], with_mse=True)
    assert np.max(np.abs(yt - y[:20])) <= 1e-6 * np.abs(y).max()
    assert np.all(mt <= 1e-8 * mp["sigma2"][0])
    with pytest.raises(g.ValidationError):
        g.predict(m, np.array([[0.5, 1.5]]))


def test_mse_extension_rows_multi_tile(g, ctx, orc):
    """MSE through the DAG extension mode across several tile rows/cols (n=700, N=300)."""
    rng = np.random.default_rng(77)
    n, d = 700, 3
    X = rng.random((n, d))
    y = np.sin(3 * X).sum(1) + 0.5 * (X * X).sum(1)
    th = np.array([4.0, 2.5, 6.0])
    m = g.model_at_theta(g.new_dataset(X, y), th, 1.95, 0.0, g.Backend(ctx))
    ref = orc.eval_batch(X, y, th[None, :], 1.95)
    L, ld, jt = orc.factorize(orc.build_corr(X, th, 1.95))
    Xt = rng.random((300, d))
    yhat, mse = g.predict(m, Xt, with_mse=True)
    mo = orc.kriging_mse(X, th, 1.95, ref["sigma2"][0], L, Xt)
    assert np.max(np.abs(mse - mo)) <= 1e-7 * ref["sigma2"][0]
    alpha = orc.solve_upper(L, orc.solve_lower(L, y - ref["mu"][0]))
    yo = orc.predict(X, th, 1.95, ref["mu"][0], alpha, Xt)
    assert np.max(np.abs(yhat - yo)) <= 1e-8 * max(np.abs(yo).max(), np.abs(y).max())
    # yhat from the cross tiles (MSE path) is the yhat-only kernel's value, bit for bit
    assert np.array_equal(yhat, g.predict(m, Xt))
    n2 = 1200  # two training blocks of 1024 rows, ragged last tile
    X2 = rng.random((n2, d))
    y2 = np.sin(3 * X2).sum(1)
    m2 = g.model_at_theta(g.new_dataset(X2, y2), th, 1.95, 0.0, g.Backend(ctx))
    Xt2 = rng.random((257, d))
    yh2, _ = g.predict(m2, Xt2, with_mse=True)
    assert np.array_equal(yh2, g.predict(m2, Xt2))
    assert np.array_equal(g.predict(m2, Xt2[100:101]), yh2[100:101])  # independent of N


@pytest.mark.parametrize("engine", ["simple", "dag"])
@pytest.mark.parametrize("name", ["x_d20_nugget", "x_p1", "x_d1"])
def test_eval_batch_extra_shapes(g, name, engine):
    """d=20 with a nugget (C4-like), the exponential kernel p=1, and d=1 (nugget 0.01)."""
    z = np.load(os.path.join(GOLD, f"{name}.npz"))
    be = g.Backend(g.Context(0, engine))
    ev = g.ProfileEvaluator(g.new_dataset(z["X"], z["y"]), float(z["p"]), float(z["nugget"]), be,
                            max_batch=16)
    r = ev.eval_batch(z["thetas"])
    assert np.array_equal(r["jitter"], z["jitter"])
    gate_neg2(r["neg2"], z)
    fin = np.isfinite(z["neg2"])
    assert rel(r["mu"][fin], z["mu"][fin]) < 1e-6
    ev.close()


def test_c4_full_size_vs_reference(g, ctx):
    """Largest config at full size (C4: n=16384, d=20, p=1.9, nugget 1e-8): the deviance record
    of two thetas against the reference's own evaluation (tests/golden/c4_full.npz,
    tools/make_golden_c4.py), gated on the reference's self-discrepancy between its two builds;
    plus batch invariance at this size."""
    path = os.path.join(GOLD, "c4_full.npz")
    if not os.path.exists(path):
        pytest.skip("c4_full golden not generated")
    z = np.load(path)
    n, d = int(z["n"]), int(z["d"])
    rng = np.random.default_rng(int(z["seed"]))
    X = np.empty((n, d))
    for k in range(d):
        X[:, k] = (rng.permutation(n) + rng.random(n)) / n
    y = (np.sin(3.0 * X + 0.37 * np.arange(d)) + 0.5 * X * X).sum(1)
    ev = g.ProfileEvaluator(g.new_dataset(X, y), float(z["p"]), float(z["nugget"]), g.Backend(ctx),
                            max_batch=2)
    r = ev.eval_batch(z["thetas"])
    assert np.array_equal(r["jitter"], z["jitter_strict"])
    for k, floor in (("neg2", 1e-9), ("log_det", 1e-9), ("mu", 1e-8), ("sigma2", 1e-8)):
        self_disc = rel(z[f"{k}_strict"], z[f"{k}_fast"])
        assert rel(r[k], z[f"{k}_strict"]) <= max(floor, 10 * self_disc), k
    r1 = ev.eval_batch(z["thetas"][1:])
    assert r1["neg2"][0] == r["neg2"][1]  # slot 0 of a batch of 1 == slot 1 of a batch of 2
    ev.close()


# ---------------------------------------------------------------- single precision
def _f32_case(seed, n, d):
    rng = np.random.default_rng(seed)
    X = rng.random((n, d))
    y = np.sin(3 * X).sum(1) + 0.3 * X[:, 0]
    th = 10 ** rng.uniform(-1.0, 0.5, size=(12, d))
    return X, y, th


@pytest.mark.parametrize("n,d", [(200, 2), (700, 3), (1100, 5)])
def test_single_precision_eval_vs_reference(g, ctx, ref_fast, n, d):
    """Precision::kSingle (core.hpp:86-96): the device float engine against the reference's
    float instantiation (ProfileEvaluator<float>). Float results differ from double by the
    float path's own error, so the gate is relative to it: per candidate with the same jitter
    step |dev - ref_f32| <= max(1e-5, 10 |ref_f32 - ref_f64|) (relative), and in aggregate
    the device float is at least as close to the double result as the reference float."""
    X, y, th = _f32_case(n + d, n, d)
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=12,
                            precision="single")
    r = ev.eval_batch(th)
    fs = ref_fast.eval_batch(X, y, th, 1.95, threads=0, precision="single")
    fd = ref_fast.eval_batch(X, y, th, 1.95, threads=0)
    same = r["jitter"] == fs["jitter"]
    assert same.sum() >= len(th) - 2  # float pivots near the ladder threshold may differ
    ref_err = np.abs(fs["neg2"] - fd["neg2"]) / np.abs(fd["neg2"])
    dev_vs_ref = np.abs(r["neg2"] - fs["neg2"]) / np.abs(fs["neg2"])
    assert np.all(dev_vs_ref[same] <= np.maximum(1e-5, 10 * ref_err[same]))
    dev_err = np.abs(r["neg2"] - fd["neg2"]) / np.abs(fd["neg2"])
    assert np.median(dev_err) <= 1.5 * np.median(ref_err) + 1e-7
    ev.close()


def test_single_precision_model_predict(g, ctx, ref_fast):
    """model_at_theta<float> + predict (predictor.hpp:20-50) against the reference float model."""
    X, y, th = _f32_case(7, 500, 3)
    Xt = np.random.default_rng(8).random((300, 3))
    m = g.model_at_theta(g.new_dataset(X, y), th[0], 1.95, 0.0, g.Backend(ctx), precision="single")
    rf = ref_fast.model_predict(X, y, th[0], 1.95, 0.0, Xt, threads=0, precision="single")
    rd = ref_fast.model_predict(X, y, th[0], 1.95, 0.0, Xt, threads=0)
    yhat, mse = g.predict(m, Xt, with_mse=True)
    scale = max(np.abs(rd["yhat"]).max(), np.abs(y).max())
    ref_err = np.max(np.abs(rf["yhat"] - rd["yhat"])) / scale
    assert np.max(np.abs(yhat - rd["yhat"])) / scale <= max(1e-5, 3 * ref_err)
    assert np.all(mse >= 0.0)
    m.close()


def test_single_precision_fit(g, ctx, ref_fast):
    """fit_gp_detailed<float> on the device. A small GA in float is path-dependent (fitness
    noise ~1e-3 changes selections), so trajectories are not compared; instead the reported
    float deviance at the device's theta-hat must match the reference float instantiation's
    evaluation there, within the float gate, and the fit must spend the GA budget."""
    z = np.load(os.path.join(GOLD, "c1p195.npz"))
    X, y = z["X"], z["y"]
    be = g.Backend(ctx)
    cfg = g.FitConfig(ga=g.GaConfig(population=20, generations=5), seed=3, p=1.95, precision="single")
    fr = g.fit_gp_detailed(g.new_dataset(X, y), cfg, be)
    th = np.array([fr.model.params.theta])
    fs = ref_fast.eval_batch(X, y, th, 1.95, threads=0, precision="single")
    fd = ref_fast.eval_batch(X, y, th, 1.95, threads=0)
    ref_err = abs(fs["neg2"][0] - fd["neg2"][0]) / abs(fd["neg2"][0])
    assert abs(fr.model.neg2_log_lik - fs["neg2"][0]) <= max(1e-5, 10 * ref_err) * abs(fs["neg2"][0])
    assert fr.ledger.factorizations == 100
    yhat = g.predict(fr.model, X[:20])  # the float model interpolates its design
    assert np.max(np.abs(yhat - y[:20])) <= 1e-2 * np.abs(y).max()


def test_reference_helpers_on_device(g, ctx):
    """mu_hat / sigma2_hat (likelihood.hpp:32-57) through the device solves agree with the batched
    evaluation record; the *_into forms; model_alpha_residual <= 1e-6 (the GpModel contract,
    likelihood.hpp:191-213); predict_set (predictor.hpp:71-79)."""
    z = np.load(os.path.join(GOLD, "c1p195.npz"))
    X, y = z["X"], z["y"]
    th = np.array([3.0, 2.0])
    be = g.Backend(ctx)
    data = g.new_dataset(X, y)
    R = g.build_corr_matrix(X, g.Hyperparameters(th, 1.95), ctx)
    f = g.CorrelationFactor(np.empty((0, 0)))
    be.factorize_into(R, f)
    mu = g.mu_hat(be, f, y)
    s2 = g.sigma2_hat(be, f, y, mu)
    ev = g.ProfileEvaluator(data, 1.95, 0.0, be, max_batch=1)
    rec = ev.eval_batch(th[None, :])
    assert rel(mu, rec["mu"][0]) <= 1e-9 and rel(s2, rec["sigma2"][0]) <= 1e-8
    x = np.empty(len(y))
    be.solve_lower_into(f, y, x)
    assert np.allclose(np.tril(f.lower) @ x, y, rtol=0, atol=1e-8 * np.abs(y).max())
    m = g.model_at_theta(data, th, 1.95, 0.0, be)
    assert m.jitter_used == rec["jitter"][0]
    assert g.model_alpha_residual(m) <= 1e-6
    ps = g.predict_set(m, z["Xt"][:50], truth=np.zeros(50))
    assert ps.predictions.shape == (50,) and ps.sspe == g.sspe(ps.predictions, np.zeros(50))
    ev.close()
    m.close()


def test_concurrent_contexts_in_threads(g):
    """Distinct contexts used concurrently from distinct host threads (the reference's concurrent
    replications, bench.hpp:503-516) give the same records as sequential use."""
    import threading
    z = np.load(os.path.join(GOLD, "c1p195.npz"))
    X, y, th = z["X"], z["y"], z["thetas"][:16]
    seq = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(g.Context(0)),
                             max_batch=16).eval_batch(th)
    out, errs = [None] * 4, []

    def work(i):
        try:
            ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(g.Context(0)), max_batch=16)
            for _ in range(3):
                out[i] = ev.eval_batch(th)
            ev.close()
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t_ in ts:
        t_.start()
    for t_ in ts:
        t_.join()
    assert not errs, errs
    for r in out:
        assert np.array_equal(r["neg2"], seq["neg2"]) and np.array_equal(r["jitter"], seq["jitter"])


@pytest.mark.parametrize("precision,tol", [("double", 1e-13), ("single", 1e-5)])
def test_profile_known_answer_n2(g, ctx, precision, tol):
    """X = [[0],[1]], y = [0, 1], theta = 2, p = 1.95 -> -2logL = -1.113952892208059,
    mu = 0.5, sigma2 = 0.28912941068741643, jitter 0; the model predicts 0.5 at x = 0.5."""
    data = g.new_dataset([[0.0], [1.0]], [0.0, 1.0])
    ev = g.ProfileEvaluator(data, 1.95, 0.0, g.Backend(ctx), max_batch=1, precision=precision)
    r = ev.eval(np.array([2.0]))
    assert rel(r.neg2_log_lik, -1.113952892208059) < tol
    assert rel(r.mu_hat, 0.5) < tol and rel(r.sigma2_hat, 0.28912941068741643) < tol
    assert r.jitter_used == 0.0
    m = g.model_at_theta(data, [2.0], 1.95, 0.0, g.Backend(ctx), precision=precision)
    assert abs(g.predict(m, [[0.5]])[0] - 0.5) < tol
    ev.close()
    m.close()


def test_fit_population_in_chunks(g, ctx):
    """A plan with fewer slots than the GA population evaluates each generation in chunks: the same
    candidates, the same stash (strict < in slot order) -- theta-hat, trace and model identical to
    the one-batch fit. fit_batch sizes the plan to device memory (whole population when it fits)."""
    z = np.load(os.path.join(GOLD, "c1p195.npz"))
    data = g.new_dataset(z["X"], z["y"])
    be = g.Backend(ctx)
    cfg = g.FitConfig(ga=g.GaConfig(population=20, generations=4), seed=3, p=1.95)
    assert g.fit_batch(data, cfg, be) == 20
    full = g.fit_gp_detailed(data, cfg, be)
    ev7 = g.ProfileEvaluator(data, 1.95, 0.0, be, max_batch=7)
    part = g.fit_gp_detailed(data, cfg, be, evaluator=ev7)
    assert np.array_equal(np.array(part.model.params.theta), np.array(full.model.params.theta))
    assert part.model.neg2_log_lik == full.model.neg2_log_lik
    assert [r.best_value for r in part.trace.generations] == [r.best_value for r in full.trace.generations]
    assert np.array_equal(part.model.alpha, full.model.alpha)
    ev7.close()


def test_single_precision_deep_ladder(g, ctx, ref_fast):
    """A near-rank-1 R (theta -> 0, n=3000) fails the float factorization until jitter 1e-5 in
    the reference's float instantiation (backend.hpp:105-119); the device float engine climbs
    the ladder to the same step and agrees within the float path's error."""
    rng = np.random.default_rng(31)
    X = rng.random((3000, 2))
    y = np.sin(3 * X).sum(1)
    th = np.array([[1e-6, 1e-6], [1.0, 2.0]])
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=2,
                            precision="single")
    r = ev.eval_batch(th)
    fs = ref_fast.eval_batch(X, y, th, 1.95, threads=0, precision="single")
    assert np.array_equal(r["jitter"], fs["jitter"]) and r["jitter"][0] == 1e-5
    assert np.all(np.abs(r["neg2"] - fs["neg2"]) <= 1e-3 * np.abs(fs["neg2"]))
    ev.close()


def test_device_memory_pool(g):
    """Plans allocate from the library's per-device pool: a destroyed plan's pages stay mapped
    (reported free by gpemu_ctx_mem_info, reused by the next plan with identical results) and go
    back to the driver when the context is destroyed."""
    import ctypes as C
    import torch
    torch.cuda.init()
    mib = 1 << 20
    n, d, B = 4096, 4, 8
    plan_bytes = g.lib().gpemu_plan_bytes(n, d, B, 0)
    assert plan_bytes > 512 * mib
    rng = np.random.default_rng(5)
    X = rng.random((n, d))
    y = np.sin(3 * X).sum(1)
    th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
    driver0 = torch.cuda.mem_get_info()[0]
    ctx = g.Context(0)

    def engine_free():
        f, t = C.c_size_t(), C.c_size_t()
        g._check(g.lib().gpemu_ctx_mem_info(ctx.handle, C.byref(f), C.byref(t)))
        return f.value

    f0 = engine_free()
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=B)
    r1 = ev.eval_batch(th)
    assert f0 - engine_free() >= 0.9 * plan_bytes
    ev.close()
    assert abs(engine_free() - f0) < 64 * mib  # idle pool pages count as free
    assert torch.cuda.mem_get_info()[0] < driver0 - plan_bytes // 2  # ...and stay mapped
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=B)
    r2 = ev.eval_batch(th)
    for k in ("neg2", "mu", "sigma2", "jitter", "log_det"):
        assert np.array_equal(r1[k], r2[k]), k
    ev.close()
    ctx.close()
    assert torch.cuda.mem_get_info()[0] > driver0 - 64 * mib  # trimmed on context destroy


@pytest.mark.parametrize("n", [127, 128, 129, 255, 256, 257])
def test_eval_tile_boundaries_vs_reference(g, ctx, ref_fast, n):
    """Sizes on either side of the 128-row tile (identity padding of the last tile, one vs two
    tile columns): the same jitter step as the reference's evaluator and deviance / mu / sigma2
    within rounding of it."""
    rng = np.random.default_rng(1000 + n)
    d = 3
    X = rng.random((n, d))
    y = np.sin(3 * X).sum(1) + 0.1 * rng.standard_normal(n)
    th = 10 ** rng.uniform(-0.5, 1.0, size=(12, d))
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=12)
    r = ev.eval_batch(th)
    f = ref_fast.eval_batch(X, y, th, 1.95, threads=0)
    assert np.array_equal(r["jitter"], f["jitter"])
    assert np.all(np.abs(r["neg2"] - f["neg2"]) <= 1e-9 * np.abs(f["neg2"]) + 1e-9)
    assert rel(r["mu"], f["mu"]) < 1e-8 and rel(r["sigma2"], f["sigma2"]) < 1e-8
    ev.close()


@pytest.mark.parametrize("budget", [7, 13, 20])
def test_refine_speculative_equals_sequential(g, ctx, budget):
    """gpemu_refine_fit_ex on an 8-slot plan (each coordinate's golden-section decision tree in
    one batch, replayed) and on a 1-slot plan (one evaluation at a time): bitwise the same
    polished theta, -2logL, evaluation count and rebuilt model, for budgets that stop
    mid-coordinate too."""
    import ctypes as C
    z = np.load(os.path.join(GOLD, "refine.npz"))
    X, y, p = z["X_0"], z["y_0"], float(z["p_0"])
    n, d = X.shape
    theta_fit = z["theta_fit_0"]
    data = g.new_dataset(X, y)
    be = g.Backend(ctx)
    neg2_fit = float(g.ProfileEvaluator(data, p, 0.0, be, max_batch=1).eval_batch(theta_fit[None, :])["neg2"][0])
    lo, hi = np.full(d, 1e-6), np.full(d, 12.0)
    outs = []
    for mb in (1, 8):
        ev = g.ProfileEvaluator(data, p, 0.0, be, max_batch=mb)
        th, sc, al = np.empty(d), np.empty(4), np.empty(n)
        nv, used, mh = C.c_double(), C.c_int(), C.c_void_p()
        g._check(g.lib().gpemu_refine_fit_ex(ev.handle, ev.handle, g._p(lo), g._p(hi), g._p(theta_fit),
                                            neg2_fit, budget, g._p(th), C.byref(nv), C.byref(used),
                                            C.byref(mh), g._p(sc), g._p(al)))
        outs.append((th.copy(), nv.value, used.value, bool(mh.value), sc.copy() if mh.value else None,
                     al.copy() if mh.value else None))
        if mh.value:
            g.lib().gpemu_model_destroy(mh)
        ev.close()
    (t1, v1, u1, m1, s1, a1), (t8, v8, u8, m8, s8, a8) = outs
    assert np.array_equal(t1, t8) and v1 == v8 and u1 == u8 == budget and m1 == m8
    if m1:
        assert np.array_equal(s1, s8) and np.array_equal(a1, a8)


def test_batch_invariance_across_kernel_instantiations(g, ctx):
    """n=1000 (36 tasks per candidate): a 100-candidate batch runs chol_dag_kernel<false> (take-
    ahead, >= 16 tickets per CTA), 8 candidates and single evaluations run chol_dag_kernel<true>
    (slab release of the sub-diagonal tile, interleaved border chain). Both must give bitwise
    the same record for the same theta."""
    rng = np.random.default_rng(77)
    n, d = 1000, 3
    X = rng.random((n, d))
    y = np.sin(3 * X).sum(1)
    th = 10 ** rng.uniform(-1.0, 0.8, size=(100, d))
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=100)
    big = ev.eval_batch(th)
    small = ev.eval_batch(th[40:48])
    one = ev.eval_batch(th[93:94])
    for k in ("neg2", "mu", "sigma2", "jitter", "log_det"):
        assert np.array_equal(big[k][40:48], small[k]), k
        assert np.array_equal(big[k][93:94], one[k]), k
    ev.close()


def test_speculative_ladder_rung_bitwise(g, ctx, monkeypatch):
    """C1 (every candidate climbs to 1e-8): once a batch showed that most candidates climb,
    the next batches evaluate jitter 0 and 1e-8 in ONE pass (speculation slots). Records,
    jitter steps, last_factor and the fit are bitwise those of the two-pass ladder."""
    z = np.load(os.path.join(GOLD, "c1.npz"))
    data = g.new_dataset(z["X"], z["y"])
    be = g.Backend(ctx)
    ev = g.ProfileEvaluator(data, 2.0, 0.0, be, max_batch=100)
    first = ev.eval_batch(z["thetas"])  # two passes; arms the speculation
    assert np.count_nonzero(first["jitter"] > 0) > 50
    n0 = ctx.launch_count
    second = ev.eval_batch(z["thetas"])
    one_pass = ctx.launch_count - n0
    L_spec = ev.last_factor(3).lower
    monkeypatch.setenv("GPEMU_SPEC_LADDER", "0")
    n0 = ctx.launch_count
    third = ev.eval_batch(z["thetas"])
    two_pass = ctx.launch_count - n0
    L_plain = ev.last_factor(3).lower
    assert one_pass < two_pass, (one_pass, two_pass)
    for k in ("neg2", "mu", "sigma2", "jitter", "log_det", "status"):
        assert np.array_equal(first[k], second[k]) and np.array_equal(second[k], third[k]), k
    assert np.array_equal(L_spec, L_plain)
    monkeypatch.delenv("GPEMU_SPEC_LADDER")
    ev.close()


def test_ladder_invariance_across_kernel_instantiations(g, ctx):
    """Candidates that fail a pivot partway through the factorization (squared exponential at
    n=1000: most thetas climb the jitter ladder) in chain-bound launches -- slab-wise
    release of L(j,j) and of the border rows, the TRSM's per-slab loads and its drop path for
    a candidate that failed meanwhile -- against the same thetas inside a 100-candidate
    throughput launch: bitwise the same records, jitter steps included."""
    rng = np.random.default_rng(2024)
    n, d = 1000, 3
    X = rng.random((n, d))
    y = np.sin(3 * X).sum(1)
    th = 10 ** rng.uniform(-4.0, 1.5, size=(100, d))  # p = 2: most climb to 1e-8, a few do not
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 2.0, 0.0, g.Backend(ctx), max_batch=100)
    big = ev.eval_batch(th)
    assert np.any(big["jitter"] > 0) and np.any(big["jitter"] == 0), "the batch should mix ladder steps"
    for lo in (0, 8, 56, 92):
        small = ev.eval_batch(th[lo:lo + 8])
        for k in ("neg2", "mu", "sigma2", "jitter", "log_det"):
            assert np.array_equal(big[k][lo:lo + 8], small[k]), (k, lo)
    for i in np.nonzero(big["jitter"] > 0)[0][:3]:
        one = ev.eval_batch(th[i:i + 1])
        assert one["jitter"][0] == big["jitter"][i] and one["neg2"][0] == big["neg2"][i]
    ev.close()


@pytest.mark.parametrize("seed", [5, 6])
def test_launch_shape_invariance_random_designs(g, ctx, seed):
    """A short run of tools/stress_dag.py's check: random designs (partial last tiles, d 1-6,
    p in {1, 1.5, 1.95, 2}, thetas from 1e-5 to 31: many candidates fail pivots at various
    columns) evaluated in a 100-candidate launch (throughput kernel), again, in an 8-candidate
    launch and alone (chain-bound kernel: slab-wise release of every OFF tile, last K-tiles
    consumed slab by slab, deferred slab issue, per-warp slab releases). Every record must
    agree bitwise across the four launches."""
    rng = np.random.default_rng(seed)
    be = g.Backend(ctx)
    for _ in range(12):
        n = int(rng.choice([257, 600, 1500, 2100]))
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
        for k in ("neg2", "mu", "sigma2", "jitter", "log_det"):
            assert np.array_equal(a[k], b[k], equal_nan=True), (n, d, p, k)
            assert np.array_equal(a[k][lo:lo + 8], c[k], equal_nan=True), (n, d, p, lo, k)
            assert np.array_equal(a[k][i:i + 1], e[k], equal_nan=True), (n, d, p, i, k)
        ev.close()
