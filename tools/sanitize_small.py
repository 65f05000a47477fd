"""Small end-to-end run of every device path (for compute-sanitizer)."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g
rng = np.random.default_rng(1)
for engine in ("dag", "simple"):
    ctx = g.Context(0, engine)
    be = g.Backend(ctx)
    X = rng.random((300, 3)); y = np.sin(3 * X).sum(1)
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, be, max_batch=4)
    r = ev.eval_batch(10 ** rng.uniform(-1, 1, (4, 3)))
    m = g.model_at_theta(g.new_dataset(X, y), np.array([2.0, 3.0, 1.0]), 1.95, 0.0, be)
    yh, mse = g.predict(m, rng.random((150, 3)), with_mse=True)
    R = g.build_corr_matrix(X[:50], g.Hyperparameters([1.0, 2.0, 3.0]), ctx)
    f = be.factorize(R)
    be.solve_full(f, np.ones(50))
    fr = g.fit_gp_detailed(g.new_dataset(X, y), g.FitConfig(ga=g.GaConfig(4, 2), seed=1), be)
    print(engine, "ok", r["neg2"][:2], yh[:2], mse[:2])
