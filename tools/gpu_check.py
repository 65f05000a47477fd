"""First-light GPU check: every device path against the oracle, printing max diffs."""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo" if len(sys.argv) < 2 else sys.argv[1])
from oracle.oracle import Oracle
import paper_1203_1269_b200.gpemu as g

o = Oracle()
rng = np.random.default_rng(0)

def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    den = np.maximum(np.abs(a), np.abs(b)); den[den == 0] = 1
    return float(np.max(np.abs(a - b) / den)) if a.size else 0.0

ctx = g.Context(0, "dag")
X = rng.random((50, 3)); th = np.array([2.0, 0.5, 3.0])
R = g.build_corr_matrix(X, g.Hyperparameters(th, 1.95, 0.01), ctx).values
print("build_corr rel", rel(R, o.build_corr(X, th, 1.95, 0.01)), flush=True)
r = g.corr_vector(X[3], X, g.Hyperparameters(th, 1.95), ctx)
print("corr_vector rel", rel(r, o.corr_vector(X[3], X, th, 1.95)), flush=True)

for engine in ("simple", "dag"):
    ctx.set_engine(engine)
    be = g.Backend(ctx)
    for n in (7, 64, 130, 300):
        Xn = rng.random((n, 2)) ; thn = np.array([30.0, 30.0])
        Rn = o.build_corr(Xn, thn, 1.95)
        t = time.time()
        f = be.factorize(g.CorrelationMatrix(Rn))
        dt = time.time() - t
        ref = o.factorize(Rn, kind=0)
        Lr, ldr, jr = ref
        print(f"{engine} factorize n={n}: L rel {rel(np.tril(f.lower), np.tril(Lr)):.3e} logdet {f.log_det:.15g} vs {ldr:.15g} jit {f.jitter_used} vs {jr} bitwise={np.array_equal(np.tril(f.lower), np.tril(Lr))} {dt*1e3:.1f}ms", flush=True)
    # NPD
    try:
        be.factorize(g.CorrelationMatrix(np.array([[1.0, 2.0], [2.0, 1.0]])))
        print(engine, "NPD: no exception!!")
    except g.NotPositiveDefiniteError as e:
        print(engine, "NPD ok:", e)

# eval batch C1-like
for engine in ("simple", "dag"):
    ctx.set_engine(engine)
    be = g.Backend(ctx)
    for (n, d, p, fn) in ((200, 2, 2.0, "gp"), (200, 2, 1.95, "gp"), (300, 3, 1.95, "smooth"), (520, 6, 1.95, "h6")):
        Xd = o.maximin_lhd(n, d, 7, 2000)
        if fn == "gp": y = o.goldstein_price_log(Xd)
        elif fn == "h6": y = o.hartman6(Xd)
        else: y = np.sin(3 * Xd).sum(1) + 0.5 * (Xd**2).sum(1)
        lo = np.full(d, np.log10(1e-6)); hi = np.full(d, np.log10(12.0))
        thetas = 10 ** o.lhs_population(lo, hi, 64, 99)
        data = g.new_dataset(Xd, y)
        ev = g.ProfileEvaluator(data, p, 0.0, be, max_batch=64)
        t = time.time(); res = ev.eval_batch(thetas); dt = time.time() - t
        ref = o.eval_batch(Xd, y, thetas, p)
        fin = np.isfinite(ref["neg2"])
        rr = np.abs(res["neg2"] - ref["neg2"]) / np.abs(ref["neg2"])
        print(f"{engine} eval n={n} d={d} p={p}: neg2 rel max {np.nanmax(rr[fin]):.3e} median {np.median(rr[fin]):.3e} "
              f"jit eq {np.array_equal(res['jitter'], ref['jitter'])} inf eq {np.array_equal(np.isinf(res['neg2']), np.isinf(ref['neg2']))} "
              f"jit set {sorted(set(ref['jitter']))} {dt*1e3:.1f} ms", flush=True)
        # batch invariance
        r2 = ev.eval_batch(thetas[5:9])
        print("   batch-invariant:", np.array_equal(r2["neg2"], res["neg2"][5:9]), flush=True)
        ev.close()

ctx.set_engine("dag")
be = g.Backend(ctx)
Xd = o.maximin_lhd(200, 2, 7, 2000); y = o.goldstein_price_log(Xd)
data = g.new_dataset(Xd, y)
cfg = g.FitConfig(ga=g.GaConfig(population=20, generations=5), seed=3, p=2.0)
t = time.time(); fr = g.fit_gp_detailed(data, cfg, be); dt = time.time() - t
of = o.fit(Xd, y, p=2.0, population=20, generations=5, seed=3)
print("fit theta eq", np.array_equal(fr.model.params.theta, of["theta"]), fr.model.params.theta, of["theta"],
      "neg2", fr.model.neg2_log_lik, of["neg2"], "alpha rel", rel(fr.model.alpha, of["alpha"]), f"{dt:.2f}s", flush=True)
Xt = o.maximin_lhd(100, 2, 11, 0)
yh, mse = g.predict(fr.model, Xt, with_mse=True)
yo = o.predict(Xd, of["theta"], 2.0, of["mu"], of["alpha"], Xt)
fo = o.fit(Xd, y, p=2.0, population=20, generations=5, seed=3, want_L=True)
mo = o.kriging_mse(Xd, of["theta"], 2.0, of["sigma2"], fo["L"], Xt)
sc = max(np.abs(yo).max(), np.abs(y).max())
print("predict max abs/scale", np.abs(yh - yo).max() / sc, "mse rel", rel(mse, mo), mse[:3], mo[:3], flush=True)
print("launches", ctx.launch_count)
