"""CPU: multi-rank host logic (gloo, world_size 2 and 3) for the sharded fit.

The per-rank evaluator is the oracle here (no GPU on this box); on the B200 it is
ProfileEvaluator.eval_batch on each rank's GPU. What is tested is everything that is not
the kernel: the GA state machine (C-ABI gpemu_ga_*), the contiguous sharding, the
per-generation all-gather in slot order, the stash rule and theta-hat bitwise equality with
the sequential reference fit."""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def small_problem(orc, n=60):
    X = orc.maximin_lhd(n, 2, 3, 500)
    y = orc.goldstein_price_log(X)
    return X, y


def test_shard_range():
    from paper_1203_1269_b200.sharded import shard_range
    for P in (1, 7, 20, 100):
        for G in (1, 2, 3, 8):
            got = [shard_range(P, G, r) for r in range(G)]
            covered = [i for lo, hi in got for i in range(lo, hi)]
            assert covered == list(range(P))
            assert all(lo <= hi for lo, hi in got)


def test_ga_state_machine_matches_reference_fit(orc):
    """gpemu_ga_* driven sequentially with the oracle objective == the reference fit (C1)."""
    import paper_1203_1269_b200.gpemu as g
    z = np.load(os.path.join(GOLD, "c1.npz"))
    X, y = z["X"], z["y"]
    cfg = g.FitConfig(ga=g.GaConfig(population=100, generations=20), seed=0, p=2.0)
    ga = g.GeneticOptimizer(2, cfg.bounds_for(2), cfg.ga, cfg.seed)
    best, stash = np.inf, None
    while not ga.status()["done"]:
        th = ga.thetas()
        f = orc.eval_batch(X, y, th, 2.0)["neg2"]
        for i in range(len(f)):
            if f[i] < best:
                best, stash = f[i], th[i].copy()
        ga.tell(f)
    st = ga.status()
    assert np.array_equal(stash, z["fit_theta"])
    assert np.array_equal(st["trace_genes"], z["trace_genes"])
    assert np.array_equal(st["trace_best"], z["trace_best"])
    assert st["best_value"] == z["fit_neg2"]


def _worker(rank, world, port, out_dir, n):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from oracle.oracle import Oracle
    import paper_1203_1269_b200.gpemu as g
    from paper_1203_1269_b200.sharded import sharded_fit, sharded_predict
    orc = Oracle()
    X, y = small_problem(orc, n)
    data = g.new_dataset(X, y)
    cfg = g.FitConfig(ga=g.GaConfig(population=20, generations=4), seed=11, p=1.95)
    calls = []

    def evaluate(th):
        calls.append(len(th))
        return orc.eval_batch(X, y, th, 1.95)

    res = sharded_fit(data, cfg, evaluate)
    Xt = orc.maximin_lhd(23, 2, 5, 0)
    L, ld, jt = orc.factorize(orc.build_corr(X, res["theta"], 1.95))
    alpha = orc.solve_upper(L, orc.solve_lower(L, y - res["mu"]))
    yhat = sharded_predict(None, Xt, predict_fn=lambda Xs: orc.predict(X, res["theta"], 1.95,
                                                                     res["mu"], alpha, Xs))
    yhat2, mse = sharded_predict(None, Xt, with_mse=True, predict_fn=lambda Xs: (
        orc.predict(X, res["theta"], 1.95, res["mu"], alpha, Xs),
        orc.kriging_mse(X, res["theta"], 1.95, res["sigma2"], L, Xs)))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), theta=res["theta"], neg2=res["neg2"],
             trace=res["trace_genes"], calls=np.array(calls), yhat=yhat, yhat2=yhat2, mse=mse)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_fit_gloo(orc, tmp_path, world):
    import torch.multiprocessing as mp
    n = 60
    mp.spawn(_worker, args=(world, free_port(), str(tmp_path), n), nprocs=world, join=True)
    X, y = small_problem(orc, n)
    ref = orc.fit(X, y, p=1.95, population=20, generations=4, seed=11)
    outs = [np.load(tmp_path / f"rank{r}.npz") for r in range(world)]
    for o in outs:
        assert np.array_equal(o["theta"], ref["theta"])       # theta-hat bitwise
        assert o["neg2"] == ref["neg2"]
        assert np.array_equal(o["trace"], ref["trace_genes"])
        assert np.array_equal(o["yhat"], outs[0]["yhat"])    # gathered in order, same everywhere
    # every rank evaluated only its contiguous share of each generation
    per = -(-20 // world)
    assert sum(int(o["calls"].sum()) for o in outs) == 20 * 4
    assert all(int(o["calls"].max()) <= per for o in outs)
    Xt = orc.maximin_lhd(23, 2, 5, 0)
    L, ld, jt = orc.factorize(orc.build_corr(X, ref["theta"], 1.95))
    alpha = orc.solve_upper(L, orc.solve_lower(L, y - ref["mu"]))
    assert np.array_equal(outs[0]["yhat"], orc.predict(X, ref["theta"], 1.95, ref["mu"], alpha, Xt))
    for o in outs:  # (yhat, mse) pairs gathered in order
        assert np.array_equal(o["yhat2"], outs[0]["yhat"])
        assert np.array_equal(o["mse"], orc.kriging_mse(X, ref["theta"], 1.95, ref["sigma2"], L, Xt))


def _ms_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from oracle.oracle import Oracle
    from paper_1203_1269_b200.sharded import sharded_argmin, sharded_multistart
    orc = Oracle()
    X, y = small_problem(orc, 50)
    th = 10.0 ** orc.lhs_population(np.full(2, -6.0), np.full(2, np.log10(12.0)), 37, 9)
    th[30] = th[4]  # a duplicate: the earliest slot must win
    res = sharded_multistart(th, lambda t: orc.eval_batch(X, y, t, 1.95))
    # ties across ranks: every rank holds the same minimum at different slots
    v, s = sharded_argmin(np.array([3.0, 1.0, 1.0]), 100 * (rank + 1))
    np.savez(os.path.join(out_dir, f"ms{rank}.npz"), neg2=res["neg2"], slot=res["slot"],
             theta=res["theta"], tie=np.array([v, s]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_multistart_min_reduce(orc, tmp_path, world):
    import torch.multiprocessing as mp
    mp.spawn(_ms_worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    X, y = small_problem(orc, 50)
    th = 10.0 ** orc.lhs_population(np.full(2, -6.0), np.full(2, np.log10(12.0)), 37, 9)
    th[30] = th[4]
    neg2 = orc.eval_batch(X, y, th, 1.95)["neg2"]
    want = int(np.argmin(neg2))  # numpy argmin = first occurrence, the reference's tie rule
    for r in range(world):
        o = np.load(tmp_path / f"ms{r}.npz")
        assert int(o["slot"]) == want and o["neg2"] == neg2[want]
        assert np.array_equal(o["theta"], th[want])
        assert o["tie"][0] == 1.0 and int(o["tie"][1]) == 101  # lowest rank's lowest slot
