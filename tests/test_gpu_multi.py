"""Candidate sharding through the C-ABI (gpemu_fit_multi / gpemu_eval_batch_multi): G plans of
the same data, one host thread each, contiguous ceil(P/G) candidate ranges (optimizer.hpp:86-92,
:116-121; likelihood.hpp:257-273). On this one-GPU pool the G plans live in G contexts of
device 0 (independent persistent launches on separate streams: no plan waits on another), so
the host logic -- split, slot-order gather, cross-shard stash, model on the owning plan -- is
what is tested; theta-hat and the trace must be bitwise the single-plan fit's and the
reference's."""
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


def _evs(g, data, p, G, max_batch):
    out = []
    for _ in range(G):
        be = g.Backend(g.Context(0))
        out.append(g.ProfileEvaluator(data, p, 0.0, be, max_batch=max_batch))
    return out


@pytest.mark.parametrize("G,max_batch", [(2, 50), (3, 34), (3, 9)])
def test_fit_multi_bitwise(g, G, max_batch):
    """C1 full GA (100 x 20) sharded over G plans (max_batch 9: each shard in chunks): theta-hat
    and every generation's best genes equal the reference's (c1.npz), the model is the
    single-plan model, and eval_batch_multi records equal one plan's bitwise."""
    z = np.load(os.path.join(GOLD, "c1.npz"))
    data = g.new_dataset(z["X"], z["y"])
    cfg = g.FitConfig(ga=g.GaConfig(population=100, generations=20), seed=0, p=2.0)
    evs = _evs(g, data, 2.0, G, max_batch)
    fr = g.fit_gp_detailed(data, cfg, evs[0].backend, evaluator=evs)
    assert np.array_equal(np.array(fr.model.params.theta), z["fit_theta"])
    assert np.array_equal(np.array([r.best_point for r in fr.trace.generations]), z["trace_genes"])
    assert fr.jitter_max == z["fit_jitter_max"]
    one = g.fit_gp_detailed(data, cfg, g.Backend(g.Context(0)))
    assert fr.model.neg2_log_lik == one.model.neg2_log_lik
    assert np.array_equal(fr.model.alpha, one.model.alpha)
    Xt = z["Xt"][:100]
    assert np.array_equal(g.predict(fr.model, Xt), g.predict(one.model, Xt))
    multi = g.eval_batch_multi(evs, z["thetas"])
    ref = g.ProfileEvaluator(data, 2.0, 0.0, g.Backend(g.Context(0)), max_batch=100).eval_batch(z["thetas"])
    for k in ("neg2", "mu", "sigma2", "jitter", "log_det", "status"):
        assert np.array_equal(multi[k], ref[k]), k


def test_multi_rejects_mismatched_plans(g):
    z = np.load(os.path.join(GOLD, "c1.npz"))
    be = g.Backend(g.Context(0))
    a = g.ProfileEvaluator(g.new_dataset(z["X"], z["y"]), 2.0, 0.0, be, max_batch=8)
    b = g.ProfileEvaluator(g.new_dataset(z["X"], z["y"] + 1.0), 2.0, 0.0, be, max_batch=8)
    c = g.ProfileEvaluator(g.new_dataset(z["X"], z["y"]), 1.95, 0.0, be, max_batch=8)
    for other in (b, c):
        with pytest.raises(g.ValidationError):
            g.eval_batch_multi([a, other], z["thetas"][:8])
