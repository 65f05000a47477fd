"""Multi-GPU fit: each GA generation sharded across ranks (one process per GPU).

The unit is an independent theta candidate: a generation of P candidates is
split into contiguous ranges of ceil(P/G) per rank, every rank evaluates its range on its
own GPU, and ONE all-gather per generation of the per-candidate records (neg2, mu, sigma2,
jitter: 32 B each) gives every rank the full fitness vector. The GA state machine
(gpemu_ga_*) is identical and deterministic on every rank, so all ranks breed the same next
generation without further communication; the candidate sequence, the stash and theta-hat
are those of the sequential reference (optimizer.hpp:93-187, likelihood.hpp:257-273).
After the GA, every rank rebuilds the model at theta-hat locally (one evaluation; results
are batch-invariant, so bitwise identical on all ranks) and predictions are sharded by
test point.
"""
from __future__ import annotations

import math
from typing import Callable, Dict

import numpy as np

from . import gpemu as g

RECORD_FIELDS = ("neg2", "mu", "sigma2", "jitter")


def shard_range(P: int, world: int, rank: int):
    """Contiguous slots [lo, hi) of rank `rank` (ceil(P/world) per rank, last ones short)."""
    per = math.ceil(P / world)
    lo = min(P, rank * per)
    return lo, min(P, lo + per)


def _all_gather_records(local: np.ndarray, P: int, world: int, device):
    """local: (n_local, 4) float64 -> (P, 4) in slot order, via one all_gather."""
    import torch
    import torch.distributed as dist
    per = math.ceil(P / world)
    buf = torch.full((per, len(RECORD_FIELDS)), float("nan"), dtype=torch.float64, device=device)
    if local.shape[0]:
        buf[: local.shape[0]] = torch.from_numpy(local).to(device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    full = torch.cat(parts, 0)[:P].cpu().numpy()
    return full


def sharded_fit(data: g.Dataset, cfg: g.FitConfig,
                evaluate: Callable[[np.ndarray], Dict[str, np.ndarray]], device="cpu") -> dict:
    """GA fit with each generation sharded over the torch.distributed world.

    evaluate(thetas_slice) -> {"neg2","mu","sigma2","jitter"} arrays for this rank's slots
    (a ProfileEvaluator.eval_batch on this rank's GPU in production; any deterministic
    evaluator in tests). Returns theta_hat, the stash record and the GaTrace (identical on
    every rank)."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    d = data.d()
    ga = g.GeneticOptimizer(d, cfg.bounds_for(d), cfg.ga, cfg.seed)
    P = cfg.ga.population
    lo, hi = shard_range(P, world, rank)
    stash = None
    stash_value = math.inf
    while not ga.status()["done"]:
        th = ga.thetas()
        rec = evaluate(th[lo:hi]) if hi > lo else {k: np.empty(0) for k in RECORD_FIELDS}
        local = np.stack([np.asarray(rec[k], dtype=np.float64) for k in RECORD_FIELDS], 1) \
            if hi > lo else np.empty((0, len(RECORD_FIELDS)))
        full = _all_gather_records(local, P, world, device)
        fitness = full[:, 0]
        for i in range(P):  # stash: strict <, earliest (generation, slot)
            if fitness[i] < stash_value:
                stash_value = fitness[i]
                stash = dict(theta=th[i].copy(), neg2=full[i, 0], mu=full[i, 1],
                             sigma2=full[i, 2], jitter=full[i, 3])
        ga.tell(fitness)
    st = ga.status()
    if not math.isfinite(stash_value):
        raise g.FitError("fit_gp: every candidate failed factorization")
    if st["best_value"] != stash_value:
        raise g.Error("fit_gp: optimizer incumbent diverged from evaluation stash")
    return dict(theta=stash["theta"], neg2=stash["neg2"], mu=stash["mu"], sigma2=stash["sigma2"],
                jitter=stash["jitter"], trace_best=st["trace_best"], trace_genes=st["trace_genes"],
                stash_generation=st["stash_generation"], stash_slot=st["stash_slot"])


def sharded_predict(model: g.GpModel, Xtest: np.ndarray, device="cpu",
                    predict_fn=None, with_mse: bool = False):
    """Predictions sharded by test point across ranks (each GPU predicts N/G
    points), gathered in order on every rank. with_mse: (yhat, mse), gathered in the same
    all-gather as (yhat, mse) pairs."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    N = Xtest.shape[0]
    lo, hi = shard_range(N, world, rank)
    cols = 2 if with_mse else 1
    if predict_fn is None:
        predict_fn = (lambda X: g.predict(model, X, with_mse=True)) if with_mse else (lambda X: g.predict(model, X))
    local = predict_fn(Xtest[lo:hi]) if hi > lo else None
    per = math.ceil(N / world)
    buf = torch.full((per, cols), float("nan"), dtype=torch.float64, device=device)
    if hi > lo:
        arr = np.stack([np.asarray(v, dtype=np.float64) for v in local], 1) if with_mse else \
            np.asarray(local, dtype=np.float64)[:, None]
        buf[: hi - lo] = torch.from_numpy(arr).to(device)
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    out = torch.cat(parts, 0)[:N].cpu().numpy()
    return (out[:, 0].copy(), out[:, 1].copy()) if with_mse else out[:, 0].copy()


def sharded_argmin(values_local: np.ndarray, slot_offset: int, device="cpu"):
    """The final min-reduce of a sharded multistart: global (min value, lowest global slot)
    with the reference's tie rule (strict <, earliest slot wins; likelihood.hpp:267,
    optimizer.hpp:125-131). Two scalar all-reduces: MIN over values, then MIN over the
    slots that attain it (NCCL's MIN cannot carry the slot alongside the value)."""
    import torch
    import torch.distributed as dist
    vals = np.asarray(values_local, dtype=np.float64)
    local_min = vals.min() if vals.size else math.inf
    t = torch.tensor([local_min], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    gmin = float(t.item())
    big = np.iinfo(np.int64).max
    hits = np.nonzero(vals == gmin)[0] if vals.size else np.empty(0, dtype=np.int64)
    s = torch.tensor([slot_offset + int(hits[0]) if hits.size else big], dtype=torch.int64,
                     device=device)
    dist.all_reduce(s, op=dist.ReduceOp.MIN)
    return gmin, int(s.item())


def sharded_multistart(thetas: np.ndarray,
                       evaluate: Callable[[np.ndarray], Dict[str, np.ndarray]],
                       device="cpu") -> dict:
    """Evaluate a fixed set of candidates (a multistart) split across ranks and return the
    global argmin, identical on every rank; no data-path collective besides the final
    min-reduce."""
    import torch.distributed as dist
    world, rank = dist.get_world_size(), dist.get_rank()
    P = thetas.shape[0]
    lo, hi = shard_range(P, world, rank)
    rec = evaluate(thetas[lo:hi]) if hi > lo else {"neg2": np.empty(0)}
    vmin, slot = sharded_argmin(np.asarray(rec["neg2"]), lo, device)
    return dict(neg2=vmin, slot=slot, theta=thetas[slot].copy())
