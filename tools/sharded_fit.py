"""Sharded GA fit on the GPUs of one node (torchrun, one rank per GPU, NCCL).

  torchrun --nproc-per-node G --master-addr 127.0.0.1 tools/sharded_fit.py [n d P gens]

Each rank evaluates ceil(P/G) candidates of every generation on its GPU; one NCCL
all-gather of the 32-byte records per generation; identical GA state on every rank. Then every
rank rebuilds the model at theta-hat (bitwise the same everywhere: one B=1 evaluation), predicts
its N/G share of the test points with the kriging MSE, and the (yhat, mse) shards are
all-gathered; rank 0 checks them bitwise against its own unsharded prediction.
"""
import os, sys, time
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_1269_b200.gpemu as g
from paper_1203_1269_b200.sharded import sharded_fit, sharded_predict, shard_range

n, d, P, G = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (4096, 10, 100, 20)))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank, world = dist.get_rank(), dist.get_world_size()
rng = np.random.default_rng(7)
X = np.empty((n, d))
for k in range(d):
    X[:, k] = (rng.permutation(n) + rng.random(n)) / n
y = (np.sin(3 * X + 0.37 * np.arange(d)) + 0.5 * X * X).sum(1)
data = g.new_dataset(X, y)
ctx = g.Context(local)
lo, hi = shard_range(P, world, rank)
ev = g.ProfileEvaluator(data, 1.95, 0.0, g.Backend(ctx), max_batch=max(1, hi - lo))
cfg = g.FitConfig(ga=g.GaConfig(population=P, generations=G), seed=1, p=1.95)
torch.cuda.synchronize(); dist.barrier(); t = time.time()
res = sharded_fit(data, cfg, ev.eval_batch, device=torch.device("cuda", local))
torch.cuda.synchronize(); dist.barrier(); dt = time.time() - t
if rank == 0:
    print(f"sharded fit n={n} d={d} GA {P}x{G} on {world} GPU(s): {dt:.2f} s, "
          f"theta_hat={np.array2string(res['theta'], precision=4)}, neg2={res['neg2']:.6f}, "
          f"stash=(gen {res['stash_generation']}, slot {res['stash_slot']})", flush=True)
model = g.model_at_theta(data, res["theta"], 1.95, 0.0, g.Backend(ctx))
Xt = np.random.default_rng(8).random((4099, d))
torch.cuda.synchronize(); dist.barrier(); t = time.time()
yhat, mse = sharded_predict(model, Xt, device=torch.device("cuda", local), with_mse=True)
torch.cuda.synchronize(); dist.barrier(); dt = time.time() - t
if rank == 0:
    y0, m0 = g.predict(model, Xt, with_mse=True)
    same = np.array_equal(yhat, y0) and np.array_equal(mse, m0)
    print(f"sharded predict+MSE of {len(Xt)} points on {world} GPU(s): {dt * 1e3:.1f} ms, "
          f"bitwise equal to the unsharded prediction: {same}", flush=True)
    if not same:
        raise SystemExit("sharded prediction differs from the unsharded one")
dist.destroy_process_group()
