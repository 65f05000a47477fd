"""Sharded GA fit on the GPUs of one node (torchrun, one rank per GPU, NCCL).

  torchrun --nproc-per-node G --master-addr 127.0.0.1 tools/sharded_fit.py [n d P gens]

Each rank evaluates ceil(P/G) candidates of every generation on its GPU; one NCCL
all-gather of the 32-byte records per generation; identical GA state on every rank.
"""
import os, sys, time
import numpy as np
import torch
import torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1203_1269_b200.gpemu as g
from paper_1203_1269_b200.sharded import sharded_fit, shard_range

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
dist.destroy_process_group()
