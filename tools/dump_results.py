"""Dump DAG / simple engine eval results on the golden sets (for offline accuracy analysis)."""
import os, sys
import numpy as np
sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g
out = {}
for engine in ("dag", "simple"):
    ctx = g.Context(0, engine)
    for name in ("c1", "c1p195", "c2"):
        z = np.load(f"tests/golden/{name}.npz")
        ev = g.ProfileEvaluator(g.new_dataset(z["X"], z["y"]), float(z["p"]), 0.0, g.Backend(ctx), max_batch=100)
        r = ev.eval_batch(z["thetas"])
        for k, v in r.items():
            out[f"{engine}_{name}_{k}"] = v
        ev.close()
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/dump.npz", **out)
print("ok")
