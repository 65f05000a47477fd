"""Quick device-time probe of one eval batch at a given (n, d, B)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_1203_1269_b200.gpemu as g

n, d, B = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 10, 100)))
p_exp = float(sys.argv[4]) if len(sys.argv) > 4 else 1.95
nug = float(sys.argv[5]) if len(sys.argv) > 5 else 0.0
rng = np.random.default_rng(0)
X = rng.random((n, d))
y = np.sin(3 * X).sum(1)
import os
ctx = g.Context(0, os.environ.get("GPEMU_PROBE_ENGINE", "dag"))
ev = g.ProfileEvaluator(g.new_dataset(X, y), p_exp, nug, g.Backend(ctx), max_batch=B)
th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
dth = torch.from_numpy(th).cuda()
out = torch.empty(B * 8, dtype=torch.float64, device="cuda")
L = g.lib()
for it in range(3):
    torch.cuda.synchronize(); t = time.time()
    g._check(L.gpemu_eval_batch_device(ev.handle, g._vp(dth.data_ptr()), B, g._vp(out.data_ptr())))
    torch.cuda.synchronize(); dt = time.time() - t
    rec = out.view(B, 8).cpu().numpy()
    print(f"n={n} d={d} B={B}: {dt*1e3:.1f} ms  {B/dt:.1f} evals/s  {B*n**3/3/dt/1e12:.2f} TFLOP/s(chol) "
          f"status={np.unique(rec[:,5])} neg2[0]={rec[0,0]:.6f}", flush=True)
