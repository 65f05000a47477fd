"""Per-task-kind mainloop counters (DIAG vs OFF): thread 0 GEMM cycles, full-barrier waits and
producer flag waits, at C3 with the bench ticket order (dag_profile counters; diagnostics)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g
n, d, B = 4096, 10, 100
rng = np.random.default_rng(0)
X = rng.random((n, d)); y = np.sin(3 * X).sum(1)
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(g.Context(0)), max_batch=B)
th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
ev.eval_batch(th); ev.dag_profile(True); ev.eval_batch(th)
p = ev.dag_profile(False, read=True)
nd = p["n_diag"].sum(); no = p["n_off"].sum()
f = 1.965e3
print("DIAG per task us: gemm", p["diag_gemm"].sum() / nd / f, "full_wait(t0)", p["diag_full_wait"].sum() / nd / f)
print("OFF per task us: gemm", (p["gemm"].sum() - p["diag_gemm"].sum()) / no / f, "full_wait(t0)", p["full_wait"].sum() / no / f)
fw = p.get("flag_wait")
for k, v in p.items():
    if k not in ("trace",) and v.ndim == 1 and v.size == 256:
        print(k, "diag", v[128:].sum() / nd / f, "off", v[:128].sum() / no / f)
# POTRF phases, summed over the 8 warps (lane 0 of each) per DIAG task
for k in ("potrf_pivot", "potrf_bd_wait", "potrf_panel", "potrf_bp_wait", "potrf_update"):
    print(f"{k:14s} per DIAG task (sum over warps) {p[k].sum() / nd / f:8.2f} us")
print("potrf (thread 0 wall) per DIAG task", p["potrf"].sum() / nd / f)
