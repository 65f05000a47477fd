"""Per-phase SM-time split of one DAG launch from the task timeline (globaltimer ns):
ticket gaps, start->mainloop end (dependency wait + GEMM), epilogue (TRSM/POTRF + store),
publish->task end. Fits mainloop time = a + b*K per task kind (K = tile-columns reduced)."""
import sys

import os

import numpy as np

# tickets are decoded here with the kernel's built-in column order: keep the list-schedule table off
os.environ["GPEMU_TICKET_ORDER"] = "0"

sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

n, d, B = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 10, 100)))
rng = np.random.default_rng(0)
X = rng.random((n, d))
y = np.sin(3 * X).sum(1)
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(g.Context(0)), max_batch=B)
th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
ev.eval_batch(th)
ev.dag_profile(True)
ev.eval_batch(th)
p = ev.dag_profile(False, read=True)
NT = (n + 127) // 128
nt = B * NT * (NT + 1) // 2
tr = p["trace"].astype(np.int64)[:nt].astype(np.float64) / 1e3  # us
kind = np.empty(nt, dtype=np.int8)  # 0 OFF, 1 DIAG
K = np.empty(nt, dtype=np.int32)
t = 0
kind[:B] = 0  # OFF(1,0)
K[:B] = 0
t = B
for jj in range(NT - 1):
    per = NT - jj
    pos = np.arange(per)
    k = np.where(pos == per - 1, 1, 0)
    kk = np.full(per, jj + 1)  # OFF(I, jj+1)... reduces over columns 0..jj; DIAG(jj+1) too
    kind[t:t + B * per] = np.tile(k, B)
    K[t:t + B * per] = np.tile(kk, B)
    t += B * per
t0 = tr[:, 0].min()
span = tr[:, 3].max() - t0
main = tr[:, 1] - tr[:, 0]
epi = tr[:, 2] - tr[:, 1]
tail = tr[:, 3] - tr[:, 2]
busy = (tr[:, 3] - tr[:, 0]).sum()
tot = 148 * span
print(f"n={n} B={B}: span {span / 1e3:.2f} ms; SM-time share: start->mainloop-end {main.sum() / tot:.3f}, "
      f"epilogue {epi.sum() / tot:.3f}, publish->end {tail.sum() / tot:.3f}, outside tasks {(tot - busy) / tot:.3f}")
peak_tile = 2 * 128 ** 3 / (37.0e12 / 148) * 1e6
print(f"ideal 128^3 DMMA tile at the per-SM measured peak: {peak_tile:.2f} us")
for kname, kv in (("OFF", 0), ("DIAG", 1)):
    m = kind == kv
    A = np.stack([np.ones(m.sum()), K[m]], 1)
    coef, *_ = np.linalg.lstsq(A, main[m], rcond=None)
    print(f"{kname}: {m.sum()} tasks, mainloop = {coef[0]:.2f} + {coef[1]:.2f}*K us; "
          f"epilogue mean {epi[m].mean():.2f} us, publish->end {tail[m].mean():.2f} us")
    for kk in (1, 8, 16, 24, 31):
        s = m & (K == kk)
        if s.any():
            print(f"   K={kk:2d}: mainloop median {np.median(main[s]):7.2f} us, epilogue median {np.median(epi[s]):6.2f}")
