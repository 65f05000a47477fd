"""Per-task timeline of one C3-shaped launch WITH the list-schedule ticket table (the bench's
order): tickets are decoded through gpemu_ticket_order. Per task kind: mainloop time (start ->
GEMM end: dependency waits + DMMA) against K, the epilogue, and the SM-time split.
usage: dag_phases_table.py [n d B]"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

n, d, B = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 10, 100)))
rng = np.random.default_rng(0)
X = rng.random((n, d))
y = np.sin(3 * X).sum(1)
ctx = g.Context(0)
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=B)
th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
ev.eval_batch(th)
ev.dag_profile(True)
ev.eval_batch(th)
p = ev.dag_profile(False, read=True)
NT = (n + 127) // 128
nt = B * NT * (NT + 1) // 2
order = np.empty(nt, dtype=np.int32)
g._check(g.lib().gpemu_ticket_order(B, NT, ctx.num_sms, order.ctypes.data_as(C.c_void_p), nt))
bpos, I, j = order >> 16, (order >> 8) & 255, order & 255
tr = p["trace"].astype(np.int64)
m = min(nt, len(tr))
tr = tr[:m].astype(np.float64) / 1e3
bpos, I, j = bpos[:m], I[:m], j[:m]
ok = tr[:, 0] > 0
t0 = tr[ok, 0].min()
span = tr[ok, 3].max() - t0
main = tr[:, 1] - tr[:, 0]
epi = tr[:, 2] - tr[:, 1]
tot = ctx.num_sms * span
print(f"n={n} B={B}: {ok.sum()} of {nt} tasks traced, span {span / 1e3:.2f} ms; SM-time: mainloop "
      f"{main[ok].sum() / tot:.3f}, epilogue {epi[ok].sum() / tot:.3f}")
tile = 2 * 128 ** 3 / (37.0e12 / ctx.num_sms) * 1e6
for name, sel, w in (("OFF", I != j, 1.0), ("DIAG", I == j, 17 / 32)):
    s = ok & sel
    A = np.stack([np.ones(s.sum()), j[s]], 1)
    coef, *_ = np.linalg.lstsq(A, main[s], rcond=None)
    print(f"{name}: {s.sum()} tasks, mainloop = {coef[0]:.2f} + {coef[1]:.2f}*K us (DMMA-bound {w * tile:.2f}*K); "
          f"epilogue mean {epi[s].mean():.2f} us; mainloop SM-share {main[s].sum() / tot:.3f}")
    for kk in (1, 8, 16, 24, 31):
        q = s & (j == kk)
        if q.any():
            print(f"   K={kk:2d}: mainloop median {np.median(main[q]):7.2f} us, epilogue median {np.median(epi[q]):6.2f}")

# Dependency slack: for every task, the publish time of its last input (stamp 2 of the producer)
# against its own start. A task that starts before its last input is published waits inside its
# mainloop (the flag wait); list-schedule estimates that are off show up here.
pub = {}
for t in np.nonzero(ok)[0]:
    pub[(int(bpos[t]), int(I[t]), int(j[t]))] = tr[t, 2]
for name, sel in (("OFF", I != j), ("DIAG", I == j)):
    late, lastk = [], []
    for t in np.nonzero(ok & sel)[0]:
        b, ii, jj = int(bpos[t]), int(I[t]), int(j[t])
        ins = [(b, jj, K) for K in range(jj)] + ([(b, ii, K) for K in range(jj)] + [(b, jj, jj)] if ii != jj else [])
        if not ins:
            continue
        lp = max(pub.get(k, 0.0) for k in ins)
        late.append(lp - tr[t, 0])
        lastk.append(tr[t, 1] - lp)  # last input published -> GEMM end
    late = np.array(late)
    lastk = np.array(lastk)
    print(f"{name}: last input published after task start in {np.mean(late > 0):.1%} of tasks; "
          f"by {np.mean(np.maximum(late, 0)):.1f} us on average ({np.median(late):.1f} median); "
          f"last input -> GEMM end median {np.median(lastk):.1f} us")
