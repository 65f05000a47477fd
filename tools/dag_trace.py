"""Per-task timeline of one DAG launch (globaltimer ns): the serial chain of a small batch.
usage: dag_trace.py n d B
Prints, per tile column j of candidate 0: DIAG(j) and OFF(j+1, j) start / GEMM end / publish
times relative to the launch start, and per-task-kind averages."""
import sys

import os

import numpy as np

# tickets are decoded here with the kernel's built-in column order: keep the list-schedule table off
os.environ["GPEMU_TICKET_ORDER"] = "0"

sys.path.insert(0, ".")
import paper_1203_1269_b200.gpemu as g  # noqa: E402

n, d, B = (int(a) for a in sys.argv[1:4])
engine = "dag"
rng = np.random.default_rng(0)
X = rng.random((n, d))
y = np.sin(3 * X).sum(1)
ctx = g.Context(0, engine)
ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=B)
th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
ev.eval_batch(th)
ev.dag_profile(True)
ev.eval_batch(th)
p = ev.dag_profile(False, read=True)
tr = p["trace"].astype(np.int64)
NT = (n + 127) // 128


def decode_left(t):
    if t < B:
        return t, 0, 0, 0
    t -= B
    jj = 0
    while t >= B * (NT - jj):
        t -= B * (NT - jj)
        jj += 1
    per = NT - jj
    b, pos = divmod(t, per)
    if pos == 0:
        return b, jj + 1, jj, 0
    if pos == per - 1:
        return b, jj + 1, jj + 1, 0
    return b, jj + pos + 1, jj, 0


nt = B * NT * (NT + 1) // 2
rows = []
for t in range(min(nt, len(tr))):
    if tr[t, 0] == 0:
        continue
    b, I, j, u = decode_left(t)
    rows.append((t, b, I, j, u, *tr[t]))
t0 = min(r[5] for r in rows)
print(f"n={n} B={B}: {len(rows)} tasks, makespan "
      f"{(max(r[8] for r in rows) - t0) / 1e3:.1f} us")
key = {(r[1], r[2], r[3], r[4]): r for r in rows}
print(" j   DIAG start/gemm/pub (us)        OFF(j+1,j) start/gemm/pub")
for j in range(NT):
    dg = key.get((0, j, j, 0))
    of = key.get((0, j + 1, j, 0))
    f = lambda r: "%8.1f %8.1f %8.1f" % ((r[5] - t0) / 1e3, (r[6] - t0) / 1e3, (r[7] - t0) / 1e3) if r else " " * 26
    print(f"{j:3d} {f(dg)}   {f(of)}")
for name, sel in (("DIAG", lambda r: r[2] == r[3]), ("OFF", lambda r: r[2] != r[3])):
    rs = [r for r in rows if sel(r)]
    if rs:
        gem = np.mean([r[6] - r[5] for r in rs]) / 1e3
        epi = np.mean([r[7] - r[6] for r in rs]) / 1e3
        print(f"{name}: {len(rs)} tasks, mean start->gemm-end {gem:.1f} us, gemm-end->publish {epi:.1f} us")
