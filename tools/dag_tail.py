"""End-of-launch tail of the DAG engine: per-task timeline of one C3 batch (B=100) and the
distribution of task end times -- how long SMs idle after the ticket counter runs dry."""
import sys

import os

import numpy as np

# tickets are decoded here with the kernel's built-in column order: keep the list-schedule table off
os.environ["GPEMU_TICKET_ORDER"] = "0"

sys.path.insert(0, "/root/repo")
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
tr = p["trace"].astype(np.int64)
NT = (n + 127) // 128
nt = B * NT * (NT + 1) // 2
tr = tr[:nt]
t0 = tr[:, 0].min()
end = tr[:, 3].max()
starts = np.sort(tr[:, 0]) - t0
ends = np.sort(tr[:, 3]) - t0
span = (end - t0) / 1e3
last_start = starts[-1] / 1e3
print(f"n={n} B={B}: {nt} tasks, span {span:.1f} us, last ticket taken at {last_start:.1f} us "
      f"({100 * (span - last_start) / span:.1f}% of the launch after the counter runs dry)")
for q in (0.5, 0.9, 0.99):
    print(f"  {int(q * 100)}% of tasks finished by {np.quantile(ends, q) / 1e3:.1f} us")
# busy fraction over the last 10% of the launch: sum over tasks of overlap with the window
w0 = t0 + 0.9 * (end - t0)
busy = np.clip(np.minimum(tr[:, 3], end) - np.maximum(tr[:, 0], w0), 0, None).sum()
print(f"  SM busy fraction in the last 10% of the launch: {busy / (148 * 0.1 * (end - t0)):.2f}")
