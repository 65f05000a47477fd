"""A/B timing of alternative builds of libgpemu_b200.so (paths in argv) on the C3 batch."""
import importlib, os, shutil, sys
import numpy as np
sys.path.insert(0, "/root/repo")
for path in sys.argv[1:]:
    import paper_1203_1269_b200.gpemu as g
    g._LIB = None
    g.LIB_PATH = os.path.abspath(path)
    n, d, B = 4096, 10, 100
    rng = np.random.default_rng(0)
    X = rng.random((n, d)); y = np.sin(3 * X).sum(1)
    ctx = g.Context(0)
    ev = g.ProfileEvaluator(g.new_dataset(X, y), 1.95, 0.0, g.Backend(ctx), max_batch=B)
    th = 10 ** rng.uniform(-1.0, 0.5, size=(B, d))
    ev.eval_batch(th)
    ev.set_profiling(True)
    for _ in range(4): r = ev.eval_batch(th)
    print(os.path.basename(path), "chol ms/step %.3f" % (ev.phase_ms(1)[0] / 4), "neg2[0] %.9f" % r["neg2"][0], flush=True)
    ev.close(); ctx.close()
