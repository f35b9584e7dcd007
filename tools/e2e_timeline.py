"""Timeline of label_batches (bench e2e path): per-batch host phases vs wall clock."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.cuda.init()
from paper_2311_01135_b200 import synth, SCFOptions, load_basis, scf as scfmod
from paper_2311_01135_b200.pipeline import label_batches
from paper_2311_01135_b200.engine import Plan
b = load_basis("sto-3g")
opts = SCFOptions(max_iterations=20, convergence_std=0.0, grid_level=0, precision="f32")
batches = [synth.batch(256, 9, seed=1000 + 7919 * k) for k in range(3)]
log = []
orig_run, orig_fetch, orig_init = Plan.run, Plan.fetch, Plan.__init__
T0 = [0.0]
def tag(name, f):
    def w(self, *a, **k):
        t = time.perf_counter(); r = f(self, *a, **k)
        log.append((threading.get_ident() % 1000, name, 1e3 * (t - T0[0]), 1e3 * (time.perf_counter() - T0[0])))
        return r
    return w
Plan.__init__ = tag("create", orig_init); Plan.run = tag("run", orig_run); Plan.fetch = tag("fetch", orig_fetch)
list(label_batches(batches, b, opts, workers=3))
log.clear()
T0[0] = time.perf_counter()
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
for k, res, w in label_batches([batches[i % 3] for i in range(steps)], b, opts, workers=3):
    log.append((0, f"done{k}", 0.0, 1e3 * (time.perf_counter() - T0[0])))
torch.cuda.synchronize()
tot = 1e3 * (time.perf_counter() - T0[0])
for e in sorted(log, key=lambda x: x[3]): print("%4d %-8s %8.1f -> %8.1f ms" % e)
print("total %.1f ms, %.1f ms/step" % (tot, tot / steps))
