"""Determinism probe: the same batch alone several times, and mixed-size batches in flight."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2311_01135_b200 import synth, SCFOptions, load_basis, scf_batch
from paper_2311_01135_b200.pipeline import label_batches
b = load_basis("sto-3g")
opts = SCFOptions(max_iterations=6, convergence_std=0.0, grid_level=0, precision="f32")
heavy = [2, 11, 3, 10, 2, 11, 4, 9, 2, 11]
batches = [synth.batch(8, h, seed=40 + k) for k, h in enumerate(heavy)]
for k in (1, 2, 7):
    e = [np.array([r.E_total for r in scf_batch(batches[k], b, opts)]) for _ in range(3)]
    print(k, "alone run-to-run max diff", max(np.abs(x - e[0]).max() for x in e))
got = {k: res for k, res, _ in label_batches(batches, b, opts, workers=4)}
for k in (1, 2, 7):
    ref = np.array([r.E_total for r in scf_batch(batches[k], b, opts)])
    g = np.array([r.E_total for r in got[k]])
    print(k, "in-flight vs alone", np.abs(g - ref).max())
