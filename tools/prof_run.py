"""Small profiling workload: N molecules x 9 heavy, f32/f64, level 0, K iterations, one plan run."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01135_b200 import synth, SCFOptions, load_basis
from paper_2311_01135_b200.engine import Plan
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
it = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prec = sys.argv[3] if len(sys.argv) > 3 else "f32"
heavy = [int(x) for x in sys.argv[4].split(",")] if len(sys.argv) > 4 else [9]
mols = synth.batch(n, heavy if len(heavy) > 1 else heavy[0], seed=1)
opts = SCFOptions(max_iterations=max(it, 5), convergence_std=0.0, grid_level=0, precision=prec)
eo = opts.engine(); eo.max_iterations = it
with Plan(mols, load_basis("sto-3g"), eo) as p:
    p.run(); r = p.fetch(want_C=False)
    print("E0", r.E_total[0])
