import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01135_b200 import synth, SCFOptions, load_basis
from paper_2311_01135_b200.engine import Plan
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mols = synth.batch(n, 9, seed=1)
for prec in ("f32", "f64"):
    opts = SCFOptions(max_iterations=20, convergence_std=0.0, grid_level=0, precision=prec)
    with Plan(mols, load_basis("sto-3g"), opts.engine()) as p:
        p.run()
        for m in range(3):
            d = p.get("dbg", m)
            print(prec, "mol", m, "N", p.pk.mol_nao[m], "post phases (Mcycles, summed over calls):",
                  [round(x / 1e6, 3) for x in d[:7]], "jacobi sweeps total", d[10], "calls", d[11],
                  "orth cycles %.3fM sweeps %d" % (d[12] / 1e6, d[13]), "jacobi angle/apply Mcycles %.3f %.3f" % (d[14] / 1e6, d[15] / 1e6))
