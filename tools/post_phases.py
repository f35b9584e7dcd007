"""Post-kernel phase cycles (clock64 ticks of thread 0, summed over iterations; scf.cu k_post):
0 J/K/V partial reduction, 1 F + energies, 2 DIIS error + B row, 3 extrapolation,
5 eigenvalue sort, 6 C, density, damping, 7 X^T F X, 8 purification (+ its density GEMMs),
9 Jacobi."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2311_01135_b200 import synth, SCFOptions, load_basis
from paper_2311_01135_b200.engine import Plan
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
mols = synth.batch(n, 9, seed=1000)
opts = SCFOptions(max_iterations=20, convergence_std=0.0, grid_level=0, precision="f32")
with Plan(mols, load_basis("sto-3g"), opts.engine()) as p:
    p.run()
    p.fetch(want_C=False)
    d = np.array([p.get("dbg", m) for m in range(n)])
names = ["reduce", "F+E", "DIIS err+B", "extrap", "purification steps (count)", "sort", "C/dens/damp", "X^T F X", "purification",
         "jacobi"]
tot = d[:, :10].sum(axis=1) - d[:, 4]
print("purification steps per molecule: mean", d[:, 4].mean(), "max", d[:, 4].max(), "min", d[:, 4].min())
print("mean cycles per molecule over 20 iterations:", tot.mean())
for k, nm in enumerate(names):
    print(f"{nm:18s} {d[:, k].mean():12.0f}  {100 * d[:, k].mean() / tot.mean():5.1f}%")
print("inside purification: bounds", d[:, 14].mean(), "steps", d[:, 15].mean())
print("jacobi sweeps (sum)", d[:, 10].mean(), "iterations", d[:, 11].mean())
