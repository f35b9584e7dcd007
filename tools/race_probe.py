"""compute-sanitizer target: one small f32 batch with an 11-heavy (N > 64) molecule mix."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01135_b200 import synth, SCFOptions, load_basis, scf_batch
b = load_basis("sto-3g")
opts = SCFOptions(max_iterations=int(sys.argv[1]) if len(sys.argv) > 1 else 4, convergence_std=0.0,
                  grid_level=0, precision="f32")
mols = synth.batch(2, 11, seed=41) + synth.batch(2, 3, seed=42)
print([r.E_total for r in scf_batch(mols, b, opts)])
