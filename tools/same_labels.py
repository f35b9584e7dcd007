"""Print a checksum of the configs[1] batch labels (f32 and f64) for bitwise A/B of two builds."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2311_01135_b200 import synth, SCFOptions, load_basis, scf_batch
mols = synth.batch(int(sys.argv[1]) if len(sys.argv) > 1 else 64, 9, seed=1000)
for prec in ("f32", "f64"):
    rs = scf_batch(mols, load_basis("sto-3g"), SCFOptions(max_iterations=20, convergence_std=0.0, grid_level=0,
                                                         precision=prec))
    e = np.array([r.E_total for r in rs])
    print(prec, hashlib.md5(e.tobytes()).hexdigest(), e[:3])
