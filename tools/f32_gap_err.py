"""configs[1] batch, f32 build vs the reference's f64 labels: error by SCF settledness (GPU box)."""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01135_b200 import SCFOptions, load_basis, properties, scf_batch, Molecule
recs = json.load(open("tests/golden/config1_batch.json"))["molecules"]
mols = [Molecule(tuple(r["Z"]), np.array(r["pos_bohr"])) for r in recs]
std5 = np.array([np.std(r["f64"]["last5"]) for r in recs])
rs = scf_batch(mols, load_basis("sto-3g"), SCFOptions(precision="f32", max_iterations=20, convergence_std=0.0, grid_level=0))
dE = np.array([r.E_total - rec["f64"]["E_total"] for r, rec in zip(rs, recs)])
dg = np.array([properties(r)["gap"] - rec["f64"]["gap_ev"] for r, rec in zip(rs, recs)])
for lo, hi in ((0, 1e-7), (1e-7, 1e-5), (1e-5, 1e-3), (1e-3, 1e-2), (1e-2, 1e9)):
    k = (std5 >= lo) & (std5 < hi)
    if k.sum():
        print(f"std5 in [{lo:g}, {hi:g}): n={k.sum():3d}  |dE| max {np.abs(dE[k]).max():.3g} mean {np.abs(dE[k]).mean():.3g} Ha   |dgap| max {np.abs(dg[k]).max():.3g} mean {np.abs(dg[k]).mean():.3g} eV")
w = np.argsort(-np.abs(dg))[:6]
print("worst gap:", [(int(i), float(std5[i]), float(dg[i]), float(dE[i])) for i in w])
