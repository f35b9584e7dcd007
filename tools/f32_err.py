"""f32 build vs the reference's golden f64 / f32 labels on the synthetic records
(tests/golden/golden.json): per-molecule |dE| (Ha) and |d gap| (eV), next to the
reference's own f32-vs-f64 spread."""
import json, os, sys
import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01135_b200 import Molecule, SCFOptions, load_basis, properties, scf_batch

g = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden.json")))
recs = list(g["synth"].values())
mols = [Molecule(tuple(r["Z"]), np.array(r["pos"])) for r in recs]
rs = scf_batch(mols, load_basis("sto-3g"), SCFOptions(precision="f32", max_iterations=20,
                                                        convergence_std=0.0, grid_level=0))
for r, rec in zip(rs, recs):
    a, b = rec["f64"], rec["f32"]
    print("n_ao %3d  dE %.2e (ref spread %.2e)  dgap %.2e eV (ref spread %.2e)  gap %.3f" % (
        r.n_ao, abs(r.E_total - a["E_total"]), abs(b["E_total"] - a["E_total"]),
        abs(properties(r)["gap"] - a["gap_ev"]), abs(b["gap_ev"] - a["gap_ev"]), a["gap_ev"]))
