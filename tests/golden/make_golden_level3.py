"""configs[4]-shaped golden records from the REFERENCE (deskdft) in this container:
11-heavy-atom synthetic molecules (paper_2311_01135_b200.synth, seed 11), STO-3G B3LYP, f64,
grid level 3, converged to std(last 5 E) < 1e-9 (max 50 iterations) -> tests/golden/level3.json.

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/confgen/src:/root/reference/pkg/tests \
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_level3.py [n_mol]

The GPU test (tests/test_gpu_parity.py::test_config5_level3_against_reference) compares the
device's energies, gaps and iteration counts with these records."""
import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from make_golden import _job  # noqa: E402  (runs deskdft.scf on one molecule)
from paper_2311_01135_b200 import synth  # noqa: E402

OPTS = {"precision": "f64", "grid_level": 3, "convergence_std": 1e-9, "max_iterations": 50}


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
    mols = synth.batch(n, 11, seed=11)
    jobs = [(list(m.atomic_numbers), m.positions.tolist(), OPTS) for m in mols]
    with ProcessPoolExecutor(max_workers=min(n, os.cpu_count() or 1)) as ex:
        recs = list(ex.map(_job, jobs))
    out = {"options": OPTS, "generator": "synth.batch(n, 11, seed=11)",
           "molecules": [{"Z": j[0], "pos_bohr": j[1], **r} for j, r in zip(jobs, recs)]}
    with open(os.path.join(HERE, "level3.json"), "w") as fh:
        json.dump(out, fh)
    for r in recs:
        print(r["E_total"], r["gap_ev"], r["iterations"], r["converged"])


if __name__ == "__main__":
    main()
