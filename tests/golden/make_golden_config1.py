"""The BASELINE configs[1] batch exactly as bench.py times it (paper_2311_01135_b200.synth
batch(256, 9, seed=1000)), labelled by the REFERENCE (deskdft) in this container at the
benchmark settings (STO-3G B3LYP, grid level 0, 20 fixed SCF iterations) in both f64 and f32
-> tests/golden/config1_batch.json.

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/confgen/src:/root/reference/pkg/tests \\
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_config1.py [n_mol]

tests/test_parity_scale.py compares the device's labels (f64 build: <= 1e-6 Ha, <= 1e-5 eV;
f32 build: the measured tolerance) with these records and
tools/parity_report.py turns them into the MAE / max tables of profiles/."""
import json
import multiprocessing as mp
import os
import sys
from concurrent.futures import ProcessPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

from make_golden import _job  # noqa: E402  (runs deskdft.scf on one molecule)
from paper_2311_01135_b200 import synth  # noqa: E402

KEEP = ("E_total", "gap_ev", "homo", "lumo", "iterations", "converged", "n_ao", "components")


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    mols = synth.batch(256, 9, seed=1000)[:n]
    jobs = []
    for m in mols:
        for prec in ("f64", "f32"):
            jobs.append((list(m.atomic_numbers), m.positions.tolist(),
                         dict(max_iterations=20, convergence_std=0.0, grid_level=0, precision=prec)))
    with ProcessPoolExecutor(os.cpu_count() or 1, mp_context=mp.get_context("spawn")) as ex:
        recs = list(ex.map(_job, jobs, chunksize=2))
    out = {"generator": "synth.batch(256, 9, seed=1000)",
           "options": {"max_iterations": 20, "convergence_std": 0.0, "grid_level": 0, "screen_eps": 1e-12},
           "molecules": []}
    for k, m in enumerate(mols):
        rec = {"id": m.id, "Z": list(m.atomic_numbers), "pos_bohr": m.positions.tolist()}
        for prec, r in zip(("f64", "f32"), recs[2 * k:2 * k + 2]):
            d = {key: r[key] for key in KEEP}
            d["last5"] = r["history"][-5:]
            rec[prec] = d
        out["molecules"].append(rec)
    with open(os.path.join(HERE, "config1_batch.json"), "w") as fh:
        json.dump(out, fh)
    print("wrote", len(out["molecules"]), "molecules")


if __name__ == "__main__":
    main()
