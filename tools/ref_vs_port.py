"""Build-container only (needs /root/reference): time the real reference (deskdft, numba)
and the oracle port on the same molecules of the bench generator, one process per core,
to state how the `--impl reference` arm (which runs the port; the reference cannot travel
to the GPU box) compares with the reference itself."""
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg/src"


def _ref_one(args):
    z, pos = args
    sys.path.insert(0, REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    os.environ["OMP_NUM_THREADS"] = "1"
    import numba
    numba.set_num_threads(1)
    from deskdft.basis import load_basis
    from deskdft.molio import Molecule
    from deskdft.scf import SCFOptions, scf
    m = Molecule(tuple(z), np.asarray(pos))
    t = time.perf_counter()
    r = scf(m, load_basis("sto-3g"), SCFOptions(precision="f32", grid_level=0, convergence_std=0.0,
                                                 max_iterations=20))
    return r.E_total, time.perf_counter() - t


def _port_one(args):
    z, pos = args
    sys.path.insert(0, ROOT)
    os.environ["OMP_NUM_THREADS"] = "1"
    from oracle import port
    t = time.perf_counter()
    r = port.scf(port.Mol(tuple(z), np.asarray(pos)), "f32", 20, 0.0, 0)
    return r.E_total, time.perf_counter() - t


def main():
    sys.path.insert(0, ROOT)
    from paper_2311_01135_b200 import synth
    cores = os.cpu_count() or 1
    mols = synth.batch(cores, 9, seed=5000)
    work = [(m.atomic_numbers, m.positions) for m in mols]
    ctx = mp.get_context("spawn")
    with ctx.Pool(cores) as pool:
        pool.map(_ref_one, work[:cores])                 # numba JIT warm-up
        t = time.perf_counter()
        ref = pool.map(_ref_one, work)
        t_ref = time.perf_counter() - t
    with ctx.Pool(cores) as pool:
        pool.map(_port_one, work[:1])
        t = time.perf_counter()
        prt = pool.map(_port_one, work)
        t_port = time.perf_counter() - t
    dE = max(abs(a[0] - b[0]) for a, b in zip(ref, prt))
    print(f"cores {cores}: deskdft {len(work) / t_ref:.3f} mol/s, oracle port {len(work) / t_port:.3f} mol/s, "
          f"ratio {t_port / t_ref:.2f}; max |dE| {dE:.2e} Ha")


if __name__ == "__main__":
    main()
