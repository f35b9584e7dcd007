"""Module-level (picklable) stand-ins for pipeline.label_batches, used by the CPU tests of the
multi-process paths: spawned processes must be able to import the labeler by name.  The
CPU oracle is test infrastructure; the product path never calls it."""
import os

import numpy as np


def oracle_label(batches, basis, opts, workers, device):
    from oracle import port
    from paper_2311_01135_b200.scf import OrbitalSolution, SCFResult

    log = os.environ.get("QM1B_TEST_DEVICE_LOG")
    for k, mols in enumerate(batches):
        out = []
        for m in mols:
            r = port.scf(port.Mol(tuple(m.atomic_numbers), np.asarray(m.positions)), opts.precision,
                         opts.max_iterations, opts.convergence_std, opts.grid_level)
            out.append(SCFResult(solution=OrbitalSolution(C=r.C, epsilon=r.epsilon, n_occ=r.n_occ),
                                 E_total=r.E_total, E_components=r.components,
                                 energy_history=list(r.history), converged=r.converged,
                                 iterations=r.iterations, n_ao=r.n_ao))
            if log:
                with open(log, "a") as fh:
                    fh.write(f"{device} {m.id}\n")
        yield k, out, 0.004 * len(mols)


def failing_label(batches, basis, opts, workers, device):
    if device == 1:
        raise RuntimeError("device 1 lost")
    yield from oracle_label(batches, basis, opts, workers, device)
