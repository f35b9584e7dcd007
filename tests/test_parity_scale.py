"""Parity at the benchmarked configuration: the exact configs[1] batch bench.py times
(synth.batch(256, 9, seed=1000), STO-3G B3LYP, grid level 0, 20 fixed SCF iterations)
against the REFERENCE's own labels of those 256 molecules
(tests/golden/config1_batch.json, produced by tests/golden/make_golden_config1.py running
deskdft.scf, reference scf.py:139-210, in the build container).

Tolerances (north_star; measured values in DESIGN.md section 5 / profiles/r2_parity_report.md):
* f64 build: |dE| <= 1e-6 Ha and |dgap| <= 1e-5 eV on ALL 256 molecules (measured max
  9.5e-8 Ha on the one molecule whose SCF swings by 26 Ha between iterations, <= 2.3e-10 Ha on
  the rest), and <= 1e-9 Ha on the molecules whose reference SCF settles in 20 iterations
  (std of the last five energies < 1e-5 Ha; measured max 3.4e-12 Ha).
* f32 build vs the reference f64 answer, over every molecule whose reference SCF is not
  divergent (std of the last five energies < 1e-2 Ha: 253 of 256): |dE| <= 3e-5 Ha (measured
  max 1.6e-5); |dgap| <= 5e-5 eV on the 235 settled molecules (std < 1e-5 Ha; measured max
  3.0e-5) and <= 1.5e-4 eV on the 18 that still oscillate after 20 iterations, where rounding
  differences are amplified (measured max 5.3e-5; it moves with the summation order of the
  J/K kernel: 3.7e-5 with 12 J/K CTAs per molecule, 5.3e-5 with 4).  The reference's own f32
  run lies up to 6.9e-4 Ha from its f64 answer on the settled molecules (it diagonalises and
  extrapolates in f32 LAPACK; the device keeps Fock / DIIS / eigensolver in f64).
"""
import json
import os

import numpy as np
import pytest

from paper_2311_01135_b200 import Molecule, SCFOptions, properties, scf_batch

pytestmark = pytest.mark.gpu

OPTS = dict(max_iterations=20, convergence_std=0.0, grid_level=0)


@pytest.fixture(scope="module")
def config1():
    with open(os.path.join(os.path.dirname(__file__), "golden", "config1_batch.json")) as fh:
        d = json.load(fh)
    recs = d["molecules"]
    mols = [Molecule(tuple(r["Z"]), np.array(r["pos_bohr"])) for r in recs]
    std5 = np.array([np.std(r["f64"]["last5"]) for r in recs])
    return recs, mols, std5


def test_config1_inputs_are_the_bench_batch(config1):
    """The fixture's molecules are the bench's own inputs (same generator and seed)."""
    from paper_2311_01135_b200 import synth

    recs, mols, _ = config1
    gen = synth.batch(256, 9, seed=1000)
    assert len(recs) == 256
    for m, g in zip(mols, gen):
        assert m.atomic_numbers == g.atomic_numbers
        np.testing.assert_array_equal(m.positions, g.positions)


def test_config1_batch_f64_vs_reference(gpu_lib, sto3g, config1):
    recs, mols, std5 = config1
    rs = scf_batch(mols, sto3g, SCFOptions(precision="f64", **OPTS))
    dE = np.array([r.E_total - rec["f64"]["E_total"] for r, rec in zip(rs, recs)])
    dg = np.array([properties(r)["gap"] - rec["f64"]["gap_ev"] for r, rec in zip(rs, recs)])
    assert all(r.n_ao == rec["f64"]["n_ao"] for r, rec in zip(rs, recs))
    assert np.abs(dE).max() <= 1e-6, np.abs(dE).max()
    assert np.abs(dg).max() <= 1e-5, np.abs(dg).max()
    settled = std5 < 1e-5
    assert settled.sum() >= 200
    assert np.abs(dE[settled]).max() <= 1e-9, np.abs(dE[settled]).max()
    for r, rec in zip(rs, recs):   # the last five energies too, not only the final one
        np.testing.assert_allclose(r.energy_history[-5:], rec["f64"]["last5"], atol=1e-6, rtol=0)


def test_config1_batch_f32_vs_reference(gpu_lib, sto3g, config1):
    recs, mols, std5 = config1
    rs = scf_batch(mols, sto3g, SCFOptions(precision="f32", **OPTS))
    dE = np.array([r.E_total - rec["f64"]["E_total"] for r, rec in zip(rs, recs)])
    dg = np.array([properties(r)["gap"] - rec["f64"]["gap_ev"] for r, rec in zip(rs, recs)])
    ok = std5 < 1e-2
    assert ok.sum() >= 250
    settled = std5 < 1e-5
    assert settled.sum() >= 200
    assert np.abs(dE[ok]).max() <= 3e-5, np.abs(dE[ok]).max()
    assert np.abs(dg[settled]).max() <= 5e-5, np.abs(dg[settled]).max()
    assert np.abs(dg[ok]).max() <= 1.5e-4, np.abs(dg[ok]).max()
    # mean error well inside the reference's own f32-vs-f64 spread
    own = np.array([abs(rec["f32"]["E_total"] - rec["f64"]["E_total"]) for rec in recs])
    assert np.abs(dE[ok]).mean() < 0.25 * own[ok].mean()
