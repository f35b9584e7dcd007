"""Pin the CPU oracle (oracle/) against vectors produced by the reference itself."""
import numpy as np
import pytest


def _mol(oracle, rec):
    return oracle.Mol(tuple(rec["Z"]), np.array(rec["pos"]))


def test_config1_water_known_answer(oracle, golden):
    """BASELINE configs[0] known answer: f64 to 1e-10 Ha."""
    rec = golden["cfg1_water"]
    r = oracle.scf(_mol(oracle, rec), "f64", max_iterations=20, convergence_std=0.0, grid_level=0)
    assert abs(r.E_total - rec["f64"]["E_total"]) < 1e-10
    assert abs(r.E_total - (-75.317748525602)) < 1e-9
    np.testing.assert_allclose(r.epsilon, rec["f64"]["epsilon"], atol=1e-10)
    np.testing.assert_allclose(r.history, rec["f64"]["history"], atol=1e-10)


@pytest.mark.parametrize("name", ["h2", "h2o", "nh3", "ch4", "hf", "dh2o"])
def test_one_electron_and_eri(oracle, golden, golden_arrays, name):
    rec = golden["small"][name]
    m = _mol(oracle, rec)
    ao = oracle.expand(m)
    np.testing.assert_allclose(ao.prim_coef, golden_arrays[f"{name}_prim_coef"], rtol=0, atol=1e-14)
    S, T, V = oracle.one_electron(ao, m)
    for k, X in (("S", S), ("T", T), ("V", V)):
        np.testing.assert_allclose(X, golden_arrays[f"{name}_{k}"], rtol=0, atol=1e-12)
    for tag, eps in (("eri0", 0.0), ("eri9", 1e-9)):
        e = oracle.eri_packed(ao, eps)
        ijkl = np.stack([e.i, e.j, e.k, e.l]).astype(np.int32)
        assert np.array_equal(ijkl, golden_arrays[f"{name}_{tag}_ijkl"])
        np.testing.assert_allclose(e.values, golden_arrays[f"{name}_{tag}_v"], rtol=1e-12, atol=1e-15)
        assert np.array_equal(e.degeneracy.astype(np.int32), golden_arrays[f"{name}_{tag}_deg"])
    J, K = oracle.build_jk(oracle.eri_packed(ao, 0.0), golden_arrays[f"{name}_rho"])
    np.testing.assert_allclose(J, golden_arrays[f"{name}_J"], atol=1e-12)
    np.testing.assert_allclose(K, golden_arrays[f"{name}_K"], atol=1e-12)


@pytest.mark.parametrize("name", ["h2o", "dh2o", "ch4"])
def test_grid_and_xc(oracle, golden, golden_arrays, name):
    rec = golden["small"][name]
    m = _mol(oracle, rec)
    ao = oracle.expand(m)
    for lvl in (0, 1):
        pts, w = oracle.build_grid(m, lvl)
        np.testing.assert_allclose(pts, golden_arrays[f"{name}_grid{lvl}_pts"], atol=1e-13)
        np.testing.assert_allclose(w, golden_arrays[f"{name}_grid{lvl}_w"], rtol=1e-12, atol=1e-16)
        phi, gphi = oracle.eval_ao(ao, pts)
        e, V = oracle.xc_matrix(w, phi, gphi, golden_arrays[f"{name}_rho"])
        assert abs(e - rec[f"exc{lvl}"]) < 1e-11
        np.testing.assert_allclose(V, golden_arrays[f"{name}_vxc{lvl}"], atol=1e-11)


def test_b3lyp_pointwise(oracle, golden_arrays):
    g = golden_arrays
    e, vr, vs = oracle.b3lyp(g["b3lyp_n"], g["b3lyp_s"])
    for a, b in ((e, g["b3lyp_exc"]), (vr, g["b3lyp_vrho"]), (vs, g["b3lyp_vsigma"])):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=0)


def test_diis_cases(oracle, golden_arrays):
    for case in range(6):
        F, E = golden_arrays[f"diis{case}_F"], golden_arrays[f"diis{case}_E"]
        out = oracle.diis_step([(F[a], E[a]) for a in range(len(F))])
        np.testing.assert_allclose(out, golden_arrays[f"diis{case}_out"], atol=1e-11)


@pytest.mark.slow
@pytest.mark.parametrize("idx", [0, 1])
def test_synthetic_scf_f64(oracle, golden, idx):
    """Full fixed-20-iteration SCF on 9-heavy synthetic molecules (reference f64 records)."""
    mid = sorted(golden["synth"])[idx]
    rec = golden["synth"][mid]
    r = oracle.scf(_mol(oracle, rec), "f64", max_iterations=20, convergence_std=0.0, grid_level=0)
    assert abs(r.E_total - rec["f64"]["E_total"]) < 1e-9
    assert abs(r.gap_ev - rec["f64"]["gap_ev"]) < 1e-8


def test_h2_known_answers(oracle, golden):
    """Szabo-Ostlund H2 textbook integrals (reference test_integrals.py:31-41) via the oracle."""
    m = oracle.Mol((1, 1), np.array([[0, 0, 0], [0, 0, 1.4]], float))
    ao = oracle.expand(m)
    S, T, V = oracle.one_electron(ao, m)
    assert S[0, 1] == pytest.approx(0.6593, abs=2e-4)
    assert T[0, 0] == pytest.approx(0.7600, abs=2e-4)
    assert V[0, 0] == pytest.approx(-1.8804, abs=2e-4)
    d = oracle.unpack(oracle.eri_packed(ao, 0.0))
    assert d[0, 0, 0, 0] == pytest.approx(0.7746, abs=2e-4)
    assert d[0, 1, 0, 1] == pytest.approx(0.2970, abs=2e-4)
