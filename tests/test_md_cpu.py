"""The device integral and functional math (csrc/md.cuh, csrc/b3lyp.cuh), compiled for the CPU
by tests/cpu_md, against the oracle: exact (eps = 0) ERIs to 1e-10 relative, S/T/V to 1e-12."""
import ctypes

import numpy as np
import pytest

from paper_2311_01135_b200 import batch, parse_xyz, synth

P = lambda a: a.ctypes.data_as(ctypes.c_void_p)


def _run(md_host, sto3g, m):
    pk = batch.pack([m], sto3g, None)
    n = int(pk.mol_nao[0])
    npp = n * (n + 1) // 2
    dense = np.zeros(npp * (npp + 1) // 2)
    S, T, V = np.zeros((n, n)), np.zeros((n, n)), np.zeros((n, n))
    xyz = np.ascontiguousarray(pk.atom_xyz[pk.shell_atom])
    md_host.md_molecule(ctypes.c_int(pk.n_shell), P(pk.shell_kind), P(pk.shell_ao), P(xyz), P(pk.shell_exp),
                        P(pk.shell_cs), P(pk.shell_cp), ctypes.c_int(n), ctypes.c_int(pk.n_atom),
                        P(pk.atom_xyz), P(pk.atom_z), ctypes.c_double(0.0), P(dense), P(S), P(T), P(V))
    return dense, S, T, V


@pytest.mark.parametrize("mol", ["dh2o", "nh3", "syn"])
def test_md_eri_and_stv_vs_oracle(md_host, oracle, sto3g, golden, mol):
    if mol == "syn":
        m = synth.batch(1, 4, seed=7)[0]
    else:
        rec = golden["small"][mol]
        from paper_2311_01135_b200 import Molecule
        m = Molecule(tuple(rec["Z"]), np.array(rec["pos"]))
    dense, S, T, V = _run(md_host, sto3g, m)
    om = oracle.Mol(m.atomic_numbers, m.positions)
    ao = oracle.expand(om)
    S0, T0, V0 = oracle.one_electron(ao, om)
    for a, b in ((S, S0), (T, T0), (V, V0)):
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)
    e = oracle.eri_packed(ao, 0.0)
    ij = e.i.astype(np.int64) * (e.i.astype(np.int64) + 1) // 2 + e.j
    kl = e.k.astype(np.int64) * (e.k.astype(np.int64) + 1) // 2 + e.l
    mine = dense[ij * (ij + 1) // 2 + kl]
    assert len(mine) == len(dense)            # the dense store is exactly the canonical set
    err = np.abs(mine - e.values)
    assert err.max() < 1e-13
    big = np.abs(e.values) > 1e-6
    assert (err[big] / np.abs(e.values[big])).max() < 1e-10


def test_b3lyp_device_math_vs_reference_vectors(md_host, golden_arrays):
    g = golden_arrays
    n, s = g["b3lyp_n"], g["b3lyp_s"]
    e, vr, vs = (np.zeros_like(n) for _ in range(3))
    md_host.md_b3lyp(ctypes.c_int64(len(n)), P(n), P(s), P(e), P(vr), P(vs))
    for a, b in ((e, g["b3lyp_exc"]), (vr, g["b3lyp_vrho"]), (vs, g["b3lyp_vsigma"])):
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=0)


def test_boys_table_against_scipy(md_host):
    from scipy.special import hyp1f1

    tab = np.zeros(431 * 16)
    md_host.md_boys_table(P(tab))
    ts = np.arange(0.0, 43.05, 0.1)
    tt, mm = np.meshgrid(ts, np.arange(16), indexing="ij")
    ref = hyp1f1(mm + 0.5, mm + 1.5, -tt) / (2 * mm + 1)
    np.testing.assert_allclose(tab.reshape(431, 16), ref, rtol=1e-13, atol=0)
