"""Binary dump formats (reference integrals.py:248-291; its test test_integrals.py:249-264):
the packed-ERI dump and the S/T/V integral-set dump.  tests/golden/dumps/*.bin were written
by the REFERENCE itself (tests/golden/make_golden.py::dump_fixtures) for the distorted water
molecule: eri_packed(ao) in f64 and f32 and one_electron(ao, m).

CPU tests: our loaders read the reference's files, and our writers reproduce them byte for
byte.  GPU test: the device's own eri_packed / one_electron of the same molecule, dumped by
our writer, match the reference's files (indices and header byte-identical, values to the
f64 / f32 parity bar)."""
import os

import numpy as np
import pytest

from paper_2311_01135_b200 import expand, load_basis, parse_xyz
from paper_2311_01135_b200 import integrals as G_int

DUMPS = os.path.join(os.path.dirname(__file__), "golden", "dumps")
DH2O = "3\n\nO 0.05 -0.1 0.1173\nH 0.02 0.7572 -0.4692\nH 0.0 -0.7572 -0.4892"


def _bytes(path):
    with open(path, "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("tag,itemsize", [("f64", 8), ("f32", 4)])
def test_reference_eri_dump_roundtrip(tmp_path, tag, itemsize):
    path = os.path.join(DUMPS, f"dh2o_eri_{tag}.bin")
    e = G_int.load_packed(path)
    assert e.n_ao == 7 and e.values.dtype.itemsize == itemsize
    q = e.quads.astype(np.int64)
    i, j, k, l = q.T
    assert (i >= j).all() and (k >= l).all()
    P, Q = i * (i + 1) // 2 + j, k * (k + 1) // 2 + l
    assert (P >= Q).all()
    assert (np.diff(P * (P + 1) // 2 + Q) > 0).all()          # composite order, no duplicates
    deg = np.where(i != j, 2, 1) * np.where(k != l, 2, 1) * np.where(P != Q, 2, 1)
    assert np.array_equal(e.degeneracy.astype(np.int64), deg)
    out = str(tmp_path / "eri.bin")
    G_int.dump_packed(e, out)
    assert _bytes(out) == _bytes(path)
    back = G_int.load_packed(out)
    assert np.array_equal(back.values, e.values) and np.array_equal(back.quads, e.quads)


def test_reference_integral_set_dump_roundtrip(tmp_path, golden_arrays):
    path = os.path.join(DUMPS, "dh2o_stv.bin")
    s = G_int.load_integral_set(path)
    assert s.n_ao == 7
    for k in ("S", "T", "V"):      # the reference's one_electron values, bit for bit
        assert np.array_equal(getattr(s, k), golden_arrays[f"dh2o_{k}"])
    out = str(tmp_path / "stv.bin")
    G_int.dump_integral_set(s, out)
    assert _bytes(out) == _bytes(path)


def test_dump_rejects_foreign_files(tmp_path):
    bad = tmp_path / "x.bin"
    bad.write_bytes(b"\0" * 64)
    with pytest.raises(ValueError):
        G_int.load_packed(str(bad))
    with pytest.raises(ValueError):
        G_int.load_integral_set(str(bad))
    with pytest.raises(ValueError):   # an integral-set file is not an ERI dump and vice versa
        G_int.load_packed(os.path.join(DUMPS, "dh2o_stv.bin"))


@pytest.mark.gpu
def test_device_dumps_match_reference_files(gpu_lib, tmp_path):
    b = load_basis("sto-3g")
    m = parse_xyz(DH2O)
    ao = expand(m, b)
    for tag, dt in (("f64", np.float64), ("f32", np.float32)):
        ref = G_int.load_packed(os.path.join(DUMPS, f"dh2o_eri_{tag}.bin"))
        mine = G_int.eri_packed(ao, dtype=dt)
        out = str(tmp_path / f"eri_{tag}.bin")
        G_int.dump_packed(mine, out)
        got = _bytes(out)
        want = _bytes(os.path.join(DUMPS, f"dh2o_eri_{tag}.bin"))
        n = ref.n_entries
        assert len(got) == len(want) and got[:17 + 8 * n] == want[:17 + 8 * n]   # header + indices
        back = G_int.load_packed(out)
        if dt == np.float64:
            assert np.abs(back.values - ref.values).max() < 1e-13
        else:
            # the device rounds the f64 integral to f32 once: at most one ulp from the
            # reference's f64 value rounded to f32 (the two f64 values agree to ~1e-13) ...
            r64 = G_int.load_packed(os.path.join(DUMPS, "dh2o_eri_f64.bin")).values.astype(np.float32)
            a, r = back.values.view(np.int32), r64.view(np.int32)
            assert np.abs(a.astype(np.int64) - r.astype(np.int64)).max() <= 1
            # ... while the reference's own f32 values accumulate the primitive contraction in
            # f32 (_kernels.py:553, block dtype = out dtype): a few ulp, its own bound 1e-5
            # (test_integrals.py:241-246)
            d = np.abs(back.values.astype(np.float64) - ref.values.astype(np.float64))
            assert (d / np.maximum(np.abs(ref.values.astype(np.float64)), 1.0)).max() < 1e-6
    ints = G_int.one_electron(ao, m)
    out = str(tmp_path / "stv.bin")
    G_int.dump_integral_set(ints, out)
    got, want = _bytes(out), _bytes(os.path.join(DUMPS, "dh2o_stv.bin"))
    assert got[:8] == want[:8]
    back = G_int.load_integral_set(out)
    ref = G_int.load_integral_set(os.path.join(DUMPS, "dh2o_stv.bin"))
    for k in ("S", "T", "V"):
        np.testing.assert_allclose(getattr(back, k), getattr(ref, k), rtol=0, atol=1e-12)
