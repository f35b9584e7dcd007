"""Pipeline through the device (tests/test_pipeline.py covers the host logic on CPU)."""
import numpy as np
import pytest

from paper_2311_01135_b200 import SCFOptions, load_basis, properties, scf, scf_batch
from paper_2311_01135_b200.constants import HARTREE_TO_EV
from paper_2311_01135_b200.molio import GeometryManifest, ManifestEntry, emit_xyz
from paper_2311_01135_b200.pipeline import label_batches, load_records, records_equal, run

from test_pipeline import FAST, _manifest, _small_molecules

pytestmark = pytest.mark.gpu


def test_records_match_single_molecule_scf(tmp_path, gpu_lib):
    man = _manifest(tmp_path)
    recs = {r.id: r for r in run(man, FAST, 2, str(tmp_path / "r.jsonl"), batch_size=3)}
    b = load_basis("sto-3g")
    for k, m in _small_molecules().items():
        r = scf(m, b, FAST)
        p = properties(r)
        assert recs[k].n_ao == r.n_ao and recs[k].converged == r.converged
        assert recs[k].iterations == r.iterations
        assert recs[k].energy == pytest.approx(r.E_total * HARTREE_TO_EV, abs=1e-7)
        assert recs[k].gap == pytest.approx(p["gap"], abs=1e-7)


def test_determinism_and_resume(tmp_path, gpu_lib):
    man = _manifest(tmp_path)
    a = {r.id: r for r in run(man, FAST, 2, str(tmp_path / "a.jsonl"), batch_size=2)}
    b = {r.id: r for r in run(man, FAST, 1, str(tmp_path / "b.jsonl"), batch_size=2)}
    assert set(a) == set(b)
    for k in a:
        assert records_equal(a[k], b[k])          # same batches -> bitwise identical labels
    part = str(tmp_path / "p.jsonl")
    run(GeometryManifest(entries=man.entries[:2]), FAST, 1, part, batch_size=2)
    resumed = {r.id: r for r in run(man, FAST, 2, part, batch_size=2, resume=True)}
    assert set(resumed) == set(a)
    for k in a:
        assert records_equal(a[k], resumed[k])
    assert len(load_records(part)) == 4


def test_failures_logged_not_fatal(tmp_path, gpu_lib, caplog):
    entries = [ManifestEntry(id="odd", xyz="1\n\nH 0 0 0"), ManifestEntry(id="garbage", xyz="??"),
               ManifestEntry(id="h2", xyz=emit_xyz(_small_molecules()["h2"]))]
    with caplog.at_level("WARNING"):
        recs = run(GeometryManifest(entries=entries), FAST, 2, str(tmp_path / "r.jsonl"))
    assert [r.id for r in recs] == ["h2"]


def test_label_batches_in_flight(gpu_lib):
    from paper_2311_01135_b200 import synth

    b = load_basis("sto-3g")
    opts = SCFOptions(max_iterations=8, convergence_std=0.0, grid_level=0, precision="f32")
    batches = [synth.batch(6, 4, seed=s) for s in range(5)]
    got = {k: res for k, res, _ in label_batches(batches, b, opts, workers=3)}
    assert sorted(got) == list(range(5))
    for k in (0, 4):                                # same labels as a lone batch
        ref = [r.E_total for r in scf_batch(batches[k], b, opts)]
        assert [r.E_total for r in got[k]] == ref


def test_mixed_size_batches_in_flight(gpu_lib):
    """Batches with different AO counts / shell counts in flight at once (different shared-
    memory sizes for the same kernels from several host threads): no batch may fail, and
    every batch's labels equal those of the batch run alone."""
    from paper_2311_01135_b200 import synth

    b = load_basis("sto-3g")
    opts = SCFOptions(max_iterations=6, convergence_std=0.0, grid_level=0, precision="f32")
    heavy = [2, 11, 3, 10, 2, 11, 4, 9, 2, 11]
    batches = [synth.batch(8, h, seed=40 + k) for k, h in enumerate(heavy)]
    got = {k: res for k, res, _ in label_batches(batches, b, opts, workers=4)}
    assert sorted(got) == list(range(len(batches)))
    for k, res in got.items():
        assert not any(isinstance(r, Exception) for r in res), (k, [r for r in res if isinstance(r, Exception)][:1])
    for k in (1, 2):
        ref = [r.E_total for r in scf_batch(batches[k], b, opts)]
        assert [r.E_total for r in got[k]] == ref


def test_scf_batch_device_outputs(gpu_lib):
    """dftb_plan_fetch_device: labels written into caller-owned torch tensors on the current
    stream equal the host results of scf_batch bit for bit."""
    import torch

    from paper_2311_01135_b200 import scf_batch_device, synth

    b = load_basis("sto-3g")
    mols = synth.batch(5, 3, seed=77)
    opts = SCFOptions(max_iterations=8, convergence_std=0.0, grid_level=0, precision="f32")
    ref = scf_batch(mols, b, opts)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        out = scf_batch_device(mols, b, opts, with_orbitals=True)
        e_host = out["E_total"].cpu()          # ordered on the same stream
    s.synchronize()
    assert out["E_total"].is_cuda and out["E_total"].dtype == torch.float64
    for m, r in enumerate(ref):
        assert e_host[m].item() == r.E_total
        n = int(out["iterations"][m])
        assert n == r.iterations
        assert out["history"][m, :n].cpu().tolist() == r.energy_history
        assert torch.isnan(out["history"][m, n:]).all()
        nmo = int(out["n_mo"][m])
        assert out["epsilon"][m, :nmo].cpu().numpy().astype(r.solution.epsilon.dtype).tolist() == \
            r.solution.epsilon.tolist()
        assert int(out["status"][m]) == 0
    out.close()
