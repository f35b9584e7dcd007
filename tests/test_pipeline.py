"""Pipeline host logic (records, checkpoint/resume, sharding, analyses) on CPU.

Mirrors the reference's pipeline tests (pkg/tests/test_pipeline.py): schema round trip,
per-entry failures logged and not fatal, resume identity, orphan lines dropped,
determinism, comparison/variance reports.  The device labeler is replaced through the
`_label` test seam by the CPU oracle (test infrastructure only), so this file needs no GPU;
tests/test_pipeline_gpu.py runs the same flows through the device.
"""
import json
import os

import numpy as np
import pytest

from paper_2311_01135_b200 import SCFOptions
from paper_2311_01135_b200.errors import DeskDFTError
from paper_2311_01135_b200.molio import (GeometryManifest, ManifestEntry, Molecule, emit_xyz,
                                         load_manifest, save_manifest)
from paper_2311_01135_b200.pipeline import (DatasetRecord, compare_basis, compare_precision, load_records,
                                            merge_outputs, records_equal, run, variance_stats,
                                            variance_to_csv)
from paper_2311_01135_b200.scf import OrbitalSolution, SCFResult

FAST = SCFOptions(convergence_std=1e-4, grid_level=0, max_iterations=30)

A = 1.8897259886  # Angstrom -> Bohr


def _small_molecules():
    """Own small closed-shell geometries (Bohr)."""
    h2 = Molecule((1, 1), np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 0.74 * A]]))
    hf = Molecule((9, 1), np.array([[0.0, 0.0, 0.0], [0.0, 0.0, 0.92 * A]]))
    d = 1.09 * A / np.sqrt(3.0)
    ch4 = Molecule((6, 1, 1, 1, 1), np.array([[0, 0, 0], [d, d, d], [-d, -d, d], [-d, d, -d], [d, -d, -d]],
                                             dtype=float))
    from paper_2311_01135_b200 import synth

    return {"h2": h2, "water": synth.water_config1(), "hf": hf, "ch4": ch4}


def _manifest(tmp_path, n=4):
    mols = list(_small_molecules().items())[:n]
    smiles = {"h2": "[HH]", "water": "O", "hf": "F", "ch4": "C"}
    return GeometryManifest(entries=[ManifestEntry(id=k, xyz=emit_xyz(m), smiles=smiles[k]) for k, m in mols],
                            base_dir=str(tmp_path))


@pytest.fixture
def oracle_label(oracle):
    """label_batches stand-in on the CPU oracle: same yield protocol as the device path."""
    calls = []

    def label(batches, basis, opts, workers, device):
        calls.append((len(batches), workers))
        for k, mols in enumerate(batches):
            out = []
            for m in mols:
                r = oracle.scf(oracle.Mol(tuple(m.atomic_numbers), np.asarray(m.positions)), opts.precision,
                               opts.max_iterations, opts.convergence_std, opts.grid_level)
                out.append(SCFResult(solution=OrbitalSolution(C=r.C, epsilon=r.epsilon, n_occ=r.n_occ),
                                     E_total=r.E_total, E_components=r.components,
                                     energy_history=list(r.history), converged=r.converged,
                                     iterations=r.iterations, n_ao=r.n_ao))
            yield k, out, 0.004 * len(mols)

    label.calls = calls
    return label


def test_empty_manifest(tmp_path, oracle_label):
    out = str(tmp_path / "r.jsonl")
    assert run(GeometryManifest(entries=[]), FAST, 1, out, _label=oracle_label) == []
    assert open(out).read() == ""
    assert open(out + ".ckpt").read() == ""


def test_bad_arguments(tmp_path):
    with pytest.raises(DeskDFTError):
        run(GeometryManifest(entries=[]), FAST, 0, str(tmp_path / "r.jsonl"))
    with pytest.raises(DeskDFTError):
        run(GeometryManifest(entries=[]), FAST, 1, str(tmp_path / "r.jsonl"), batch_size=0)


def test_run_and_schema_roundtrip(tmp_path, oracle_label):
    out = str(tmp_path / "r.jsonl")
    recs = run(_manifest(tmp_path), FAST, 2, out, batch_size=3, _label=oracle_label)
    assert oracle_label.calls == [(2, 2)]          # 4 molecules in batches of 3, 2 in flight
    assert {r.id for r in recs} == {"h2", "water", "hf", "ch4"}
    loaded = load_records(out)
    assert len(loaded) == 4
    for r in loaded:
        assert r.gap == pytest.approx(r.lumo - r.homo, abs=1e-9)
        assert (r.basis, r.precision) == ("sto-3g", "f64")
        assert r.converged
        assert records_equal(DatasetRecord.from_json(r.to_json()), r)
        assert set(json.loads(r.to_json())) == set(DatasetRecord.__dataclass_fields__)
    assert sorted(open(out + ".ckpt").read().split()) == sorted(r.id for r in recs)


def test_failures_logged_not_fatal(tmp_path, oracle_label, caplog):
    entries = [ManifestEntry(id="odd", xyz="1\n\nH 0 0 0"),          # odd electron count
               ManifestEntry(id="garbage", xyz="not xyz at all"),
               ManifestEntry(id="na", xyz="2\n\nNa 0 0 0\nH 0 0 1.9"),  # no STO-3G data on the device path
               ManifestEntry(id="h2", xyz=emit_xyz(_small_molecules()["h2"]))]
    out = str(tmp_path / "r.jsonl")
    with caplog.at_level("WARNING"):
        recs = run(GeometryManifest(entries=entries), FAST, 1, out, _label=oracle_label)
    assert [r.id for r in recs] == ["h2"]
    for bad in ("odd", "garbage", "na"):
        assert any(bad in m for m in caplog.messages)


def test_resume_identity(tmp_path, oracle_label):
    man = _manifest(tmp_path)
    full = {r.id: r for r in run(man, FAST, 1, str(tmp_path / "full.jsonl"), _label=oracle_label)}
    part = str(tmp_path / "part.jsonl")
    run(GeometryManifest(entries=man.entries[:2]), FAST, 1, part, _label=oracle_label)
    resumed = {r.id: r for r in run(man, FAST, 1, part, resume=True, _label=oracle_label)}
    assert set(resumed) == set(full)
    for k in full:
        assert records_equal(full[k], resumed[k])
    assert len(load_records(part)) == 4


def test_resume_drops_orphan_lines(tmp_path, oracle_label):
    man = _manifest(tmp_path, n=2)
    out = str(tmp_path / "r.jsonl")
    run(GeometryManifest(entries=man.entries[:1]), FAST, 1, out, _label=oracle_label)
    with open(out, "a") as fh:
        fh.write('{"id": "water", "truncated...')            # killed mid-write
    resumed = run(man, FAST, 1, out, resume=True, _label=oracle_label)
    assert {r.id for r in load_records(out)} == {"h2", "water"}
    assert len(load_records(out)) == 2
    assert {r.id for r in resumed} == {"h2", "water"}


def test_resume_without_checkpointed_lines_relabels(tmp_path, oracle_label):
    man = _manifest(tmp_path, n=2)
    out = str(tmp_path / "r.jsonl")
    run(man, FAST, 1, out, _label=oracle_label)
    os.remove(out + ".ckpt")                                 # records present, checkpoint lost
    recs = run(man, FAST, 1, out, resume=True, _label=oracle_label)
    assert {r.id for r in recs} == {"h2", "water"}
    assert len(load_records(out)) == 2


def test_sharding_and_merge(tmp_path, oracle_label):
    man = _manifest(tmp_path)
    outs = []
    for rank in range(2):
        o = str(tmp_path / f"r{rank}.jsonl")
        recs = run(man, FAST, 1, o, rank=rank, world=2, _label=oracle_label)
        assert [r.id for r in recs] == [e.id for e in man.entries[rank::2]]
        outs.append(o)
    merged = merge_outputs(outs, str(tmp_path / "all.jsonl"))
    assert {r.id for r in merged} == {e.id for e in man.entries}


def test_manifest_file_roundtrip(tmp_path):
    man = _manifest(tmp_path)
    p = str(tmp_path / "m.jsonl")
    save_manifest(man, p)
    back = load_manifest(p)
    assert [e.id for e in back.entries] == [e.id for e in man.entries]
    m0 = back.load_molecule(back.entries[1])
    assert m0.id == "water" and m0.smiles == "O"
    with pytest.raises(Exception, match="duplicate"):
        GeometryManifest(entries=[ManifestEntry(id="a", xyz="x"), ManifestEntry(id="a", xyz="y")])


def _mk(id, e, gap, conv=True, smiles=None):
    return DatasetRecord(id=id, smiles=smiles, n_ao=7, energy=e, homo=-1.0, lumo=-1.0 + gap, gap=gap,
                         converged=conv, iterations=9, precision="f32", basis="sto-3g", wall_ms=1)


def test_compare_reports():
    a = [_mk("a", -2000.0, 10.0), _mk("b", -2100.0, 9.0)]
    assert compare_precision(a, a).mae_energy_mev == 0.0
    b = [_mk("a", -2000.002, 10.001), _mk("b", -2100.004, 8.999)]
    rep = compare_precision(a, b)
    assert rep.mae_energy_mev == pytest.approx(3.0, rel=1e-6)
    assert rep.mae_gap_mev == pytest.approx(1.0, rel=1e-6)
    c = [_mk("a", -2000.1, 10.0), _mk("b", -2100.0, 9.0, conv=False)]
    rep = compare_basis(c, b)
    assert rep.n_molecules == 1 and rep.convergence_rate_a == 0.5
    with pytest.raises(DeskDFTError, match="id mismatch"):
        compare_precision([_mk("a", 0, 1)], [_mk("b", 0, 1)])
    with pytest.raises(DeskDFTError, match="no molecule converged"):
        compare_precision([_mk("a", 0, 1, conv=False)], [_mk("a", 0, 1)])


def test_variance_stats(tmp_path):
    recs = [_mk("a1", 0, 10.0, smiles="C"), _mk("a2", 0, 10.2, smiles="C"), _mk("b1", 0, 9.0, smiles="O"),
            _mk("c1", 0, 8.0, smiles="N", conv=False), _mk("c2", 0, 8.5, smiles="N")]
    st = variance_stats(recs, bins=4)
    assert set(st.per_smiles_std) == {"C"}
    assert st.per_smiles_std["C"] == pytest.approx(np.std([10.0, 10.2], ddof=1))
    assert sum(st.hist_counts) == 1 and len(st.hist_edges) == 5
    p = str(tmp_path / "v.csv")
    variance_to_csv(st, p)
    assert open(p).read().startswith("smiles,gap_std_ev\nC,")
    empty = variance_stats([], bins=3)
    assert empty.per_smiles_std == {} and empty.hist_counts == [0, 0, 0]


def test_run_on_several_devices_merges_shards(tmp_path, monkeypatch):
    """run(devices=[0, 1]): one spawned process per device labels entries[k::2] into its own
    file; the merged output holds every entry once and equals a single-process run."""
    from helpers.cpu_label import oracle_label

    man = _manifest(tmp_path)
    log = tmp_path / "devices.log"
    monkeypatch.setenv("QM1B_TEST_DEVICE_LOG", str(log))
    out2 = str(tmp_path / "two.jsonl")
    recs2 = run(man, FAST, 1, out2, devices=[0, 1], batch_size=1, _label=oracle_label)
    out1 = str(tmp_path / "one.jsonl")
    recs1 = run(man, FAST, 1, out1, batch_size=1, _label=oracle_label)
    a = {r.id: r for r in recs2}
    b = {r.id: r for r in recs1}
    assert set(a) == set(b) == {e.id for e in man.entries}
    assert all(records_equal(a[k], b[k]) for k in a)
    assert {r.id for r in load_records(out2)} == set(a)
    assert sorted(open(out2 + ".ckpt").read().split()) == sorted(a)
    assert not any(p.name.startswith("two.jsonl.dev") for p in tmp_path.iterdir())   # shards merged away
    seen = [ln.split() for ln in log.read_text().splitlines()]
    by_dev = {d: {i for dd, i in seen if dd == d} for d, _ in seen}
    ids = [e.id for e in man.entries]
    assert by_dev["0"] >= set(ids[0::2]) and by_dev["1"] >= set(ids[1::2])


def test_run_on_several_devices_failure_keeps_shards(tmp_path):
    from helpers.cpu_label import failing_label, oracle_label

    man = _manifest(tmp_path)
    out = str(tmp_path / "r.jsonl")
    with pytest.raises(DeskDFTError, match="device"):
        run(man, FAST, 1, out, devices=[0, 1], batch_size=1, _label=failing_label)
    assert os.path.exists(out + ".dev0")                 # the healthy shard is kept for resume
    recs = run(man, FAST, 1, out, devices=[0, 1], batch_size=1, resume=True, _label=oracle_label)
    assert {r.id for r in recs} == {e.id for e in man.entries}
