"""Batch dataset labeling on the device, with JSONL records and checkpoint/resume.

Drop-in for deskdft.pipeline (pkg/src/deskdft/pipeline.py): the record schema
(`RECORD_FIELDS` :28-29, `DatasetRecord` :32-55, energies in eV), `run` (:154-219) with its
resume contract (:163-183: keep one valid line per checkpointed id, drop partial/orphan
lines, rewrite both files atomically), per-entry failures logged and never fatal
(:112-117), `load_records`, `records_equal`, `compare_precision` / `compare_basis`
(:222-265) and `variance_stats` / `variance_to_csv` (:268-296).

What changes is how the work is scheduled.  The reference labels one molecule per task
in a spawn pool of CPU workers (:85-127).  Here the manifest is labeled in device batches
of `batch_size` molecules (one `scf_batch` plan each), and `workers` is the number of
batches in flight on the GPU at once: each in-flight batch is driven by its own host
thread and CUDA stream, so one batch's integral stage overlaps another's SCF loop (plans
never synchronize the host inside a fixed-iteration run).  Records are appended and the
checkpoint rewritten (atomically) after every completed batch; `wall_ms` is the
molecule's share of its batch's wall time.  Multi-GPU: `run(..., devices=[0, 1, ...])`
starts one process per GPU, each labeling its round-robin shard into its own output file,
and merges them (`merge_outputs`); a caller that runs its own ranks passes `rank`/`world`.
No collective is involved.
"""

from __future__ import annotations

import json
import logging
import os
import queue
import threading
import time
from dataclasses import asdict, dataclass

import numpy as np

from .basis import load_basis
from .batch import check
from .constants import HARTREE_TO_EV
from .errors import DeskDFTError
from .molio import GeometryManifest
from .scf import SCFOptions, finish_batch, properties, scf_batch, start_batch

log = logging.getLogger("paper_2311_01135_b200.pipeline")

RECORD_FIELDS = ("id", "smiles", "n_ao", "energy", "homo", "lumo", "gap",
                 "converged", "iterations", "precision", "basis", "wall_ms")


@dataclass(frozen=True)
class DatasetRecord:
    """One labeled conformer; energies in eV."""

    id: str
    smiles: str | None
    n_ao: int
    energy: float
    homo: float
    lumo: float
    gap: float
    converged: bool
    iterations: int
    precision: str
    basis: str
    wall_ms: int

    def to_json(self) -> str:
        return json.dumps(asdict(self))

    @staticmethod
    def from_json(line: str) -> "DatasetRecord":
        d = json.loads(line)
        return DatasetRecord(**{k: d[k] for k in RECORD_FIELDS})


@dataclass(frozen=True)
class ComparisonReport:
    n_molecules: int
    mae_energy_mev: float
    mae_gap_mev: float
    convergence_rate_a: float
    convergence_rate_b: float
    deltas: list

    def to_json(self) -> str:
        return json.dumps(asdict(self), indent=2)


@dataclass(frozen=True)
class VarianceStats:
    per_smiles_std: dict
    hist_edges: list
    hist_counts: list


# ------------------------------------------------------------------ batched device labeling
def label_batches(batches, basis, opts: SCFOptions, workers: int = 3, device: int | None = None):
    """Label a sequence of molecule lists with up to `workers` batches in flight.

    Yields (batch_index, results, wall_s) in completion order; `results[k]` is the
    SCFResult of batch[k] or the exception for that molecule (scf_batch errors="return").
    Each worker thread owns one CUDA stream; a batch's upload, SCF and result copy all
    run on it."""
    import torch

    if workers < 1:
        raise DeskDFTError("workers must be >= 1")
    dev = torch.cuda.current_device() if device is None else int(device)
    todo: queue.Queue = queue.Queue()
    done: queue.Queue = queue.Queue()
    n = 0
    for k, mols in enumerate(batches):
        todo.put((k, mols))
        n += 1
    nthr = min(workers, max(n, 1))
    for _ in range(nthr):
        todo.put(None)

    def worker():
        # one batch queued ahead on this worker's stream: the next batch is packed, planned and
        # enqueued before the current one is waited for, so the host work (packing, plan
        # creation, result objects) never leaves the GPU without this worker's next batch
        torch.cuda.set_device(dev)
        stream = torch.cuda.Stream(device=dev)
        pending = None

        def finish(job):
            k, mols, plan, t0, err = job
            if err is None:
                try:
                    res = finish_batch(plan, opts, errors="return")
                except Exception as exc:       # a failure of the whole batch: every slot gets it
                    res = [exc] * len(mols)
            else:
                res = [err] * len(mols)
            done.put((k, res, time.monotonic() - t0))

        while True:
            item = todo.get()
            if item is None:
                break
            k, mols = item
            t0 = time.monotonic()
            try:
                job = (k, mols, start_batch(mols, basis, opts, stream=stream.cuda_stream), t0, None)
            except Exception as exc:
                job = (k, mols, None, t0, exc)
            if pending is not None:
                finish(pending)
            pending = job
        if pending is not None:
            finish(pending)

    threads = [threading.Thread(target=worker, daemon=True) for _ in range(nthr)]
    for t in threads:
        t.start()
    for _ in range(n):
        yield done.get()
    for t in threads:
        t.join()


# ------------------------------------------------------------------ files
def _atomic_write(path: str, text: str) -> None:
    tmp = path + ".tmp"
    with open(tmp, "w", encoding="utf-8") as fh:
        fh.write(text)
    os.replace(tmp, path)


def _read_checkpoint(path: str) -> set:
    if not os.path.exists(path):
        return set()
    with open(path, encoding="utf-8") as fh:
        return {ln.strip() for ln in fh if ln.strip()}


def load_records(path: str) -> list:
    with open(path, encoding="utf-8") as fh:
        return [DatasetRecord.from_json(ln) for ln in (x.strip() for x in fh) if ln]


def _resume_state(out_path: str, ckpt_path: str, resume: bool) -> tuple[set, list]:
    """The reference's resume rule: one valid line per checkpointed id survives."""
    done, kept = set(), []
    if resume and os.path.exists(out_path):
        ck = _read_checkpoint(ckpt_path)
        with open(out_path, encoding="utf-8") as fh:
            for ln in fh:
                ln = ln.strip()
                if not ln:
                    continue
                try:
                    rec = DatasetRecord.from_json(ln)
                except (json.JSONDecodeError, KeyError, TypeError):
                    continue                    # partial line of a killed run
                if rec.id in ck and rec.id not in done:
                    kept.append(ln)
                    done.add(rec.id)
    _atomic_write(out_path, "".join(x + "\n" for x in kept))
    _atomic_write(ckpt_path, "".join(x + "\n" for x in sorted(done)))
    return done, kept


def _record(entry_id: str, smiles, r, opts: SCFOptions, basis_name: str, wall_ms: int) -> DatasetRecord:
    p = properties(r)
    return DatasetRecord(id=entry_id, smiles=smiles, n_ao=r.n_ao, energy=r.E_total * HARTREE_TO_EV,
                         homo=p["homo"] * HARTREE_TO_EV, lumo=p["lumo"] * HARTREE_TO_EV, gap=p["gap"],
                         converged=r.converged, iterations=r.iterations, precision=opts.precision,
                         basis=basis_name, wall_ms=wall_ms)


def run(manifest: GeometryManifest, opts: SCFOptions, workers: int, out_path: str,
        basis_name: str = "sto-3g", resume: bool = False, *, batch_size: int = 256,
        rank: int = 0, world: int = 1, device: int | None = None, devices=None, _label=None,
        _skip: frozenset = frozenset()) -> list:
    """Label every manifest entry once; append records to out_path as JSONL (pipeline.py:154-219).

    `workers`: device batches in flight per GPU (>= 1).  `devices`: CUDA device indices; with
    more than one, this call labels the whole manifest on all of them - one process per GPU,
    each labeling its round-robin shard into out_path.dev<k>, merged into out_path at the end
    (the reference labels with one call too, pipeline.py:200-213).  `rank`/`world`: for a
    caller that runs the ranks itself, this process labels entries[rank::world].  `_label` is
    a test seam with label_batches' signature."""
    if workers < 1:
        raise DeskDFTError("workers must be >= 1")
    if batch_size < 1:
        raise DeskDFTError("batch_size must be >= 1")
    if devices is not None:
        devices = [int(d) for d in devices]
        if not devices:
            raise DeskDFTError("devices must name at least one device")
        if len(devices) > 1:
            if world != 1 or rank != 0:
                raise DeskDFTError("devices= runs its own ranks: leave rank/world at their defaults")
            return _run_devices(manifest, opts, workers, out_path, basis_name, resume, batch_size,
                                devices, _label)
        device = devices[0]
    ckpt_path = out_path + ".ckpt"
    done, kept = _resume_state(out_path, ckpt_path, resume)
    records = [DatasetRecord.from_json(x) for x in kept]
    todo = [e for e in manifest.entries[rank::world] if e.id not in done and e.id not in _skip]
    if not todo:
        return records
    basis = load_basis(basis_name)
    # parse + validate per entry: failures are logged and skipped, never fatal
    good = []
    for e in todo:
        try:
            good.append((e, manifest.load_molecule(e)))
        except Exception as exc:
            log.warning("entry %s failed: %s: %s", e.id, type(exc).__name__, exc)
    errs = check([m for _, m in good], basis)
    for (e, _), err in zip(good, errs):
        if err is not None:
            log.warning("entry %s failed: %s: %s", e.id, type(err).__name__, err)
    good = [g for g, err in zip(good, errs) if err is None]
    batches = [good[k:k + batch_size] for k in range(0, len(good), batch_size)]
    label = _label or label_batches
    for k, res, wall in label([[m for _, m in b] for b in batches], basis, opts, workers, device):
        lines = []
        wall_ms = int(round(wall * 1000.0 / max(len(res), 1)))
        for (e, m), r in zip(batches[k], res):
            if isinstance(r, Exception):
                log.warning("entry %s failed: %s: %s", e.id, type(r).__name__, r)
                continue
            try:
                rec = _record(m.id or e.id, e.smiles, r, opts, basis_name, wall_ms)
            except Exception as exc:
                log.warning("entry %s failed: %s: %s", e.id, type(exc).__name__, exc)
                continue
            records.append(rec)
            lines.append(rec.to_json())
            done.add(rec.id)
        if lines:
            with open(out_path, "a", encoding="utf-8") as fh:
                fh.write("".join(x + "\n" for x in lines))
        _atomic_write(ckpt_path, "".join(x + "\n" for x in sorted(done)))
    return records


def _device_worker(manifest, opts, workers, path, basis_name, resume, batch_size, rank, world, device,
                   skip, label):
    run(manifest, opts, workers, path, basis_name, resume, batch_size=batch_size, rank=rank, world=world,
        device=device, _label=label, _skip=skip)


def _run_devices(manifest, opts, workers, out_path, basis_name, resume, batch_size, devices, label) -> list:
    """One spawned process per device, shard k = entries[k::G] (no collective: the molecules
    are independent); every shard checkpoints into its own file, so a killed run resumes per
    shard, and the shards are merged into out_path (records already in it first)."""
    import multiprocessing as mp

    done, _ = _resume_state(out_path, out_path + ".ckpt", resume)
    g = len(devices)
    paths = [f"{out_path}.dev{k}" for k in range(g)]
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_device_worker,
                         args=(manifest, opts, workers, paths[k], basis_name, resume, batch_size, k, g,
                               devices[k], frozenset(done), label))
             for k in range(g)]
    for p in procs:
        p.start()
    for p in procs:
        p.join()
    bad = [k for k, p in enumerate(procs) if p.exitcode != 0]
    if bad:
        raise DeskDFTError(f"labeling process(es) for device(s) {[devices[k] for k in bad]} failed "
                           f"(exit codes {[procs[k].exitcode for k in bad]}); completed shards are kept "
                           "for resume=True")
    recs = merge_outputs([out_path] + [p for p in paths if os.path.exists(p)], out_path)
    for p in paths:
        for f in (p, p + ".ckpt"):
            if os.path.exists(f):
                os.remove(f)
    return recs


def merge_outputs(paths: list, out_path: str) -> list:
    """Join per-rank JSONL outputs (first record per id wins) into out_path + checkpoint."""
    seen, lines, recs = set(), [], []
    for p in paths:
        for r in load_records(p):
            if r.id not in seen:
                seen.add(r.id)
                recs.append(r)
                lines.append(r.to_json())
    _atomic_write(out_path, "".join(x + "\n" for x in lines))
    _atomic_write(out_path + ".ckpt", "".join(x + "\n" for x in sorted(seen)))
    return recs


# ------------------------------------------------------------------ analyses
def records_equal(a: DatasetRecord, b: DatasetRecord) -> bool:
    """Physical equality; wall_ms is a measurement, not a label."""
    da, db = asdict(a), asdict(b)
    da.pop("wall_ms")
    db.pop("wall_ms")
    return da == db


def _compare(run_a: list, run_b: list) -> ComparisonReport:
    ia, ib = {r.id: r for r in run_a}, {r.id: r for r in run_b}
    if set(ia) != set(ib):
        raise DeskDFTError(f"id mismatch between runs (a-only {sorted(set(ia) - set(ib))[:5]}, "
                           f"b-only {sorted(set(ib) - set(ia))[:5]})")
    deltas, de, dg = [], [], []
    for k in sorted(ia):
        ra, rb = ia[k], ib[k]
        if not (ra.converged and rb.converged):
            continue
        d_e, d_g = (ra.energy - rb.energy) * 1000.0, (ra.gap - rb.gap) * 1000.0
        deltas.append({"id": k, "d_energy_mev": d_e, "d_gap_mev": d_g})
        de.append(abs(d_e))
        dg.append(abs(d_g))
    if not de:
        raise DeskDFTError("no molecule converged in both runs")
    return ComparisonReport(n_molecules=len(de), mae_energy_mev=float(np.mean(de)),
                            mae_gap_mev=float(np.mean(dg)),
                            convergence_rate_a=sum(r.converged for r in run_a) / len(run_a),
                            convergence_rate_b=sum(r.converged for r in run_b) / len(run_b),
                            deltas=deltas)


def compare_precision(run_a: list, run_b: list) -> ComparisonReport:
    """MAE (meV) between two precisions over molecules converged in both runs."""
    return _compare(run_a, run_b)


def compare_basis(run_a: list, run_b: list) -> ComparisonReport:
    return _compare(run_a, run_b)


def variance_stats(records: list, bins: int = 40) -> VarianceStats:
    """Std of the gap over each SMILES's converged conformers (>= 2 required)."""
    groups: dict = {}
    for r in records:
        if r.smiles and r.converged:
            groups.setdefault(r.smiles, []).append(r.gap)
    stds = {s: float(np.std(g, ddof=1)) for s, g in groups.items() if len(g) >= 2}
    if stds:
        counts, edges = np.histogram(list(stds.values()), bins=bins)
    else:
        counts, edges = np.zeros(bins, dtype=int), np.linspace(0.0, 1.0, bins + 1)
    return VarianceStats(per_smiles_std=stds, hist_edges=[float(e) for e in edges],
                         hist_counts=[int(c) for c in counts])


def variance_to_csv(stats: VarianceStats, path: str) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("smiles,gap_std_ev\n")
        for s, v in sorted(stats.per_smiles_std.items()):
            fh.write(f"{s},{v:.9f}\n")
        fh.write("\nbin_lo,bin_hi,count\n")
        for lo, hi, c in zip(stats.hist_edges[:-1], stats.hist_edges[1:], stats.hist_counts):
            fh.write(f"{lo:.9f},{hi:.9f},{c}\n")
