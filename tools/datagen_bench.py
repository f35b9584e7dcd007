#!/usr/bin/env python
"""BASELINE configs[3]: full data-generation throughput on this GPU's queue.

100,000 seeded synthetic molecules with 9-11 heavy atoms (uniform over 9/10/11, the
configs[1] generator), STO-3G, B3LYP, f32 build, grid level 0, 20 fixed SCF iterations,
labelled through the public batched API (`pipeline.label_batches`: batches of 256, 3 in
flight, host molecules in, host results out).  Under torchrun each rank takes molecules
rank::world (independent per-GPU queues, no collective); rank 0 prints the line.
Molecule generation (host, multiprocessing) is outside the timed region.

    python tools/datagen_bench.py [--mols 100000] [--batch 256] [--workers 3] [--out FILE]
"""
import argparse
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _gen(args):
    idx, seed = args
    from paper_2311_01135_b200 import synth

    out = []
    for k in idx:
        rng = np.random.default_rng((seed, k))
        nh = int(rng.choice([9, 10, 11]))
        out.append(synth.random_molecule(nh, rng, mol_id=f"q{seed}-{k}"))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mols", type=int, default=100_000)
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--workers", type=int, default=3)
    ap.add_argument("--seed", type=int, default=31)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    ws, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    import torch

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    from paper_2311_01135_b200 import SCFOptions, load_basis
    from paper_2311_01135_b200.pipeline import label_batches

    mine = list(range(rank, args.mols, ws))
    t0 = time.perf_counter()
    cores = os.cpu_count() or 1
    step = max(1, len(mine) // (4 * cores) + 1)
    chunks = [(mine[i:i + step], args.seed) for i in range(0, len(mine), step)]
    with Pool(cores) as pool:
        parts = pool.map(_gen, chunks)
    mols = [m for part in parts for m in part]
    gen_s = time.perf_counter() - t0
    b = load_basis("sto-3g")
    opts = SCFOptions(max_iterations=20, convergence_std=0.0, grid_level=0, precision="f32")
    batches = [mols[k:k + args.batch] for k in range(0, len(mols), args.batch)]
    list(label_batches(batches[:args.workers], b, opts, workers=args.workers))   # warm
    torch.cuda.synchronize()
    t = time.perf_counter()
    ok = bad = 0
    e_sum = 0.0
    for _k, res, _w in label_batches(batches, b, opts, workers=args.workers):
        for r in res:
            if isinstance(r, Exception):
                bad += 1
            else:
                ok += 1
                e_sum += float(r.E_total)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    line = {"metric": "SCF molecules/sec (configs[3] data generation)", "rank": rank, "world": ws,
            "molecules": len(mols), "labelled": ok, "failed": bad, "wall_s": wall, "value": ok / wall,
            "unit": "molecules/s (this rank)", "generation_s": gen_s, "batch": args.batch,
            "in_flight": args.workers, "mean_E_total": e_sum / max(ok, 1),
            "config": "100k synthetic molecules, 9-11 heavy (uniform), B3LYP/STO-3G, f32, grid level 0, "
                      "20 fixed iterations, label_batches (host molecules in, host results out)"}
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
        v = torch.tensor([float(ok), wall], device="cuda")
        s = v.clone()
        dist.all_reduce(s[:1], op=dist.ReduceOp.SUM)
        dist.all_reduce(v[1:], op=dist.ReduceOp.MAX)
        line["job_labelled"], line["job_wall_s"] = float(s[0]), float(v[1])
        line["job_value"] = float(s[0]) / float(v[1])
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(line))
        if args.out:
            with open(args.out, "w") as fh:
                json.dump(line, fh, indent=1)


if __name__ == "__main__":
    main()
