#!/usr/bin/env python
"""BASELINE configs[2]: ERI-only microbenchmark on one B200.

4096 seeded synthetic molecules with 10 heavy atoms (the configs[1] generator), STO-3G
fused S/SP shells, every unique shell quartet under 8-fold symmetry, Schwarz 1e-9, in the
f64 build (f64 store) and the f32 build (f32 store, f64 recurrences), plus J/K digestion
against a seeded random symmetric positive-semidefinite density (rho = A A^T / N per
molecule, the reference's PSD test pattern).  Molecules go through the device in plans of
256 (one dense ERI store per plan); times are CUDA events on the plan's stream.

Reports split-shell quartets/s (SURVEY 8(d) unit, counted from the device's own (ij|ij)),
canonical AO integrals/s, algorithmic TFLOP/s against the measured FP64 FMA peak, and
J/K store GB/s against HBM.

    python tools/eri_bench.py [--mols 4096] [--chunk 256] [--out profiles/r1_eri_bench.json]
"""
import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mols", type=int, default=4096)
    ap.add_argument("--chunk", type=int, default=256)
    ap.add_argument("--heavy", type=int, default=10)
    ap.add_argument("--eps", type=float, default=1e-9)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    torch.cuda.init()
    from bench import split_quartet_flops, _hbm_peak
    from paper_2311_01135_b200 import _lib, load_basis, synth
    from paper_2311_01135_b200.engine import EngineOptions, Plan

    b = load_basis("sto-3g")
    lib = _lib.load()
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    peak64 = ctypes.c_double(0.0)
    _lib.check(lib.dftb_fma_peak(1, ctypes.byref(peak64), sp))
    hbm, hbm_src = _hbm_peak()
    out = {"workload": f"configs[2]: {args.mols} molecules x {args.heavy} heavy atoms, STO-3G, Schwarz "
                       f"{args.eps:g}, plans of {args.chunk}", "data": "synthetic (seeded generator)",
           "fp64_peak_tflops": peak64.value, "hbm_peak_gbs": hbm, "hbm_peak_source": hbm_src}
    for prec in ("f64", "f32"):
        tot_ms = jk_ms = 0.0
        nq = flops = n_ints = eri_bytes = 0.0
        nmol = 0
        t_wall = time.perf_counter()
        for c0 in range(0, args.mols, args.chunk):
            n = min(args.chunk, args.mols - c0)
            mols = synth.batch(n, args.heavy, seed=20000 + c0)
            opts = EngineOptions(precision=prec, screen_eps=args.eps, grid_level=None, max_iterations=1)
            with Plan(mols, b, opts, stream=sp) as p:
                p.eri(True)                                   # warm (allocations, caches)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                p.eri(True)
                e1.record(stream)
                torch.cuda.synchronize()
                tot_ms += e0.elapsed_time(e1)
                rng = np.random.default_rng(777 + c0)
                rho = []
                for nao in p.pk.mol_nao:
                    a = rng.standard_normal((int(nao), int(nao)))
                    rho.append((a @ a.T / nao).reshape(-1))
                p.jk(np.concatenate(rho))                      # uploads rho, checks the path
                ms_jk, _ = p.kernel_times(5, xc=False)
                jk_ms += ms_jk
                f, q = split_quartet_flops(mols, p, args.eps)
                flops += f
                nq += q
                nao = np.asarray(p.pk.mol_nao, dtype=np.float64)
                npp = nao * (nao + 1) / 2
                n_ints += float(np.sum(npp * (npp + 1) / 2))
                eri_bytes += p.info()["eri_bytes"]
                nmol += n
        out[prec] = {
            "molecules": nmol, "eri_ms_total": tot_ms, "eri_ms_per_molecule": tot_ms / nmol,
            "split_quartets": nq, "quartets_per_s": nq / (tot_ms / 1e3),
            "ao_integrals_per_s": n_ints / (tot_ms / 1e3),
            "eri_tflops_algorithmic": flops / (tot_ms / 1e3) / 1e12,
            "eri_frac_fp64_peak": flops / (tot_ms / 1e3) / 1e12 / peak64.value,
            "jk_ms_total": jk_ms, "jk_store_gbs": eri_bytes / (jk_ms / 1e3) / 1e9,
            "jk_frac_hbm": eri_bytes / (jk_ms / 1e3) / 1e9 / hbm,
            "store_bytes": eri_bytes, "wall_s": time.perf_counter() - t_wall}
        print(prec, json.dumps(out[prec]), flush=True)
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
