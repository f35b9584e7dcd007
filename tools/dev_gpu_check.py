"""Developer check on a GPU box: config-1 water, golden synthetic molecules, a timing run."""
import json, os, sys, time, traceback
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01135_b200 import synth, scf, scf_batch, SCFOptions, load_basis, Molecule, properties
from paper_2311_01135_b200.engine import Plan

b = load_basis("sto-3g")
g = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "golden.json")))

def section(name):
    print(f"\n===== {name}", flush=True)

try:
    section("water config-1 f64")
    t = time.time()
    r = scf(synth.water_config1(), b, SCFOptions(max_iterations=20, convergence_std=0.0, grid_level=0))
    print("time", time.time() - t)
    ref = g["cfg1_water"]["f64"]
    print("E", r.E_total, "ref", ref["E_total"], "dE", r.E_total - ref["E_total"])
    print("eps", np.asarray(r.solution.epsilon) - np.asarray(ref["epsilon"]))
    print("hist diff", np.asarray(r.energy_history) - np.asarray(ref["history"]))
    print("comps", {k: r.E_components[k] - ref["components"][k] for k in r.E_components})
except Exception:
    traceback.print_exc()

for prec in ("f64", "f32"):
    try:
        section(f"golden synth {prec}")
        mols, refs = [], []
        for mid, rec in g["synth"].items():
            mols.append(Molecule(tuple(rec["Z"]), np.array(rec["pos"])))
            refs.append(rec[prec])
        t = time.time()
        rs = scf_batch(mols, b, SCFOptions(max_iterations=20, convergence_std=0.0, grid_level=0, precision=prec))
        print("time", time.time() - t)
        for r, ref in zip(rs, refs):
            p = properties(r)
            print(r.n_ao, "dE %.3e  dgap_eV %.3e" % (r.E_total - ref["E_total"], p["gap"] - ref["gap_ev"]))
    except Exception:
        traceback.print_exc()

try:
    section("timing 256 x 9 heavy f32 level0 20 it")
    mols = synth.batch(256, 9, seed=1)
    opts = SCFOptions(max_iterations=20, convergence_std=0.0, grid_level=0, precision="f32")
    import ctypes
    with Plan(mols, b, opts.engine()) as p:
        print(p.info())
        p.set_timing(True)
        for rep in range(3):
            t = time.time()
            p.run()
            res = p.fetch(want_C=False)
            dt = time.time() - t
            print("rep", rep, "wall %.3f s" % dt, "mol/s %.1f" % (256 / dt), "stages ms", p.stage_times(), "launches", p.launch_count())
        print("E sample", res.E_total[:4], "status", np.unique(res.status))
except Exception:
    traceback.print_exc()

try:
    section("pipelined: plans in flight on separate streams, 256 x 9 heavy f32, 12 steps")
    import torch
    opts = SCFOptions(max_iterations=20, convergence_std=0.0, grid_level=0, precision="f32")
    nmax_fl = int(os.environ.get("MAX_INFLIGHT", "4"))
    streams = [torch.cuda.Stream() for _ in range(nmax_fl)]
    plans = [Plan(synth.batch(256, 9, seed=1 + k), b, opts.engine(), stream=s.cuda_stream)
             for k, s in enumerate(streams)]
    for p in plans:
        p.run()
    torch.cuda.synchronize()
    for nfl in range(1, nmax_fl + 1):
        K = 12
        t = time.time()
        for k in range(K):
            plans[k % nfl].run()
        torch.cuda.synchronize()
        dt = time.time() - t
        print("in_flight", nfl, "wall %.3f s" % dt, "mol/s %.1f" % (256 * K / dt))
    # staggered: batch k+1's setup/ERI waits for batch k's setup/ERI, so it overlaps k's SCF loop
    for nfl in range(2, nmax_fl + 1):
        K = 12
        evs = [torch.cuda.Event() for _ in range(nfl)]
        t = time.time()
        for k in range(K):
            s_k, p = streams[k % nfl], plans[k % nfl]
            if k > 0:
                s_k.wait_event(evs[(k - 1) % nfl])
            p.begin()
            evs[k % nfl].record(s_k)
            for it in range(20):
                p.iterate(it)
        torch.cuda.synchronize()
        dt = time.time() - t
        print("staggered in_flight", nfl, "wall %.3f s" % dt, "mol/s %.1f" % (256 * K / dt))
    for p in plans:
        p.close()
    big = Plan(synth.batch(512, 9, seed=11), b, opts.engine())
    big.run(); torch.cuda.synchronize()
    t = time.time()
    for k in range(4):
        big.run()
    torch.cuda.synchronize()
    dt = time.time() - t
    print("single plan 512 mols", "mol/s %.1f" % (512 * 4 / dt))
    big.close()
except Exception:
    traceback.print_exc()
