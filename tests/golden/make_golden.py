"""Generate tests/golden/* by running the REFERENCE implementation (deskdft) in this container.

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/confgen/src:/root/reference/pkg/tests \
    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

/root/reference exists only in the build container, so the fixtures are committed; the
GPU box and the CPU test suite read the files, never the reference.  Inputs are small
fixed molecules (the reference's own test geometries), seeded synthetic molecules from
paper_2311_01135_b200.synth (geometry stored in the fixture, in Bohr), and a subset of
the reference's own cached golden study records (pkg/.acceptance_cache).
"""

from __future__ import annotations

import json
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from deskdft import integrals as R_int  # noqa: E402
from deskdft import xc as R_xc  # noqa: E402
from deskdft.basis import expand as R_expand, load_basis as R_load  # noqa: E402
from deskdft.molio import Molecule as R_Molecule, parse_xyz as R_parse  # noqa: E402
from deskdft.scf import SCFOptions, diis_step as R_diis, properties as R_props  # noqa: E402
from deskdft.scf import scf as R_scf, solve_roothaan as R_roothaan  # noqa: E402

SMALL_XYZ = {  # reference test geometries (pkg/tests/suites.py:53-64, test_integrals.py:19)
    "h2": "2\nid=h2\nH 0.0 0.0 0.0\nH 0.0 0.0 0.7408481\n",
    "h2o": "3\nid=h2o\nO 0.0 0.0 0.1173\nH 0.0 0.7572 -0.4692\nH 0.0 -0.7572 -0.4692\n",
    "nh3": ("4\nid=nh3\nN 0.0 0.0 0.1173\nH 0.0 0.9377 -0.2737\n"
            "H 0.8121 -0.4689 -0.2737\nH -0.8121 -0.4689 -0.2737\n"),
    "ch4": ("5\nid=ch4\nC 0.0 0.0 0.0\nH 0.6276 0.6276 0.6276\n"
            "H -0.6276 -0.6276 0.6276\nH -0.6276 0.6276 -0.6276\n"
            "H 0.6276 -0.6276 -0.6276\n"),
    "hf": "2\nid=hf\nF 0.0 0.0 0.0\nH 0.0 0.0 0.9168\n",
    "dh2o": "3\n\nO 0.05 -0.1 0.1173\nH 0.02 0.7572 -0.4692\nH 0.0 -0.7572 -0.4892",
}
WATER_CFG1 = np.array([[0.0, 0.0, 0.0], [1.4302354483800725, 1.1074066044277557, 0.0],
                       [-1.4302354483800725, 1.1074066044277557, 0.0]])


def _scf_record(m, opts):
    r = R_scf(m, R_load("sto-3g"), opts)
    p = R_props(r)
    return {"E_total": r.E_total, "epsilon": r.solution.epsilon.astype(float).tolist(),
            "n_occ": r.solution.n_occ, "components": r.E_components,
            "history": [float(x) for x in r.energy_history], "converged": r.converged,
            "iterations": r.iterations, "n_ao": r.n_ao, "homo": p["homo"], "lumo": p["lumo"],
            "gap_ev": p["gap"]}


def _job(args):
    Z, pos, kw = args
    return _scf_record(R_Molecule(tuple(Z), np.asarray(pos)), SCFOptions(**kw))


def small_fixtures(b):
    out_json, arrs = {}, {}
    rng = np.random.default_rng(1234)
    for name, xyz in SMALL_XYZ.items():
        m = R_parse(xyz)
        ao = R_expand(m, b)
        n = ao.n_ao
        rec = {"Z": list(m.atomic_numbers), "pos": m.positions.tolist(), "n_ao": n}
        ints = R_int.one_electron(ao, m)
        for k in ("S", "T", "V"):
            arrs[f"{name}_{k}"] = getattr(ints, k)
        arrs[f"{name}_prim_coef"] = ao.prim_coef
        for eps in (0.0, 1e-9):
            e = R_int.eri_packed(ao, screen_eps=eps)
            tag = "eri0" if eps == 0.0 else "eri9"
            arrs[f"{name}_{tag}_ijkl"] = np.stack([e.i, e.j, e.k, e.l]).astype(np.int32)
            arrs[f"{name}_{tag}_v"] = e.values
            arrs[f"{name}_{tag}_deg"] = e.degeneracy.astype(np.int32)
        pairs = R_int._PairTables(ao)
        qp, qa = pairs.schwarz()
        arrs[f"{name}_q_ao"] = qa
        a = rng.standard_normal((n, n))
        rho = a @ a.T / n
        arrs[f"{name}_rho"] = rho
        J, K = R_int.build_jk(R_int.eri_packed(ao, screen_eps=0.0), rho)
        arrs[f"{name}_J"] = J
        arrs[f"{name}_K"] = K
        for lvl in (0, 1):
            g = R_xc.build_grid(m, level=lvl)
            rec[f"npts{lvl}"] = g.n_points
            if name in ("h2o", "dh2o", "ch4"):
                arrs[f"{name}_grid{lvl}_pts"] = g.points
                arrs[f"{name}_grid{lvl}_w"] = g.weights
            aov = R_xc.eval_ao(ao, g)
            x = R_xc.xc_matrix(g, aov, rho)
            rec[f"exc{lvl}"] = x.E_xc
            arrs[f"{name}_vxc{lvl}"] = x.V_xc
            if name == "dh2o" and lvl == 0:
                arrs["dh2o_phi0"] = aov.phi
                arrs["dh2o_gphi0"] = aov.grad_phi
        # f32 operators (the reference's f32 working dtype): f32-stored ERIs
        # and f32 rho through build_jk; f32 AO values and rho through xc_matrix at level 0
        rho32 = rho.astype(np.float32)
        J32, K32 = R_int.build_jk(R_int.eri_packed(ao, screen_eps=0.0, dtype=np.float32), rho32)
        arrs[f"{name}_J32"] = J32
        arrs[f"{name}_K32"] = K32
        g0 = R_xc.build_grid(m, level=0)
        x32 = R_xc.xc_matrix(g0, R_xc.eval_ao(ao, g0, dtype=np.float32), rho32)
        rec["exc0_f32"] = x32.E_xc
        arrs[f"{name}_vxc0_f32"] = x32.V_xc
        sol = R_roothaan(ints.V + ints.T, ints.S)
        arrs[f"{name}_core_eps"] = sol.epsilon
        out_json[name] = rec
    return out_json, arrs


def b3lyp_fixture():
    rng = np.random.default_rng(7)
    n = 10.0 ** rng.uniform(-10, 3, 1000)
    s = 10.0 ** rng.uniform(-12, 4, 1000)
    n[:5] = [0.0, 1e-13, 5e-13, 1e-12, 2e-12]
    exc, vr, vs = R_xc.b3lyp(n, s)
    return {"b3lyp_n": n, "b3lyp_s": s, "b3lyp_exc": exc, "b3lyp_vrho": vr, "b3lyp_vsigma": vs}


def diis_fixture():
    rng = np.random.default_rng(99)
    arrs = {}
    for case in range(6):
        m = 2 + case
        n = 6
        F = rng.standard_normal((m, n, n))
        F = F + F.transpose(0, 2, 1)
        E = rng.standard_normal((m, n, n)) * (0.3 ** np.arange(m))[:, None, None]
        if case == 0:  # identical errors -> singular B -> damped fallback
            E[:] = E[0]
        hist = [(F[a], E[a]) for a in range(m)]
        arrs[f"diis{case}_F"] = F
        arrs[f"diis{case}_E"] = E
        arrs[f"diis{case}_out"] = R_diis(hist)
    return arrs


def synth_fixtures(pool):
    from paper_2311_01135_b200 import synth
    mols = synth.batch(4, 9, seed=11) + synth.batch(2, 10, seed=12) + synth.batch(2, 11, seed=13)
    jobs, meta = [], []
    for m in mols:
        for prec in ("f64", "f32"):
            kw = dict(max_iterations=20, convergence_std=0.0, grid_level=0, precision=prec)
            jobs.append((m.atomic_numbers, m.positions.tolist(), kw))
            meta.append((m.id, prec))
    # screen 1e-9 variant for one molecule (config-3 threshold)
    kw = dict(max_iterations=20, convergence_std=0.0, grid_level=0, precision="f64", screen_eps=1e-9)
    jobs.append((mols[0].atomic_numbers, mols[0].positions.tolist(), kw))
    meta.append((mols[0].id, "f64_s9"))
    res = list(pool.map(_job, jobs))
    out = {}
    for (mid, prec), r, (Z, pos, kw) in zip(meta, res, jobs):
        out.setdefault(mid, {"Z": list(Z), "pos": pos})[prec] = r
    return out


def synth_eri_fixture(b):
    """Size-independent ERI properties for one 10-heavy synthetic molecule: count and
    checksums of the eps=1e-9 kept set, plus a seeded sample of exact (eps=0) values."""
    from paper_2311_01135_b200 import synth
    m = synth.batch(1, 10, seed=21)[0]
    rm = R_Molecule(m.atomic_numbers, m.positions)
    ao = R_expand(rm, b)
    e9 = R_int.eri_packed(ao, screen_eps=1e-9)
    e0 = R_int.eri_packed(ao, screen_eps=0.0)
    rng = np.random.default_rng(5)
    pick = np.sort(rng.choice(e0.n_entries, 20000, replace=False))
    rec = {"Z": list(m.atomic_numbers), "pos": m.positions.tolist(), "n_ao": ao.n_ao,
           "count9": e9.n_entries, "sum9": float(e9.values.sum()),
           "sumsq9": float((e9.values.astype(float) ** 2).sum()),
           "count0": e0.n_entries, "sum0": float(e0.values.sum()),
           "sumsq0": float((e0.values.astype(float) ** 2).sum())}
    n = ao.n_ao
    a = np.random.default_rng(3).standard_normal((n, n))
    rho = a @ a.T / n
    J, K = R_int.build_jk(e0, rho)
    arrs = {"syneri_ijkl": np.stack([e0.i[pick], e0.j[pick], e0.k[pick], e0.l[pick]]).astype(np.int32),
            "syneri_v": e0.values[pick], "syneri_rho": rho, "syneri_J": J, "syneri_K": K}
    # the f32 operators at full molecule size: J/K over the f32 store, V_xc from f32 AO values
    rho32 = rho.astype(np.float32)
    J32, K32 = R_int.build_jk(R_int.eri_packed(ao, screen_eps=0.0, dtype=np.float32), rho32)
    arrs["syneri_J32"], arrs["syneri_K32"] = J32, K32
    g0 = R_xc.build_grid(rm, level=0)
    for tag, dt in (("64", np.float64), ("32", np.float32)):
        x = R_xc.xc_matrix(g0, R_xc.eval_ao(ao, g0, dtype=dt), rho.astype(dt))
        rec[f"exc0_{tag}"] = x.E_xc
        arrs[f"syneri_vxc0_{tag}"] = x.V_xc
    return rec, arrs


def dump_fixtures(b):
    """Binary dumps written by the reference (integrals.py:248-291): the packed ERIs of the
    distorted water in f64 and f32, and its S/T/V set -> tests/golden/dumps/*.bin."""
    d = os.path.join(HERE, "dumps")
    os.makedirs(d, exist_ok=True)
    m = R_parse(SMALL_XYZ["dh2o"])
    ao = R_expand(m, b)
    R_int.dump_packed(R_int.eri_packed(ao), os.path.join(d, "dh2o_eri_f64.bin"))
    R_int.dump_packed(R_int.eri_packed(ao, dtype=np.float32), os.path.join(d, "dh2o_eri_f32.bin"))
    R_int.dump_integral_set(R_int.one_electron(ao, m), os.path.join(d, "dh2o_stv.bin"))


def study_records(k=48):
    base = "/root/reference/pkg/.acceptance_cache"
    recs = [json.loads(x) for x in open(os.path.join(base, "study-f64-8f4bf9381a67.jsonl"))]
    recs = sorted(recs, key=lambda r: r["id"])[::max(1, len(recs) // k)][:k]
    for r in recs:
        with open(os.path.join(base, "suite_study", r["id"] + ".xyz")) as fh:
            r["xyz"] = fh.read()
        r.pop("wall_ms", None)
    return recs


def main():
    b = R_load("sto-3g")
    out = {}
    import multiprocessing as mp
    with ProcessPoolExecutor(8, mp_context=mp.get_context("spawn")) as pool:
        cfg1 = {}
        for prec in ("f64", "f32"):
            cfg1[prec] = _scf_record(R_Molecule((8, 1, 1), WATER_CFG1),
                                     SCFOptions(max_iterations=20, convergence_std=0.0,
                                                grid_level=0, precision=prec))
        out["cfg1_water"] = {"Z": [8, 1, 1], "pos": WATER_CFG1.tolist(), **cfg1}
        small, arrs = small_fixtures(b)
        out["small"] = small
        # converged SCF records for the small molecules (f64, level 1, conv 1e-6)
        for name in ("h2o", "nh3", "ch4", "hf"):
            rm = R_parse(SMALL_XYZ[name])
            small[name]["scf_l1"] = _scf_record(rm, SCFOptions(convergence_std=1e-6))
        h2 = R_parse("2\n\nH 0 0 0\nH 0 0 1.4", unit="bohr")
        out["h2_l3"] = {"Z": [1, 1], "pos": h2.positions.tolist(),
                        **_scf_record(h2, SCFOptions(convergence_std=1e-8, grid_level=3,
                                                     max_iterations=60))}
        arrs.update(b3lyp_fixture())
        arrs.update(diis_fixture())
        out["synth"] = synth_fixtures(pool)
        rec, a2 = synth_eri_fixture(b)
        out["synth_eri"] = rec
        arrs.update(a2)
    dump_fixtures(b)
    out["study"] = study_records()
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    np.savez_compressed(os.path.join(HERE, "golden_arrays.npz"), **arrs)
    print("wrote", sorted(out), len(arrs), "arrays")


if __name__ == "__main__":
    main()
