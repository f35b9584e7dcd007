"""f32 operator errors vs the reference's own f32 operators (tests/golden): build_jk over an
f32-stored packed tensor with f32 rho, and xc_matrix from f32 AO values (grid level 0).
Prints max |diff| / max |ref| per molecule (relative to the matrix scale)."""
import json, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2311_01135_b200 import Molecule, expand, load_basis
from paper_2311_01135_b200 import integrals as G_int, xc as G_xc

g = json.load(open(os.path.join(ROOT, "tests/golden/golden.json")))
a = np.load(os.path.join(ROOT, "tests/golden/golden_arrays.npz"))
b = load_basis("sto-3g")
out = {}
cases = [(n, g["small"][n], f"{n}_rho", f"{n}_J32", f"{n}_K32", f"{n}_vxc0_f32", "exc0_f32")
         for n in ("h2", "h2o", "nh3", "ch4", "hf", "dh2o")]
cases.append(("syneri", g["synth_eri"], "syneri_rho", "syneri_J32", "syneri_K32", "syneri_vxc0_32", "exc0_32"))
for name, rec, kr, kj, kk, kv, ke in cases:
    m = Molecule(tuple(rec["Z"]), np.array(rec["pos"]))
    ao = expand(m, b)
    rho32 = a[kr].astype(np.float32)
    J, K = G_int.build_jk(G_int.eri_packed(ao, screen_eps=0.0, dtype=np.float32), rho32)
    gr = G_xc.build_grid(m, 0)
    x = G_xc.xc_matrix(gr, G_xc.eval_ao(ao, gr, dtype=np.float32), rho32)
    rel = lambda u, v: float(np.abs(u.astype(float) - v.astype(float)).max() / np.abs(v).max())
    out[name] = {"J": rel(J, a[kj]), "K": rel(K, a[kk]), "Vxc": rel(x.V_xc, a[kv]),
                 "Exc_abs": abs(x.E_xc - rec[ke]), "Vxc_scale": float(np.abs(a[kv]).max())}
    print(name, ao.n_ao, json.dumps(out[name]))
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
