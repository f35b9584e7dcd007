"""f32 build_jk error vs the f64-accumulated reference formula for different J/K CTA splits (GPU box).
usage: QM1B_JK_SPLIT=k python tools/jkerr.py"""
import os, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01135_b200 import synth, load_basis, expand, integrals
m = synth.batch(1, 9, seed=1000)[0]
ao = expand(m, load_basis("sto-3g"))
eri = integrals.eri_packed(ao, screen_eps=0.0, dtype=np.float32)
rng = np.random.default_rng(3)
n = ao.n_ao
A = rng.standard_normal((n, n)); rho = (A @ A.T / n).astype(np.float32)
J, K = integrals.build_jk(eri, rho.astype(np.float64))   # f64-typed rho: the outputs are not rounded to f32
# f64 reference from the dense tensor
D = integrals.unpack_eri(eri).astype(np.float64)
r64 = rho.astype(np.float64)
Jr = np.einsum("ijkl,kl->ij", D, r64); Kr = -0.5 * np.einsum("ikjl,kl->ij", D, r64)
print(json.dumps({"split": os.environ.get("QM1B_JK_SPLIT"), "n": n, "J": float(np.abs(J - Jr).max() / np.abs(Jr).max()), "K": float(np.abs(K - Kr).max() / np.abs(Kr).max())}))
