"""Mixed-size batch (1..13 heavy atoms, every AO-count bucket in one plan): f32 build vs f64 build labels."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2311_01135_b200 import synth, SCFOptions, load_basis, scf_batch, properties
rng = np.random.default_rng(7)
mols = [synth.random_molecule(int(h), rng) for h in rng.integers(1, 14, size=96)]
b = load_basis("sto-3g")
o = dict(max_iterations=20, convergence_std=0.0, grid_level=0)
r32 = scf_batch(mols, b, SCFOptions(precision="f32", **o))
r64 = scf_batch(mols, b, SCFOptions(precision="f64", **o))
dE = np.array([a.E_total - c.E_total for a, c in zip(r32, r64)])
dg = np.array([properties(a)["gap"] - properties(c)["gap"] for a, c in zip(r32, r64)])
nao = np.array([a.n_ao for a in r32])
std5 = np.array([np.std(c.energy_history[-5:]) for c in r64])
ok = std5 < 1e-5
print("n_ao range", nao.min(), nao.max(), "settled", int(ok.sum()), "of", len(mols))
print("settled: |dE| max %.3g mean %.3g Ha, |dgap| max %.3g eV" % (np.abs(dE[ok]).max(), np.abs(dE[ok]).mean(), np.abs(dg[ok]).max()))
w = np.argsort(-np.abs(dE * ok))[:4]
print("worst settled:", [(int(nao[i]), float(dE[i])) for i in w])
for lo, hi in ((0, 17), (17, 33), (33, 49), (49, 65), (65, 81), (81, 97)):
    k = ok & (nao >= lo) & (nao < hi)
    if k.sum():
        print(f"N in [{lo}, {hi}): n={int(k.sum()):2d} |dE| max {np.abs(dE[k]).max():.3g}")
