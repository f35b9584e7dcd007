import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
torch.cuda.init()
from paper_2311_01135_b200 import synth, SCFOptions, load_basis, scf_batch
from paper_2311_01135_b200 import batch
from paper_2311_01135_b200.engine import Plan
b = load_basis("sto-3g")
mols = synth.batch(256, 9, seed=1)
opts = SCFOptions(max_iterations=20, convergence_std=0.0, grid_level=0, precision="f32")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); pk = batch.pack(mols, b, 0)
    t1 = time.perf_counter(); p = Plan(pk, None, opts.engine()); torch.cuda.synchronize()
    t2 = time.perf_counter(); p.run(); torch.cuda.synchronize()
    t3 = time.perf_counter(); r = p.fetch(); 
    t4 = time.perf_counter(); p.close(); torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"pack {1e3*(t1-t0):.1f} create {1e3*(t2-t1):.1f} run {1e3*(t3-t2):.1f} fetch {1e3*(t4-t3):.1f} close {1e3*(t5-t4):.1f} ms")
    t = time.perf_counter(); out = scf_batch(mols, b, opts); torch.cuda.synchronize(); print("scf_batch total %.1f ms" % (1e3*(time.perf_counter()-t)))
