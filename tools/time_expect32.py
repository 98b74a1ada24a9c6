"""Config-4 Hamiltonian (5,000 strings) expectation timing on a random 32 q state."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2208_10978_b200 import statevector as sv, workloads as W
cfg = W.config4(seed=0)
h = cfg["hamiltonian"]
s = sv.StateVector._empty(32)
view = torch.as_tensor(s, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
view.copy_(torch.randn(view.shape, dtype=torch.float64, device="cuda", generator=g))
view /= torch.linalg.vector_norm(view)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); re, im, _ = sv.expectation_terms(s, h); t1 = time.perf_counter()
    print(f"expect32 TERMS={os.environ.get('QSV_SWEEP_TERMS','24')} {t1-t0:.3f}s sweeps={sv.last_plan_stats()['n_passes']} E={re:.15f}", flush=True)
