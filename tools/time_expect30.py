"""Config-3 expectation timing (30q random state, 10k strings)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2208_10978_b200 import statevector as sv, workloads as W
h = W.config3_hamiltonian(seed=0)
s = sv.StateVector._empty(30)
view = torch.as_tensor(s, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
view.copy_(torch.randn(view.shape, dtype=torch.float64, device="cuda", generator=g))
view /= torch.linalg.vector_norm(view)
torch.cuda.synchronize()
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    t0 = time.perf_counter(); re, im, _ = sv.expectation_terms(s, h); t1 = time.perf_counter()
    print(f"expect30 {t1-t0:.3f}s sweeps={sv.last_plan_stats()['n_passes']} E={re:.15f}", flush=True)
