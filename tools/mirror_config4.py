"""Config 4 at full size (32 qubits, 64 GiB state): the UCC circuit followed by
its inverse (reversed order, negated angles) must return the Hartree-Fock
basis state -- the size-independent check where no CPU oracle can run."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
from paper_2208_10978_b200 import statevector as sv, workloads as W

cfg = W.config4(seed=0)
n = cfg["n_qubits"]
fwd = cfg["circuit"]
back = W.rotations_circuit(n, cfg["strings"][::-1], -cfg["thetas"][::-1])
t0 = time.perf_counter()
psi = sv.evolve(sv.init_state(cfg["reference"]), fwd)
psi = sv.evolve(psi, back)
psi.synchronize()
dt = time.perf_counter() - t0
view = torch.as_tensor(psi, device="cuda")           # (2^n, 2) float64, zero-copy
hf = int(cfg["reference"][::-1], 2)                   # char k = qubit k
amp = view[hf].cpu().numpy()
view[hf] = 0.0
rest = float(torch.linalg.vector_norm(view).item())
print(f"config4 32q mirror ({2 * len(cfg['strings'])} rotations, {dt:.1f} s): "
      f"<HF|psi> = {amp[0]:.15f} {amp[1]:+.3e}i, ||psi - |HF>|| off-HF = {rest:.3e}")
assert abs(amp[0] - 1.0) <= 1e-10 and abs(amp[1]) <= 1e-10 and rest <= 1e-10
print("PASS")
