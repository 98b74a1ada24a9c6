"""Two evolves of the 30q UCC-shaped circuit (fused30 extra) for ncu."""
import os, sys
sys.path.insert(0, os.getcwd())
from paper_2208_10978_b200 import engine, statevector as sv, workloads as W
cfg = W.config4(seed=0, n_qubits=30, n_electrons=15, n_doubles=2000, n_terms=10)
be = engine.StateVectorBackend()
s0 = be.prepare(cfg["reference"])
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    psi = be.evolve(s0, cfg["circuit"]); psi.synchronize(); del psi
print("ok", sv.last_plan_stats())
