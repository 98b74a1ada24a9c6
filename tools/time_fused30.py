"""Timing of the 30q UCC-shaped evolve (fused30 extra) under the current env knobs."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2208_10978_b200 import engine, statevector as sv, workloads as W
cfg = W.config4(seed=0, n_qubits=30, n_electrons=15, n_doubles=2000, n_terms=10)
be = engine.StateVectorBackend()
s0 = be.prepare(cfg["reference"])
psi = be.evolve(s0, cfg["circuit"]); psi.synchronize(); del psi
t0 = time.perf_counter()
psi = be.evolve(s0, cfg["circuit"]); psi.synchronize()
dt = time.perf_counter() - t0
st = sv.last_plan_stats()
print(f"fused30 {dt:.3f} s, passes {st['n_passes']}, HBM frac {st['n_passes'] * 32 * 2**30 / dt / 6545.3e9:.3f}")
