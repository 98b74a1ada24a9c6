"""Full-size parity of the headline workload: config 2 (28-qubit brickwork,
830 gates) on the B200 vs the C oracle (oracle/liboracle.so; ORACLE_THREADS
OpenMP threads, bit-identical to one core, which takes ~10-20 min), same seeded
gates.  Prints max |d psi|, ||d psi||_2 and the norms."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from oracle import oracle as O
from paper_2208_10978_b200 import statevector as sv, workloads as W

O.set_threads(int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1)))
n = 28
circ = W.brickwork(n, 20, seed=0)
t0 = time.perf_counter()
gpu = sv.evolve(sv.init_state("0" * n), circ).amplitudes
t1 = time.perf_counter()
print(f"B200 evolve + download {t1 - t0:.2f} s", flush=True)
ref = O.evolve(O.init_state("0" * n), circ.gates)
t2 = time.perf_counter()
d = gpu - ref
print(f"oracle evolve {t2 - t1:.0f} s")
print(f"config2 28q: max|d psi| = {np.abs(d).max():.3e}, ||d psi||_2 = {np.linalg.norm(d):.3e}, "
      f"norm gpu = {np.linalg.norm(gpu):.15f}, norm oracle = {np.linalg.norm(ref):.15f}")
assert np.abs(d).max() <= 1e-10
print("PASS (tolerance 1e-10 max-abs, BASELINE.json north_star)")
