"""Phase timing of the config-1 energy evaluation (12q UCC + 500-term H)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2208_10978_b200 import _lib, engine, statevector as sv, workloads as W
cfg = W.config1(seed=0)
be = engine.StateVectorBackend()
s0 = be.prepare(cfg["reference"])
t0 = time.perf_counter()
for _ in range(3):
    e = be.expectation(be.evolve(s0, cfg["circuit"]), cfg["hamiltonian"])
print(f"warm-up (incl. any JIT compile) {time.perf_counter() - t0:.2f} s, E = {e!r}, jit {_lib.jit_info()}")
for _ in range(3):
    t0 = time.perf_counter(); psi = be.evolve(s0, cfg["circuit"]); t1 = time.perf_counter()
    psi.synchronize(); t2 = time.perf_counter()
    e = be.expectation(psi, cfg["hamiltonian"]); t3 = time.perf_counter()
    print(f"evolve host {1e3*(t1-t0):.2f} ms, evolve gpu-drain {1e3*(t2-t1):.2f} ms, expectation {1e3*(t3-t2):.2f} ms, stats {sv.last_plan_stats()}")
t0 = time.perf_counter()
for _ in range(50):
    e = be.expectation(be.evolve(s0, cfg["circuit"]), cfg["hamiltonian"])
print(f"{50 / (time.perf_counter() - t0):.1f} evals/s")
