"""Config-4 (32q UCC) evolve + expectation timing (one warm run)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2208_10978_b200 import engine, statevector as sv, workloads as W
cfg = W.config4(seed=0)
be = engine.StateVectorBackend()
s0 = be.prepare(cfg["reference"])
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t0 = time.perf_counter(); psi = be.evolve(s0, cfg["circuit"]); psi.synchronize(); t1 = time.perf_counter()
    st = sv.last_plan_stats()
    e = be.expectation(psi, cfg["hamiltonian"]); t2 = time.perf_counter()
    print(f"ucc32 c={os.environ.get('QSV_MIN_CONTIG','5')} evolve {t1-t0:.2f}s ({st['n_passes']} passes) expectation {t2-t1:.2f}s ({sv.last_plan_stats()['n_passes']} sweeps) E={e:.12f}", flush=True)
    del psi
