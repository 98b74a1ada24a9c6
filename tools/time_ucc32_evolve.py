"""Config-4 evolve-only timing (32q UCC), warm."""
import os, sys, time
sys.path.insert(0, os.getcwd())
from paper_2208_10978_b200 import engine, statevector as sv, workloads as W
cfg = W.config4(seed=0, n_terms=10)
be = engine.StateVectorBackend()
s0 = be.prepare(cfg["reference"])
psi = be.evolve(s0, cfg["circuit"]); psi.synchronize(); del psi
t0 = time.perf_counter(); psi = be.evolve(s0, cfg["circuit"]); psi.synchronize(); t1 = time.perf_counter()
st = sv.last_plan_stats()
print(f"ucc32 evolve c={os.environ.get('QSV_MIN_CONTIG','3')} {t1-t0:.2f}s passes={st['n_passes']} GB/s={st['n_passes']*32*2**32/(t1-t0)/1e9:.0f}", flush=True)
