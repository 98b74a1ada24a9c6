"""Host-side phase breakdown of the config-1 evolve (QSV_HOST_PROFILE=1 lines on stderr)."""
import os, sys, time
os.environ["QSV_HOST_PROFILE"] = "1"
sys.path.insert(0, os.getcwd())
from paper_2208_10978_b200 import engine, statevector as sv, workloads as W
cfg = W.config1(seed=0)
be = engine.StateVectorBackend()
s0 = be.prepare(cfg["reference"])
for _ in range(4):
    psi = be.evolve(s0, cfg["circuit"]); psi.synchronize()
for _ in range(3):
    t0 = time.perf_counter(); flat = sv._flat(cfg["circuit"]); t1 = time.perf_counter()
    out = sv.StateVector._empty(12, s0.device); t2 = time.perf_counter()
    sv.apply_circuit_inplace(out, cfg["circuit"]); t3 = time.perf_counter()
    out.synchronize()
    print(f"py: flat {1e6*(t1-t0):.1f} us, empty {1e6*(t2-t1):.1f} us, apply {1e6*(t3-t2):.1f} us", file=sys.stderr)
