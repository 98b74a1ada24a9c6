"""Profiling driver: first N gate-passes of the config-4 (32q UCC) evolve only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2208_10978_b200 import statevector as sv  # noqa: E402
from paper_2208_10978_b200 import workloads as W  # noqa: E402
from paper_2208_10978_b200.circuit import Circuit  # noqa: E402

cfg = W.config4()
ngates = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
circ = Circuit(32, cfg["circuit"].gates[:ngates], 0)
s0 = sv.init_state(cfg["reference"])
for _ in range(2):
    t0 = time.perf_counter()
    psi = sv.evolve(s0, circ)
    psi.synchronize()
    print("evolve", ngates, "gates", time.perf_counter() - t0, sv.last_plan_stats())
    del psi
