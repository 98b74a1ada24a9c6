"""Where the config-1 energy evaluation spends host time: cProfile of 300
evaluations (evolve + expectation through the backend), sorted by own time,
and the library's per-phase host profile of one evolve and one expectation."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.getcwd())
from paper_2208_10978_b200 import engine, workloads as W
cfg = W.config1(seed=0)
be = engine.StateVectorBackend()
s0 = be.prepare(cfg["reference"])
c, h = cfg["circuit"], cfg["hamiltonian"]
for _ in range(10):
    be.expectation(be.evolve(s0, c), h)
t0 = time.perf_counter()
for _ in range(300):
    be.expectation(be.evolve(s0, c), h)
print(f"{300 / (time.perf_counter() - t0):.1f} evals/s")
pr = cProfile.Profile()
pr.enable()
for _ in range(300):
    be.expectation(be.evolve(s0, c), h)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
os.environ["QSV_HOST_PROFILE"] = "1"
for _ in range(3):
    be.expectation(be.evolve(s0, c), h)
