"""Host cost of one config-1 evolve call: the raw C entry (qsv_evolve_basis_prepared,
no sync) and the Python evolve wrapper, averaged over 200 calls each, each started on an idle device."""
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2208_10978_b200 import _lib, engine, statevector as sv, workloads as W
from paper_2208_10978_b200.circuit import bind
cfg = W.config1(seed=0)
param = W.parametric_rotations_circuit(12, cfg["strings"])
b = bind(param, cfg["thetas"])
be = engine.StateVectorBackend()
s0 = be.prepare(cfg["reference"])
for _ in range(5):
    be.expectation(be.evolve(s0, b), cfg["hamiltonian"])
pid = b._plan.program_id()
vals = b.flat()[2]
out = sv.StateVector._empty(12, 0)
L = _lib.lib()
h = out.handle
idx = s0.basis_index
for label, fn in [("C entry", lambda: L.qsv_evolve_basis_prepared(h, idx, pid, _lib.dptr(vals), None)),
                  ("python evolve", lambda: be.evolve(s0, b)),
                  ("expectation", lambda: be.expectation(out, cfg["hamiltonian"]))]:
    tot = 0.0
    for _ in range(200):
        out.synchronize()
        t0 = time.perf_counter()
        fn()
        tot += time.perf_counter() - t0
    out.synchronize()
    print(f"{label}: {1e6 * tot / 200:.1f} us per call (host, device idle at entry)")
print("values", vals.size, "rotations", len(cfg["strings"]))
