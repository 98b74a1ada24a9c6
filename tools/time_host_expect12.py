"""Host cost of the config-1 expectation (500 strings, 12 q) on an idle device:
the backend call vs the raw C entry with pre-built pointers."""
import ctypes, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2208_10978_b200 import _lib, engine, statevector as sv, workloads as W
cfg = W.config1(seed=0)
be = engine.StateVectorBackend()
s0 = be.prepare(cfg["reference"])
psi = be.evolve(s0, cfg["circuit"])
h = cfg["hamiltonian"]
for _ in range(5):
    be.expectation(psi, h)
x, y, z, cr, ci = sv._hamiltonian(h, 12)
L = _lib.lib()
re, im = ctypes.c_double(), ctypes.c_double()
per = np.zeros(len(cr))
args = (psi.handle, len(cr), _lib.u64ptr(x), _lib.u64ptr(y), _lib.u64ptr(z), _lib.dptr(cr), _lib.dptr(ci),
        ctypes.byref(re), ctypes.byref(im), _lib.dptr(per), None)
for label, fn in [("backend.expectation", lambda: be.expectation(psi, h)),
                  ("expectation_terms", lambda: sv.expectation_terms(psi, h)),
                  ("C entry", lambda: L.qsv_expectation(*args))]:
    tot = 0.0
    for _ in range(300):
        psi.synchronize()
        t0 = time.perf_counter()
        fn()
        tot += time.perf_counter() - t0
    print(f"{label}: {1e6 * tot / 300:.1f} us")
