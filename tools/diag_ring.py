"""Diagnostic: brickwork evolve at several sizes; prints norm + checksum per size."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2208_10978_b200 import statevector as sv, workloads as W
for n in [int(a) for a in sys.argv[1:]]:
    circ = W.brickwork(n, 4, seed=1)
    t0 = time.time()
    psi = sv.evolve(sv.init_state("0" * n), circ)
    psi.synchronize()
    a = psi.amplitudes
    print(n, "t=%.3f" % (time.time() - t0), "norm=%.15f" % np.linalg.norm(a), "chk=%.15e" % float(np.abs(a[::7]).sum()), flush=True)
