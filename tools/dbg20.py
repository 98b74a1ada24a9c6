import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2208_10978_b200 import statevector as sv, workloads as W
from oracle import oracle as O
circ = W.brickwork(20, 6, seed=5)
ref = O.evolve(O.init_state("0"*20), circ.gates)
out = sv.evolve(sv.init_state("0"*20), circ).amplitudes
err = np.abs(out-ref)
bad = np.nonzero(err > 1e-10)[0]
print(os.environ.get("QSV_TILE_GRID"), "maxerr", err.max(), "nbad", len(bad), "first", bad[:4], "hi bits of bad", sorted(set((bad >> 12).tolist()))[:20])
