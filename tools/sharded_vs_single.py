"""Config-5 structure at a size one B200 holds: the 10-layer brickwork on 29
qubits sharded over P = 8 logical shards (top 3 qubits global; exchanges are
device copies, distributed.LoopbackComm) vs the single-GPU engine on the same
gates; reports the relayouts the light-cone scheduler needed."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2208_10978_b200 import distributed as D, statevector as sv, workloads as W

n, P = int(os.environ.get("N", "29")), int(os.environ.get("P", "8"))
circ = W.brickwork(n, 10, seed=5)
t0 = time.perf_counter()
single = sv.evolve(sv.init_state("0" * n), circ).amplitudes
t1 = time.perf_counter()
be = D.DistributedBackend(D.LoopbackComm(P))
psi = be.evolve(be.prepare("0" * n), circ)
t2 = time.perf_counter()
sharded = psi.amplitudes()
d = np.abs(sharded - single).max()
print(f"brickwork {n}q x10 layers, P={P}: single {t1 - t0:.1f} s, sharded {t2 - t1:.1f} s, "
      f"relayouts {psi.stats['relayouts']}, bytes sent/shard {psi.stats['relayout_bytes_sent'] / P:.3e}; "
      f"max |sharded - single| = {d:.3e}")
assert d <= 1e-10
print("PASS")
