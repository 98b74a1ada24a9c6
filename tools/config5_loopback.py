"""Config-5 structure at config 5's TOTAL size that one B200 can hold:
the 10-layer brickwork on 33 qubits (2^33 amplitudes = 128 GiB) sharded over
P = 8 logical shards of 2^30 (top 3 qubits global; exchanges are device
copies, LoopbackComm) -- the same shard-count / global-qubit structure as
config 5 at P = 8, at 1/8 of its per-shard size.

Checks: (1) device memory in use after the evolve of the lazy |0...0> is one
state (+ workspace), not two; (2) mirror parity at full size -- the circuit,
then its inverse applied in place on the sharded state, returns |0...0>
(|<0|psi>| - 1 and the rest of the norm within 1e-10); reports the
relayouts the light-cone scheduler needed and the evolve time."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_2208_10978_b200 import distributed as D  # noqa: E402
from paper_2208_10978_b200 import statevector as sv  # noqa: E402
from paper_2208_10978_b200 import workloads as W  # noqa: E402
from paper_2208_10978_b200.circuit import Circuit, dagger_gate, flatten_bound  # noqa: E402

n, P = int(os.environ.get("N", "33")), int(os.environ.get("P", "8"))
circ = W.brickwork(n, 10, seed=5)
free0, total = sv.mem_info(0)
be = D.DistributedBackend(D.LoopbackComm(P, piece_bytes=256 << 20), D.CudaEngine(0))
s0 = be.prepare("0" * n)
t0 = time.perf_counter()
psi = be.evolve(s0, circ)
for sh in psi.shards.values():
    sh.synchronize()
t1 = time.perf_counter()
free1, _ = sv.mem_info(0)
used = free0 - free1
state = 16 * (1 << n)
print(f"{n}q brickwork x10 ({len(circ.gates)} gates), P={P} loopback shards of 2^{n - 3}: "
      f"evolve {t1 - t0:.2f} s, relayouts {psi.stats['relayouts']}, "
      f"bytes sent per shard {psi.stats['relayout_bytes_sent'] / P:.3e}; device memory in use "
      f"{used / 2**30:.1f} GiB for a {state / 2**30:.0f} GiB state ({used / state:.3f}x)")
assert used <= 1.1 * state
inv = Circuit(n, tuple(dagger_gate(g) for g in reversed(circ.gates)), 0)
t2 = time.perf_counter()
psi.apply_flat(*flatten_bound(inv))
for sh in psi.shards.values():
    sh.synchronize()
t3 = time.perf_counter()
# |0...0> is physical index 0 under any qubit map: rank 0, local 0
amp0 = torch.as_tensor(psi.shards[0], device="cuda")[0]
a0 = complex(float(amp0[0]), float(amp0[1]))
rest = 0.0
for r, sh in psi.shards.items():
    t = torch.as_tensor(sh, device="cuda")
    rest += float((t * t).sum())
rest -= abs(a0) ** 2
print(f"mirror: inverse applied in place in {t3 - t2:.2f} s, relayouts total "
      f"{psi.stats['relayouts']}; |<0|psi>| - 1 = {abs(a0) - 1:.3e}, norm elsewhere {rest:.3e}")
assert abs(abs(a0) - 1) <= 1e-10 and rest <= 1e-10
print("PASS")
