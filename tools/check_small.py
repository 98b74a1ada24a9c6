"""Small end-to-end check on the GPU: specialised + interpreted tile passes,
fused rotation groups, expectation sweeps and sampling, each against the
oracle (run with QSV_JIT_MIN_QUBITS=14 to force the specialised kernels)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np

from oracle import oracle as O
from paper_2208_10978_b200 import statevector as sv
from paper_2208_10978_b200 import workloads as W
from paper_2208_10978_b200.pauli import PauliString

n = int(sys.argv[1]) if len(sys.argv) > 1 else 14
circ = W.brickwork(n, 4, seed=3)
out = sv.evolve(sv.init_state("0" * n), circ).amplitudes
assert np.abs(out - O.evolve(O.init_state("0" * n), circ.gates)).max() < 1e-10
cfg = W.config1(seed=1, n_qubits=n, n_electrons=6, n_terms=120)
psi = sv.evolve(sv.init_state(cfg["reference"]), cfg["circuit"])
ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
assert np.abs(psi.amplitudes - ref).max() < 1e-10
rng = np.random.default_rng(2)
h = W.sparse_random_hamiltonian(n, 80, rng, z_only=20)
e = sv.expectation(psi, h)
assert abs(e - O.expectation(ref, h, n)) < 1e-10 * max(1, abs(e))
m = sv.sample(psi, PauliString.from_label("Z0 X3"), 2000, 5)
assert m == O.sample(ref, PauliString.from_label("Z0 X3"), 2000, 5)
print("check_small ok", n)
