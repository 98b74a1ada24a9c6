"""Sharded path (distributed.py) on the GPU through libqsv: P logical shards
on one device (LoopbackComm, exchanges are device copies), checked against
the CPU oracle.  Tolerances: amplitudes 1e-10 max-abs, energies 1e-10
relative (BASELINE.json north_star)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2208_10978_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_2208_10978_b200 import distributed

    return distributed


@pytest.mark.parametrize("P,n,layers", [(2, 14, 6), (4, 18, 5), (8, 20, 4)])
def test_sharded_brickwork_vs_oracle(D, P, n, layers):
    circ = W.brickwork(n, layers, seed=20 + P)
    ref = O.evolve(O.init_state("0" * n), circ.gates)
    comm = D.LoopbackComm(P)
    s = D.evolve(D.init_state("0" * n, comm), circ)
    assert np.abs(s.amplitudes() - ref).max() < 1e-10


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_ucc_energy_vs_oracle(D, P):
    cfg = W.config1(seed=2, n_qubits=12, n_electrons=6, n_terms=300)
    ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    e_ref = O.expectation(ref, cfg["hamiltonian"], 12)
    be = D.DistributedBackend(D.LoopbackComm(P))
    psi = be.evolve(be.prepare(cfg["reference"]), cfg["circuit"])
    assert np.abs(psi.amplitudes() - ref).max() < 1e-10
    e = be.expectation(psi, cfg["hamiltonian"])  # dense strings: relayout + pairwise paths
    assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))


def test_sharded_sparse_hamiltonian_20q(D):
    n, P = 20, 4
    circ = W.brickwork(n, 3, seed=9)
    ref = O.evolve(O.init_state("0" * n), circ.gates)
    rng = np.random.default_rng(4)
    h = W.sparse_random_hamiltonian(n, 400, rng, z_only=120)
    e_ref = O.expectation(ref, h, n)
    be = D.DistributedBackend(D.LoopbackComm(P))
    e = be.expectation(be.evolve(be.prepare("0" * n), circ), h)
    assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))
