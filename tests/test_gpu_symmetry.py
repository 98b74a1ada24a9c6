"""Parity-reduced evolves (symmetry.py) on the B200 vs the oracle.

Config 4's construction (UCC singles + doubles: even flips) from the
Hartree-Fock state at 14-18 q: the evolve runs as an (n-1)-qubit half
(ParityReduced); amplitudes (materialised by qsv_embed_parity), energies
(transformed terms on the half) and chained operations must match the CPU
oracle (oracle.evolve / oracle.expectation, statevector.py:65-110) and the
unreduced device path (QSV_PARITY=0).  Tolerances: 1e-10 (north_star)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2208_10978_b200 import engine
from paper_2208_10978_b200 import statevector as sv
from paper_2208_10978_b200 import workloads as W

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.mark.parametrize("n,ne,nd", [(14, 6, 60), (16, 8, 80), (18, 8, 40)])
def test_ucc_parity_reduced_vs_oracle(n, ne, nd, monkeypatch):
    cfg = W.config4(seed=n, n_qubits=n, n_electrons=ne, n_doubles=nd, n_terms=150)
    be = engine.StateVectorBackend()
    s0 = be.prepare(cfg["reference"])
    psi = be.evolve(s0, cfg["circuit"])
    assert isinstance(psi, sv.ParityReduced) and psi.reduced
    assert sv.last_reduction()["n_eff"] == n - 1
    e = be.expectation(psi, cfg["hamiltonian"])
    assert psi.reduced  # the energy ran on the half
    ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    e_ref = O.expectation(ref, cfg["hamiltonian"], n)
    assert abs(e - e_ref) <= TOL * max(1.0, abs(e_ref))
    amps = psi.amplitudes  # materialises the full state
    assert not psi.reduced
    assert np.abs(amps - ref).max() <= TOL
    assert abs(be.expectation(psi, cfg["hamiltonian"]) - e_ref) <= TOL * max(1.0, abs(e_ref))
    monkeypatch.setenv("QSV_PARITY", "0")
    full = be.evolve(s0, cfg["circuit"])
    assert not isinstance(full, sv.ParityReduced)
    assert np.abs(full.amplitudes - ref).max() <= TOL


def test_parity_reduced_chained_operations():
    n = 15
    cfg = W.config4(seed=3, n_qubits=n, n_electrons=7, n_doubles=40, n_terms=80)
    s0 = sv.init_state(cfg["reference"])
    a = sv.evolve(s0, cfg["circuit"])
    b = sv.evolve(s0, cfg["circuit"])
    assert isinstance(a, sv.ParityReduced) and isinstance(b, sv.ParityReduced)
    assert abs(a.norm() - 1.0) <= 1e-12
    assert abs(sv.vdot(a, b) - 1.0) <= 1e-12
    ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    c = sv.evolve(b, cfg["circuit"])  # from a non-basis (materialised) state: full path
    ref2 = O.evolve(ref.copy(), cfg["circuit"].gates)
    assert np.abs(c.amplitudes - ref2).max() <= TOL
    hp = sv.apply_operator(sv.evolve(s0, cfg["circuit"]), cfg["hamiltonian"])
    assert np.abs(hp.amplitudes - O.apply_operator(ref, cfg["hamiltonian"], n)).max() <= TOL
