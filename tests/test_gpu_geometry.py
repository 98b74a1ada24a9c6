"""Oracle pins for the tile geometries behind the measured numbers.

Round 1 measured the 30-qubit fused-gate roofline and the config-4 evolve on
tiles with 2 contiguous low qubits (64-B segments), picked by the planner for
rotation-dominated programs at n >= 22 (`pick_contig`), but only mirror tests
(C then C^dagger) covered that geometry.  Here every geometry the planner can
produce is compared with the CPU oracle (`oracle.evolve`, the reference's gate
loop restated, statevector.py:65-74) on the same seeded gates:

* QSV_MIN_CONTIG = 1 / 2 / 4 forced on specialised (NVRTC) passes from 14
  qubits, for UCC rotation programs (the config-4 construction at 18 q) and
  brickwork;
* default knobs at n = 22, where the planner chooses c = 2 by itself;
* config 2's own circuit family (depth-20 brickwork) at 26 q, default knobs.

Tolerances (north_star): amplitudes 1e-10 max-abs; energies 1e-10 relative.
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2208_10978_b200 import _lib
from paper_2208_10978_b200 import statevector as sv
from paper_2208_10978_b200 import workloads as W

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10
REL_TOL = 1e-10


def plan_contig(n, circ):
    kinds, qubits, values = sv._flat(circ)
    plan = _lib.debug_plan(n, kinds, qubits, values)
    return [p["c"] for p in plan["passes"] if not p["global"]]


@pytest.fixture
def jit14(monkeypatch):
    monkeypatch.setenv("QSV_JIT_MIN_QUBITS", "14")
    available, _ = _lib.jit_info()
    assert available, "NVRTC / driver API not loadable on the GPU box"


@pytest.mark.parametrize("contig", ["1", "2", "4"])
def test_ucc_forced_contig_vs_oracle(jit14, monkeypatch, contig):
    """Config-4 construction at 18 q (8 electrons: 160 single + 320 double
    strings = 480 rotations) on tiles with `contig` contiguous low qubits,
    specialised passes, vs the oracle; then the energy of a config-3-style
    Hamiltonian on the result."""
    monkeypatch.setenv("QSV_MIN_CONTIG", contig)
    monkeypatch.setenv("QSV_PARITY", "0")  # full-size tiles (the half: test_gpu_symmetry.py)
    n = 18
    cfg = W.config4(seed=40 + int(contig), n_qubits=n, n_electrons=8, n_doubles=40, n_terms=300)
    assert len(cfg["strings"]) >= 300
    cs = plan_contig(n, cfg["circuit"])
    assert min(cs) == int(contig)
    _, before = _lib.jit_info()
    psi = sv.evolve(sv.init_state(cfg["reference"]), cfg["circuit"])
    _, after = _lib.jit_info()
    # every tile pass ran specialised (a failed launch would fall back silently)
    assert after - before == len(cs), "specialised passes did not run"
    ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    assert np.abs(psi.amplitudes - ref).max() <= AMP_TOL
    e = sv.expectation(psi, cfg["hamiltonian"])
    e_ref = O.expectation(ref, cfg["hamiltonian"], n)
    assert abs(e - e_ref) <= REL_TOL * max(abs(e_ref), 1e-300)


@pytest.mark.parametrize("contig", ["1", "2", "4"])
def test_brickwork_forced_contig_vs_oracle(jit14, monkeypatch, contig):
    monkeypatch.setenv("QSV_MIN_CONTIG", contig)
    n = 18
    circ = W.brickwork(n, 8, seed=60 + int(contig))
    cs = plan_contig(n, circ)
    assert min(cs) == int(contig)
    _, before = _lib.jit_info()
    out = sv.evolve(sv.init_state("0" * n), circ).amplitudes
    assert _lib.jit_info()[1] - before == len(cs)
    ref = O.evolve(O.init_state("0" * n), circ.gates)
    assert np.abs(out - ref).max() <= AMP_TOL


def test_ucc_default_knobs_22q_picks_two_contiguous_vs_oracle(monkeypatch):
    """Default knobs at 22 q: a rotation-dominated program (480 rotations of
    the config-4 construction) makes the planner choose c = 2 on its own --
    the geometry of the fused30 / config-4 numbers -- and the result matches
    the oracle."""
    for k in ("QSV_MIN_CONTIG", "QSV_JIT_MIN_QUBITS", "QSV_JIT"):
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setenv("QSV_PARITY", "0")  # the full 22 q program (the half: test_gpu_symmetry.py)
    n = 22
    cfg = W.config4(seed=22, n_qubits=n, n_electrons=10, n_doubles=30, n_terms=200)
    assert len(cfg["strings"]) >= 300
    assert min(plan_contig(n, cfg["circuit"])) == 2
    _, before = _lib.jit_info()
    psi = sv.evolve(sv.init_state(cfg["reference"]), cfg["circuit"])
    _, after = _lib.jit_info()
    assert after > before
    ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    assert np.abs(psi.amplitudes - ref).max() <= AMP_TOL
    e = sv.expectation(psi, cfg["hamiltonian"])
    assert abs(e - O.expectation(ref, cfg["hamiltonian"], n)) <= REL_TOL * max(abs(e), 1e-300)


def test_config2_family_26q_depth20_vs_oracle(monkeypatch):
    """Config 2's circuit family (Haar U3 layer + alternating CNOTs, depth 20)
    at 26 q with default knobs (specialised passes, 3 contiguous low qubits,
    first pass synthesises |0...0>) vs the oracle."""
    for k in ("QSV_MIN_CONTIG", "QSV_JIT_MIN_QUBITS", "QSV_JIT"):
        monkeypatch.delenv(k, raising=False)
    n = 26
    circ = W.brickwork(n, 20, seed=0)
    out = sv.evolve(sv.init_state("0" * n), circ).amplitudes
    ref = O.evolve(O.init_state("0" * n), circ.gates)
    d = np.abs(out - ref)
    assert d.max() <= AMP_TOL
    assert float(np.sqrt((d * d).sum())) <= 1e-10


def test_singular_u3_angles_fall_back_to_plain_forms(jit14):
    """U3s at theta = pi (cos(theta/2) = 0) cannot take the normalised forms:
    the call runs a plan without them (specialised passes) and matches the
    oracle; the same structure at regular angles keeps the normalised plan."""
    from paper_2208_10978_b200.circuit import Circuit, Constant, Gate

    n = 18
    base = W.brickwork(n, 8, seed=71)
    gates = list(base.gates)
    for i, g in enumerate(gates):
        if g.kind == "U3" and i % 9 == 4:
            gates[i] = Gate("U3", g.qubits, (Constant(np.pi),) + tuple(g.params[1:]))
    for circ in (Circuit(n, tuple(gates), 0), base):
        out = sv.evolve(sv.init_state("0" * n), circ).amplitudes
        ref = O.evolve(O.init_state("0" * n), circ.gates)
        assert np.all(np.isfinite(out))
        assert np.abs(out - ref).max() <= AMP_TOL
