"""Edge cases of the CUDA path vs the CPU oracle: tiny and tile-boundary
state sizes, empty circuits and Hamiltonians, identity strings, identity
rotations (global phase), the specialised-pass threshold, invalid inputs.
Tolerances: amplitudes 1e-10 max-abs, energies 1e-10 relative."""

import numpy as np
import pytest

from conftest import random_state
from oracle import oracle as O
from paper_2208_10978_b200 import statevector as sv
from paper_2208_10978_b200 import workloads as W
from paper_2208_10978_b200.circuit import Circuit, Constant, Gate
from paper_2208_10978_b200.errors import ResourceLimitError
from paper_2208_10978_b200.pauli import PauliString, PauliSum, PauliTerm

pytestmark = pytest.mark.gpu


def _mixed(n, G, seed):
    rng = np.random.default_rng(seed)
    kinds = ["H", "HY", "X", "CNOT", "SWAP", "RZ", "RY", "U3", "CU3"]
    npar = {"RZ": 1, "RY": 1, "U3": 3, "CU3": 3}
    gates = []
    for _ in range(G):
        k = kinds[rng.integers(len(kinds))]
        nq = 2 if k in ("CNOT", "SWAP", "CU3") else 1
        if nq > n:
            k, nq = "U3", 1
        qs = tuple(int(q) for q in rng.choice(n, size=nq, replace=False))
        gates.append(Gate(k, qs, tuple(Constant(float(v)) for v in rng.uniform(-3, 3, npar.get(k, 0)))))
    return Circuit(n, tuple(gates), 0)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 11, 12, 13])
def test_sizes_around_the_tile(n):
    rng = np.random.default_rng(n)
    circ = _mixed(n, 60, n)
    st = random_state(n, rng)
    out = sv.evolve(sv.from_amplitudes(st), circ).amplitudes
    assert np.abs(out - O.evolve(st, circ.gates)).max() <= 1e-10
    h = W.dense_random_hamiltonian(n, 30, rng)
    ref = O.evolve(st, circ.gates)
    e = sv.expectation(sv.from_amplitudes(ref), h)
    e_ref = O.expectation(ref, h, n)
    assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))


@pytest.mark.parametrize("n", [21, 22])
def test_specialisation_threshold(n):
    # QSV_JIT_MIN_QUBITS defaults to 22: both sides of the switch
    circ = W.brickwork(n, 3, seed=n)
    out = sv.evolve(sv.init_state("0" * n), circ).amplitudes
    assert np.abs(out - O.evolve(O.init_state("0" * n), circ.gates)).max() <= 1e-10


def test_empty_circuit_and_hamiltonian():
    n = 6
    st = random_state(n, np.random.default_rng(0))
    s = sv.from_amplitudes(st)
    out = sv.evolve(s, Circuit(n, (), 0))
    assert np.array_equal(out.amplitudes, st)
    assert sv.expectation(s, PauliSum(())) == 0.0


def test_identity_string_and_identity_rotation():
    n = 7
    rng = np.random.default_rng(1)
    st = random_state(n, rng)
    h = PauliSum((PauliTerm(2.5, PauliString(())), PauliTerm(-0.5, PauliString.from_label("Z3 X1"))))
    e = sv.expectation(sv.from_amplitudes(st), h)
    assert abs(e - O.expectation(st, h, n)) <= 1e-12
    # exp(-i t/2 I) is the global phase exp(-i t/2) (statevector semantics of a rotation list)
    x = np.array([0, 0b101], dtype=np.uint64)
    y = np.array([0, 0], dtype=np.uint64)
    z = np.array([0, 0b10], dtype=np.uint64)
    theta = np.array([0.7, -0.3])
    out = sv.apply_rotations(sv.from_amplitudes(st), x, y, z, theta).amplitudes
    ref = st * np.exp(-0.35j)
    scratch = np.empty_like(ref)
    O.apply_pauli(ref, 0b101, 0, 0b10, scratch)
    ref = np.cos(-0.15) * ref - 1j * np.sin(-0.15) * scratch
    assert np.abs(out - ref).max() <= 1e-12


def test_invalid_inputs_raise():
    s = sv.init_state("0000")
    with pytest.raises(ValueError):
        sv.evolve(s, Circuit(5, (Gate("H", (4,)),), 0))
    with pytest.raises(ValueError):
        sv.expectation(s, PauliSum((PauliTerm(1.0, PauliString.from_label("X4")),)))
    with pytest.raises(ValueError):
        sv.sample(s, PauliString.from_label("Z0"), 0, 1)
    with pytest.raises(ValueError):
        sv.from_amplitudes(np.ones(3))


@pytest.mark.parametrize("n,ne", [(12, 6), (13, 6)])
def test_hot_program_specialisation(n, ne, monkeypatch):
    """Below the specialisation threshold a structure is compiled once it has
    run QSV_JIT_HOT_USES (3) times; every run -- interpreted, then
    specialised, with new angles each time -- matches the oracle.  (Tile
    passes forced: at 12 q a rotation-only program otherwise runs as a
    small-state program, tests/test_gpu_small.py, and from 13 q as a
    parity-reduced half, tests/test_gpu_symmetry.py.)"""
    monkeypatch.setenv("QSV_SMALL", "0")
    monkeypatch.setenv("QSV_PARITY", "0")  # full-size passes (the half: test_gpu_symmetry.py)
    from paper_2208_10978_b200 import _lib
    from paper_2208_10978_b200.circuit import bind

    strings = W.ucc_rotation_strings(n, ne)[:160]
    param = W.parametric_rotations_circuit(n, strings)
    ref = W.hf_bitstring(ne, n)
    rng = np.random.default_rng(n)
    _, before = _lib.jit_info()
    for k in range(4):
        theta = rng.uniform(-0.3, 0.3, len(strings))
        bound = bind(param, theta)
        psi = sv.evolve(sv.init_state(ref), bound)
        exp = O.evolve(O.init_state(ref), W.rotations_circuit(n, strings, theta).gates)
        assert np.abs(psi.amplitudes - exp).max() <= 1e-10
    _, after = _lib.jit_info()
    assert after > before  # the later runs used specialised passes


def test_prepared_program_and_async_download_errors():
    """Prepared programs: unknown ids, qubit-count mismatch and non-finite
    values fail loudly; a bound circuit on a state of another size is
    rejected; download_wait without a pending copy is a no-op."""
    import ctypes

    from paper_2208_10978_b200 import _lib
    from paper_2208_10978_b200.circuit import bind

    strings = W.ucc_rotation_strings(6, 2)[:8]
    param = W.parametric_rotations_circuit(6, strings)
    b = bind(param, np.full(len(strings), 0.1))
    pid = b._plan.program_id()
    s6, s7 = sv.init_state("000000"), sv.init_state("0000000")
    vals = b.flat()[2].copy()
    L = _lib.lib()
    assert L.qsv_apply_prepared(s6.handle, 987654321, _lib.dptr(vals), None) != 0
    assert L.qsv_apply_prepared(s7.handle, pid, _lib.dptr(vals), None) != 0
    vals[3] = np.nan
    assert L.qsv_apply_prepared(s6.handle, pid, _lib.dptr(vals), None) != 0
    with pytest.raises(ValueError):
        sv.evolve(s7, b)
    out = sv.evolve(s6, b)
    out.wait_download()  # nothing pending
    ref = O.evolve(O.init_state("000000"), W.rotations_circuit(6, strings, np.full(len(strings), 0.1)).gates)
    assert np.abs(out.amplitudes - ref).max() <= 1e-10


def _dense_ref(st, m, qubits):
    """The apply_2q convention (_cykernels.pyx:41-73: row = 2*bit(q0) +
    bit(q1)) for k targets: row bit (k-1-i) is the bit of qubits[i]."""
    k = len(qubits)
    out = st.copy()
    idx = np.arange(st.size, dtype=np.int64)
    mask = sum(1 << q for q in qubits)
    base = idx[(idx & mask) == 0]
    offs = [sum(((r >> (k - 1 - i)) & 1) << q for i, q in enumerate(qubits)) for r in range(1 << k)]
    a = np.stack([st[base | o] for o in offs])  # [2^k, cosets]
    b = m @ a
    for r, o in enumerate(offs):
        out[base | o] = b[r]
    return out


@pytest.mark.parametrize("n,qubits", [(9, (4,)), (9, (2, 7)), (10, (0, 5, 3)), (11, (8, 1, 9, 2)),
                                      (12, (3, 11, 0, 6, 1)), (14, (13, 12, 11, 10, 9))])
def test_apply_matrix_general_k(n, qubits):
    """qsv_apply_matrix (k = 1..5) vs a NumPy restatement of the apply_2q index
    convention; k = 1, 2 also vs the reference's own apply_1q / apply_2q
    (oracle); a Kronecker product equals the single-qubit gates in sequence."""
    from oracle import oracle as O
    from paper_2208_10978_b200 import kernels

    rng = np.random.default_rng(n + len(qubits))
    k = len(qubits)
    a = rng.standard_normal((1 << k, 1 << k)) + 1j * rng.standard_normal((1 << k, 1 << k))
    m, _ = np.linalg.qr(a)
    st = random_state(n, rng)
    s = sv.from_amplitudes(st)
    kernels.apply_matrix(s, m, qubits)
    out = s.amplitudes
    assert np.abs(out - _dense_ref(st, m, qubits)).max() <= 1e-12
    if k == 1:
        ref = st.copy()
        O.apply_1q(ref, m, qubits[0])
        assert np.abs(out - ref).max() <= 1e-12
    if k == 2:
        ref = st.copy()
        O.apply_2q(ref, m, qubits[0], qubits[1])
        assert np.abs(out - ref).max() <= 1e-12
    # Kronecker convention: qubits[0] is the most significant factor
    us = [np.linalg.qr(rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2)))[0] for _ in qubits]
    kr = us[0]
    for u in us[1:]:
        kr = np.kron(kr, u)
    s2 = sv.from_amplitudes(st)
    kernels.apply_matrix(s2, kr, qubits)
    ref = st.copy()
    for u, q in zip(us, qubits):
        O.apply_1q(ref, u, q)
    assert np.abs(s2.amplitudes - ref).max() <= 1e-12


def test_apply_matrix_errors():
    from paper_2208_10978_b200 import kernels

    s = sv.from_amplitudes(random_state(8, np.random.default_rng(1)))
    with pytest.raises(ValueError):
        kernels.apply_matrix(s, np.eye(4), (3, 3))  # duplicate qubit
    with pytest.raises(ValueError):
        kernels.apply_matrix(s, np.eye(4), (3, 8))  # out of range
    with pytest.raises(ValueError):
        kernels.apply_matrix(s, np.eye(8), (1, 2))  # shape mismatch
    with pytest.raises(ResourceLimitError):
        kernels.apply_matrix(s, np.eye(64), (0, 1, 2, 3, 4, 5))  # k > 5
