"""CUDA engine vs the reference golden vectors and the CPU oracle.

Tolerances (north_star): amplitudes within 1e-10 max-abs, energies within
1e-10 relative, FP64 throughout."""

import numpy as np
import pytest

from conftest import parse_h, random_state
from oracle import oracle as O
from paper_2208_10978_b200 import engine, kernels
from paper_2208_10978_b200 import statevector as sv
from paper_2208_10978_b200 import workloads as W
from paper_2208_10978_b200.circuit import (Circuit, Constant, Gate, bind, circuit_from_json,
                                           evolution_gates, gate_matrix)
from paper_2208_10978_b200.errors import ResourceLimitError
from paper_2208_10978_b200.pauli import PauliString, PauliSum, PauliTerm

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10
REL_TOL = 1e-10


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def test_kernels_implementation_is_cuda():
    assert kernels.IMPLEMENTATION == "cuda-sm_100a"


@pytest.mark.parametrize("n", [5, 9])
def test_golden_mixed_circuits(golden, n):
    circ = circuit_from_json(str(golden[f"mixed_n{n}_circuit"]))
    s0 = sv.from_amplitudes(golden[f"mixed_n{n}_in"])
    s1 = sv.evolve(s0, circ)
    assert np.abs(s1.amplitudes - golden[f"mixed_n{n}_out"]).max() <= AMP_TOL
    # input untouched (statevector.py:71)
    assert np.array_equal(s0.amplitudes, golden[f"mixed_n{n}_in"])


@pytest.mark.parametrize("n", [6, 10])
def test_golden_brickwork(golden, n):
    circ = circuit_from_json(str(golden[f"brick_n{n}_circuit"]))
    out = sv.evolve(sv.init_state("0" * n), circ).amplitudes
    assert np.abs(out - golden[f"brick_n{n}_out"]).max() <= AMP_TOL


def test_golden_apply_pauli(golden):
    s = sv.from_amplitudes(golden["pauli_in"])
    for (x, y, z), ref in zip(golden["pauli_masks"], golden["pauli_out"]):
        out = sv.StateVector._empty(s.n_qubits)
        kernels.apply_pauli(s, int(x), int(y), int(z), out)
        assert np.abs(out.amplitudes - ref).max() <= 1e-15


def test_golden_expectation(golden):
    s = sv.from_amplitudes(golden["expect_state"])
    h = parse_h(golden["expect_h"])
    e = sv.expectation(s, h)
    assert rel(e, float(golden["expect_value"])) <= REL_TOL
    _, _, per = sv.expectation_terms(s, h)
    assert np.abs(per - golden["expect_per_term"].real).max() <= 1e-12
    out = sv.apply_operator(s, h).amplitudes
    assert np.abs(out - golden["apply_operator_out"]).max() <= AMP_TOL


def test_golden_uccsd8(golden):
    circ = circuit_from_json(str(golden["uccsd8_circuit"]))
    be = engine.StateVectorBackend()
    psi = be.evolve(be.prepare(str(golden["uccsd8_reference"])), circ)
    assert np.abs(psi.amplitudes - golden["uccsd8_out"]).max() <= AMP_TOL
    e = be.expectation(psi, parse_h(golden["uccsd8_h"]))
    assert rel(e, float(golden["uccsd8_energy"])) <= REL_TOL


def test_h2_fixture_energies(h2_fixtures):
    be = engine.StateVectorBackend()
    for name, fx in h2_fixtures.items():
        h = parse_h(fx["hamiltonian"])
        s0 = be.prepare(fx["reference"])
        assert rel(be.expectation(s0, h), fx["fixture_hf_energy"]) <= REL_TOL, name
        ansatz = circuit_from_json(fx["ansatz"])
        psi = be.evolve(s0, bind(ansatz, fx["theta_opt"]))
        assert rel(be.expectation(psi, h), fx["fixture_fci_energy"]) <= REL_TOL, name
        assert abs(be.overlap(psi, psi) - 1.0) <= 1e-12


def test_config1_full(config1_golden):
    cfg = W.config1(seed=0)
    psi = sv.evolve(sv.init_state(cfg["reference"]), cfg["circuit"])
    st = sv.last_plan_stats()
    assert st["n_rotations"] == 1872 and st["n_passes"] == 4  # parameter budget per pass
    assert np.abs(psi.amplitudes - config1_golden["amplitudes"]).max() <= AMP_TOL
    assert rel(sv.expectation(psi, cfg["hamiltonian"]), float(config1_golden["energy"])) <= REL_TOL


@pytest.mark.parametrize("n", [3, 7, 12, 13, 15])
def test_apply_1q_2q_every_position(n):
    rng = np.random.default_rng(n)
    st = random_state(n, rng)
    s = sv.from_amplitudes(st)
    ref = st.copy()
    for q in range(n):
        m = O.gate_matrix("U3", tuple(rng.uniform(-3, 3, size=3)))
        kernels.apply_1q(s, m, q)
        O.apply_1q(ref, m, q)
    for _ in range(2 * n):
        q0, q1 = (int(v) for v in rng.choice(n, size=2, replace=False))
        m = O.gate_matrix("CU3", tuple(rng.uniform(-3, 3, size=3)))
        kernels.apply_2q(s, m, q0, q1)
        O.apply_2q(ref, m, q0, q1)
    assert np.abs(s.amplitudes - ref).max() <= AMP_TOL


def random_mixed(n, n_gates, rng):
    kinds = ["H", "HY", "X", "CNOT", "SWAP", "RZ", "RY", "U3", "CU3"]
    nparams = {"RZ": 1, "RY": 1, "U3": 3, "CU3": 3}
    gates = []
    for _ in range(n_gates):
        k = kinds[rng.integers(len(kinds))]
        nq = 2 if k in ("CNOT", "SWAP", "CU3") else 1
        qs = tuple(int(q) for q in rng.choice(n, size=nq, replace=False))
        ps = tuple(Constant(float(v)) for v in rng.uniform(-3, 3, size=nparams.get(k, 0)))
        gates.append(Gate(k, qs, ps))
    return Circuit(n, tuple(gates), 0)


@pytest.mark.parametrize("n,g", [(14, 300), (17, 400)])
def test_random_mixed_multi_tile(n, g):
    rng = np.random.default_rng(100 + n)
    circ = random_mixed(n, g, rng)
    st = random_state(n, rng)
    out = sv.evolve(sv.from_amplitudes(st), circ).amplitudes
    ref = O.evolve(st, circ.gates)
    assert np.abs(out - ref).max() <= AMP_TOL


def random_rotations(n, count, rng, max_w=6):
    strings, thetas = [], []
    for _ in range(count):
        w = int(rng.integers(1, max_w + 1))
        pos = rng.choice(n, size=w, replace=False)
        axes = rng.choice(list("XYZ"), size=w)
        strings.append(PauliString(tuple(zip((int(p) for p in pos), axes))))
        thetas.append(float(rng.uniform(-1, 1)))
    return strings, thetas


@pytest.mark.parametrize("n", [13, 18])
def test_rotations_vs_decomposed_oracle(n):
    rng = np.random.default_rng(7 * n)
    strings, thetas = random_rotations(n, 120, rng)
    # repeat flips to exercise same-flip groups
    strings += strings[:10]
    thetas += thetas[:10]
    circ = W.rotations_circuit(n, strings, thetas)
    st = random_state(n, rng)
    out = sv.evolve(sv.from_amplitudes(st), circ)
    assert sv.last_plan_stats()["n_rotations"] == len(strings)
    ref = O.evolve(st, circ.gates)
    assert np.abs(out.amplitudes - ref).max() <= AMP_TOL
    # direct rotation API agrees too
    x, y, z = W.string_masks(strings)
    out2 = sv.apply_rotations(sv.from_amplitudes(st), x, y, z, np.array(thetas))
    assert np.abs(out2.amplitudes - ref).max() <= AMP_TOL


def test_wide_flip_global_fallback():
    n = 18
    rng = np.random.default_rng(3)
    s = PauliString(tuple((q, "XY"[q % 2]) for q in range(2, 16)) + ((17, "Z"),))
    circ = W.rotations_circuit(n, [s, s], [0.7, -0.2])
    st = random_state(n, rng)
    out = sv.evolve(sv.from_amplitudes(st), circ)
    assert sv.last_plan_stats()["n_fallback"] >= 1
    ref = O.evolve(st, circ.gates)
    assert np.abs(out.amplitudes - ref).max() <= AMP_TOL
    h = PauliSum((PauliTerm(0.8, s), PauliTerm(-1.1, PauliString.from_label("X3 Y9 Z17"))))
    e = sv.expectation(sv.from_amplitudes(ref), h)
    assert rel(e, O.expectation(ref, h, n)) <= REL_TOL


@pytest.mark.parametrize("n,S", [(12, 400), (16, 600), (20, 300)])
def test_expectation_vs_oracle(n, S):
    rng = np.random.default_rng(n * 31 + S)
    h = W.sparse_random_hamiltonian(n, S, rng, z_only=S // 3)
    h = PauliSum(h.terms + (PauliTerm(0.5, PauliString()),))  # identity term
    st = random_state(n, rng)
    s = sv.from_amplitudes(st)
    e = sv.expectation(s, h)
    ref, per_ref = O.expectation(st, h, n, per_term=True)
    assert rel(e, ref) <= REL_TOL
    _, _, per = sv.expectation_terms(s, h)
    assert np.abs(per - per_ref[:, 0]).max() <= 1e-12


def test_dense_hamiltonian_config1_shape():
    rng = np.random.default_rng(11)
    h = W.dense_random_hamiltonian(12, 500, rng)
    st = random_state(12, rng)
    assert rel(sv.expectation(sv.from_amplitudes(st), h), O.expectation(st, h, 12)) <= REL_TOL


def test_brickwork_vs_oracle_20q():
    circ = W.brickwork(20, 6, seed=5)
    out = sv.evolve(sv.init_state("0" * 20), circ).amplitudes
    ref = O.evolve(O.init_state("0" * 20), circ.gates)
    assert np.abs(out - ref).max() <= AMP_TOL


def inverse(circ):
    gates = []
    for g in reversed(circ.gates):
        if g.kind == "U3":
            th, ph, la = g.bound_values()
            gates.append(Gate("U3", g.qubits, (Constant(-th), Constant(-la), Constant(-ph))))
        else:
            gates.append(g)
    return Circuit(circ.n_qubits, tuple(gates), 0)


@pytest.mark.parametrize("n,layers", [(26, 6), (28, 20)])
def test_brickwork_mirror_large(n, layers):
    circ = W.brickwork(n, layers, seed=0)
    psi = sv.evolve(sv.init_state("0" * n), circ)
    assert abs(psi.norm() - 1.0) <= 1e-12
    back = sv.evolve(psi, inverse(circ))
    a = back.amplitudes
    assert abs(a[0] - 1.0) <= 1e-10
    a[0] = 0
    assert np.abs(a).max() <= 1e-10


def test_backend_protocol_and_errors():
    be = engine.StateVectorBackend()
    assert be.name == "sv-b200" and be.supports_reverse_gradient is False
    s0 = be.prepare("1100")
    assert s0.amplitudes[3] == 1.0
    circ = Circuit(4, (Gate("H", (0,)),), 0)
    with pytest.raises(ValueError):
        be.evolve(be.prepare("110"), circ)
    from paper_2208_10978_b200.circuit import Affine
    with pytest.raises(RuntimeError):
        be.evolve(s0, Circuit(4, (Gate("RZ", (0,), (Affine(0, 1.0),)),), 1))
    with pytest.raises(ValueError):
        be.expectation(s0, PauliSum((PauliTerm(1j, PauliString.from_label("Z0")),)))
    with pytest.raises(ValueError):
        be.expectation(s0, PauliSum((PauliTerm(1.0, PauliString.from_label("Z7")),)))
    with pytest.raises(ValueError):
        sv.init_state("01x")
    with pytest.raises(ResourceLimitError):
        sv.init_state("0" * 40)
    psi = be.evolve(s0, circ)
    assert abs(be.overlap(psi, s0) + np.sqrt(0.5)) <= 1e-15  # H|1> = (|0> - |1>)/sqrt2 on qubit 0


@pytest.fixture
def jit_from_14(monkeypatch):
    """Specialise (NVRTC) tile passes from 14 qubits so the JIT path is
    checked against the oracle at sizes the oracle finishes quickly."""
    from paper_2208_10978_b200 import _lib

    monkeypatch.setenv("QSV_JIT_MIN_QUBITS", "14")
    available, _ = _lib.jit_info()
    assert available, "NVRTC / driver API not loadable on the GPU box"
    return _lib


@pytest.mark.parametrize("fuse", ["0", "1", "2"])
def test_jit_brickwork_vs_oracle(jit_from_14, monkeypatch, fuse):
    monkeypatch.setenv("QSV_FUSE_QUBITS", fuse)
    _, before = jit_from_14.jit_info()
    circ = W.brickwork(16, 8, seed=12 + int(fuse))  # distinct structure per setting (plan cache)
    out = sv.evolve(sv.init_state("0" * 16), circ).amplitudes
    ref = O.evolve(O.init_state("0" * 16), circ.gates)
    assert np.abs(out - ref).max() <= AMP_TOL
    _, after = jit_from_14.jit_info()
    assert after > before  # the specialised kernels ran


@pytest.mark.parametrize("n,g", [(14, 400), (17, 500)])
def test_jit_random_mixed_vs_oracle(jit_from_14, n, g):
    # every gate kind: H HY X CNOT SWAP RZ RY U3 CU3 -> U1 classes, U2, diagonals,
    # permutations folded into the tile map
    rng = np.random.default_rng(300 + n)
    circ = random_mixed(n, g, rng)
    st = random_state(n, rng)
    out = sv.evolve(sv.from_amplitudes(st), circ).amplitudes
    ref = O.evolve(st, circ.gates)
    assert np.abs(out - ref).max() <= AMP_TOL


@pytest.mark.parametrize("n,ne", [(14, 6), (16, 8)])
def test_jit_ucc_groups_vs_oracle(jit_from_14, n, ne, monkeypatch):
    # UCC-shaped circuits: fused same-flip groups (OP_GMAT) in specialised passes
    # at full size (the parity reduction, tests/test_gpu_symmetry.py, off)
    monkeypatch.setenv("QSV_PARITY", "0")
    cfg = W.config1(seed=n, n_qubits=n, n_electrons=ne, n_terms=200)
    _, before = jit_from_14.jit_info()
    psi = sv.evolve(sv.init_state(cfg["reference"]), cfg["circuit"])
    _, after = jit_from_14.jit_info()
    ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    assert np.abs(psi.amplitudes - ref).max() <= AMP_TOL
    assert after > before
    e = sv.expectation(psi, cfg["hamiltonian"])
    assert rel(e, O.expectation(ref, cfg["hamiltonian"], n)) <= REL_TOL


def test_jit_rotations_mixed_vs_oracle(jit_from_14):
    n = 16
    rng = np.random.default_rng(77)
    strings, thetas = random_rotations(n, 150, rng, max_w=4)
    strings += strings[:20]
    thetas += thetas[:20]
    circ = W.rotations_circuit(n, strings, thetas)
    st = random_state(n, rng)
    out = sv.evolve(sv.from_amplitudes(st), circ).amplitudes
    ref = O.evolve(st, circ.gates)
    assert np.abs(out - ref).max() <= AMP_TOL


@pytest.mark.parametrize("n,S,zq", [(16, 400, 120), (18, 300, 0)])
def test_jit_expectation_sweeps_vs_oracle(jit_from_14, n, S, zq):
    # specialised flip-group sweeps + interpreted Z-only sweeps
    rng = np.random.default_rng(500 + n)
    h = W.sparse_random_hamiltonian(n, S, rng, z_only=zq)
    st = random_state(n, rng)
    s = sv.from_amplitudes(st)
    _, before = jit_from_14.jit_info()
    re, im, per = sv.expectation_terms(s, h)
    _, after = jit_from_14.jit_info()
    assert after > before
    _, ref_per = O.expectation(st, h, n, per_term=True)
    assert np.abs(per - ref_per[:, 0]).max() <= 1e-12
    e_ref = O.expectation(st, h, n)
    assert rel(re, e_ref) <= REL_TOL


@pytest.mark.parametrize("case,n", [("ucc", 8), ("mixed", 7)])
def test_reverse_gradient_golden(case, n):
    """Device reverse-mode gradient (statevector.reverse_gradient) vs the
    reference's gradients (tests/golden/gradient_golden.npz)."""
    g = np.load(f"{__import__('conftest').GOLDEN}/gradient_golden.npz")
    circ = circuit_from_json(str(g[f"{case}_circuit"]))
    h = parse_h(g[f"{case}_h"])
    grad = sv.reverse_gradient(circ, g[f"{case}_theta"], h, sv.init_state(str(g[f"{case}_ref"])))
    assert np.abs(grad - g[f"{case}_grad"]).max() <= 1e-10


def test_reverse_gradient_ucc_vs_oracle_14q():
    from paper_2208_10978_b200.circuit import Affine, Circuit, evolution_gates
    n = 14
    rng = np.random.default_rng(8)
    strings = W.ucc_rotation_strings(n, 6)[:120]
    gates = []
    for k, s in enumerate(strings):
        gates.extend(evolution_gates(s, Affine(k, -0.5)))
    circ = Circuit(n, tuple(gates), len(strings))
    theta = rng.uniform(-0.2, 0.2, len(strings))
    h = W.sparse_random_hamiltonian(n, 80, rng)
    ref = W.hf_bitstring(6, n)
    grad = sv.reverse_gradient(circ, theta, h, sv.init_state(ref))
    grad_ref = O.reverse_gradient(circ, theta, h, O.init_state(ref), n)
    assert np.abs(grad - grad_ref).max() <= 1e-10


def test_sample_golden_and_outcomes():
    """Device shot sampling: same estimates as the reference (golden) and the
    same drawn outcomes as the oracle (Philox stream reproduced on device)."""
    import ctypes

    from paper_2208_10978_b200 import _lib
    from paper_2208_10978_b200.pauli import PauliString

    g = np.load(f"{__import__('conftest').GOLDEN}/sample_golden.npz")
    for k in range(3):
        p = PauliString.from_label(str(g[f"c{k}_label"]))
        s = sv.from_amplitudes(g[f"c{k}_amps"])
        m = sv.sample(s, p, int(g[f"c{k}_shots"]), int(g[f"c{k}_seed"]))
        assert m == float(g[f"c{k}_mean"])
    # outcome-level parity on a Z string (no rotation) at 16 qubits
    rng = np.random.default_rng(3)
    st = random_state(16, rng)
    p = PauliString.from_label("Z0 Z5 Z15")
    mean_ref, out_ref = O.sample(st, p, 100000, 42, return_outcomes=True)
    key = np.ascontiguousarray(np.random.Philox(42).state["state"]["key"], dtype=np.uint64)
    outs = np.zeros(100000, dtype=np.int64)
    mean = ctypes.c_double()
    s = sv.from_amplitudes(st)
    _lib.check(_lib.lib().qsv_sample_parity(s.handle, (1 << 0) | (1 << 5) | (1 << 15), 100000,
                                            _lib.u64ptr(key), ctypes.byref(mean),
                                            outs.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    assert np.array_equal(outs, out_ref)
    assert mean.value == mean_ref


@pytest.mark.parametrize("jit", [False, True])
def test_config3_shaped_wide_groups_vs_oracle(jit, monkeypatch):
    """Config-3 construction at 16 qubits: 900 Z-only strings and 16 flip
    groups of 25-78 strings (X/Y on one qubit times Z patterns) -- the
    tile-wide Walsh-Hadamard path -- next to narrow groups (specialised
    sweeps when jit)."""
    if jit:
        monkeypatch.setenv("QSV_JIT_MIN_QUBITS", "14")
    n = 16
    h = W.config3_hamiltonian(seed=1, n_qubits=n, n_terms=3000)
    rng = np.random.default_rng(5)
    st = random_state(n, rng)
    s = sv.from_amplitudes(st)
    ref, per_ref = O.expectation(st, h, n, per_term=True)
    re, im, per = sv.expectation_terms(s, h)
    assert rel(re, ref) <= REL_TOL
    assert np.abs(per - per_ref[:, 0]).max() <= 1e-12
    # the same strings with coefficients changed: plan cache hit, same sweeps
    h2 = PauliSum(tuple(PauliTerm(2.0 * t.coefficient, t.string) for t in h.terms))
    assert rel(sv.expectation(s, h2), 2.0 * ref) <= REL_TOL


def test_download_async_snapshot_and_reuse():
    """download_async copies the state as of the call: work queued on the same
    state afterwards waits for the copy; other states run alongside."""
    n = 20
    rng = np.random.default_rng(21)
    circ = W.brickwork(n, 4, seed=3)
    st = random_state(n, rng)
    a = sv.from_amplitudes(st)
    ref_a = O.evolve(st, circ.gates)
    a2 = sv.evolve(a, circ)
    buf = np.empty(1 << n, dtype=np.complex128)
    a2.download_async(buf)
    sv.apply_circuit_inplace(a2, circ)      # modifies a2 right after: must wait for the copy
    b = sv.evolve(sv.init_state("0" * n), circ)  # independent work alongside
    a2.wait_download()
    assert np.abs(buf - ref_a).max() <= AMP_TOL
    assert np.abs(a2.amplitudes - O.evolve(ref_a, circ.gates)).max() <= AMP_TOL
    assert np.abs(b.amplitudes - O.evolve(O.init_state("0" * n), circ.gates)).max() <= AMP_TOL
    # dropping a state with a copy in flight: the pool waits before reuse
    bufs = [np.empty(1 << n, dtype=np.complex128) for _ in range(3)]
    for k in range(3):
        s = sv.evolve(sv.from_amplitudes(st), circ)
        s.download_async(bufs[k])
        del s
    for k in range(3):
        assert np.abs(bufs[k] - ref_a).max() <= AMP_TOL


@pytest.mark.parametrize("kernel", ["runs", "smem"])
@pytest.mark.parametrize("n,ne,count", [(10, 4, 200), (14, 6, 150)])
def test_rotation_adjoint_matches_general_path(monkeypatch, n, ne, count, kernel):
    """qsv_rotation_adjoint (one device sweep; shared-memory kernel at
    n <= 12, two launches per rotation above) vs the gate-level reverse
    sweep and the CPU oracle; shared parameters (several blocks on one
    theta, scale / offset) accumulate like the reference's per-gate loop."""
    from paper_2208_10978_b200.circuit import Affine, Circuit, evolution_gates

    rng = np.random.default_rng(n)
    strings = W.ucc_rotation_strings(n, ne)[:count]
    gates = []
    for k, s in enumerate(strings):
        gates.extend(evolution_gates(s, Affine(k % 60, -0.5 * (1 + (k % 3)), 0.01 * (k % 5))))
    circ = Circuit(n, tuple(gates), 60)
    assert sv._rotation_program(circ) is not None
    theta = rng.uniform(-0.3, 0.3, 60)
    h = W.sparse_random_hamiltonian(n, 60, rng, z_only=10)
    ref = W.hf_bitstring(ne, n)
    monkeypatch.setenv("QSV_ADJOINT", kernel)  # smem: single-CTA kernel (n <= 12 only)
    fast = sv.reverse_gradient(circ, theta, h, sv.init_state(ref))
    monkeypatch.setenv("QSV_ROTATION_ADJOINT", "0")
    slow = sv.reverse_gradient(circ, theta, h, sv.init_state(ref))
    assert np.abs(fast - slow).max() <= 1e-10
    grad_ref = O.reverse_gradient(circ, theta, h, O.init_state(ref), n)
    assert np.abs(fast - grad_ref).max() <= 1e-10


def test_jit_fast_path_repeated_angles(jit_from_14):
    """A specialised program re-run with new angles takes the fast path
    (cached geometry tables, OP_GMAT tables filled on the device): every run
    matches the oracle."""
    from paper_2208_10978_b200.circuit import bind

    n, ne = 16, 8
    strings = W.ucc_rotation_strings(n, ne)[:300]
    param = W.parametric_rotations_circuit(n, strings)
    ref = W.hf_bitstring(ne, n)
    rng = np.random.default_rng(5)
    for _ in range(3):
        theta = rng.uniform(-0.4, 0.4, len(strings))
        psi = sv.evolve(sv.init_state(ref), bind(param, theta))
        exp = O.evolve(O.init_state(ref), W.rotations_circuit(n, strings, theta).gates)
        assert np.abs(psi.amplitudes - exp).max() <= AMP_TOL


def test_ucc_mirror_24q_two_contiguous_bits():
    """24-qubit UCC-shaped circuit followed by its inverse returns to the HF
    state (1e-10): rotation-dominated programs at n >= 22 are planned with 2
    contiguous low qubits when that needs fewer HBM passes (pick_contig)."""
    from paper_2208_10978_b200 import _lib

    n, ne = 24, 12
    rng = np.random.default_rng(24)
    strings = W.ucc_rotation_strings(n, ne)[:400]
    theta = rng.uniform(-0.5, 0.5, len(strings))
    fwd = W.rotations_circuit(n, strings, theta)
    back = W.rotations_circuit(n, strings[::-1], -theta[::-1])
    circ = Circuit(n, fwd.gates + back.gates, 0)
    kinds, qubits, values = sv._flat(fwd)
    plan = _lib.debug_plan(n, kinds, qubits, values)
    assert min(p["c"] for p in plan["passes"] if not p["global"]) == 2  # (tiles may extend it)
    ref = W.hf_bitstring(ne, n)
    out = sv.evolve(sv.init_state(ref), circ).amplitudes
    expect = np.zeros(1 << n, dtype=np.complex128)
    expect[O.init_state(ref).argmax()] = 1.0
    assert np.abs(out - expect).max() <= AMP_TOL
