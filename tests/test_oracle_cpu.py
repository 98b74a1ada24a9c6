"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py) and the reference's own H2 fixtures
(pkg/tests/fixtures/reference.json, copied into h2_sto3g.json)."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, parse_h, random_state
from oracle import oracle as O
from paper_2208_10978_b200.circuit import bind, circuit_from_json


@pytest.mark.parametrize("n", [5, 9])
def test_oracle_mixed_circuits(golden, n):
    circ = circuit_from_json(str(golden[f"mixed_n{n}_circuit"]))
    out = O.evolve(golden[f"mixed_n{n}_in"], circ.gates)
    assert np.abs(out - golden[f"mixed_n{n}_out"]).max() <= 1e-14


@pytest.mark.parametrize("n", [6, 10])
def test_oracle_brickwork(golden, n):
    circ = circuit_from_json(str(golden[f"brick_n{n}_circuit"]))
    out = O.evolve(O.init_state("0" * n), circ.gates)
    assert np.abs(out - golden[f"brick_n{n}_out"]).max() <= 1e-14


def test_oracle_apply_pauli(golden):
    st = golden["pauli_in"]
    for (x, y, z), ref in zip(golden["pauli_masks"], golden["pauli_out"]):
        out = np.empty_like(st)
        O.apply_pauli(st, int(x), int(y), int(z), out)
        assert np.array_equal(out, ref)
        out2 = np.empty_like(st)
        O.np_apply_pauli(st, int(x), int(y), int(z), out2)
        assert np.abs(out2 - ref).max() <= 1e-15


def test_oracle_expectation(golden):
    st = golden["expect_state"]
    h = parse_h(golden["expect_h"])
    val, per = O.expectation(st, h, 10, per_term=True)
    assert abs(val - float(golden["expect_value"])) <= 1e-13
    ref = golden["expect_per_term"]
    assert np.abs(per[:, 0] + 1j * per[:, 1] - ref).max() <= 1e-14
    out = O.apply_operator(st, h, 10)
    assert np.abs(out - golden["apply_operator_out"]).max() <= 1e-13


def test_oracle_uccsd8(golden):
    circ = circuit_from_json(str(golden["uccsd8_circuit"]))
    psi = O.evolve(O.init_state(str(golden["uccsd8_reference"])), circ.gates)
    assert np.abs(psi - golden["uccsd8_out"]).max() <= 1e-14
    e = O.expectation(psi, parse_h(golden["uccsd8_h"]), 8)
    assert abs(e - float(golden["uccsd8_energy"])) <= 1e-13


def test_oracle_h2_fixture_energies(h2_fixtures):
    for name, fx in h2_fixtures.items():
        h = parse_h(fx["hamiltonian"])
        hf = O.init_state(fx["reference"])
        e_hf = O.expectation(hf, h, 4)
        assert abs(e_hf - fx["fixture_hf_energy"]) <= 1e-12, name
        ansatz = circuit_from_json(fx["ansatz"])
        assert sum(g.kind == "CNOT" for g in ansatz.gates) == 64  # Table 1 H2 row
        assert ansatz.n_params == 2
        psi = O.evolve(hf, bind(ansatz, fx["theta_opt"]).gates)
        e = O.expectation(psi, h, 4)
        assert abs(e - fx["fixture_fci_energy"]) <= 1e-10, name


def test_oracle_config1(config1_golden):
    from paper_2208_10978_b200 import workloads as W

    cfg = W.config1(seed=0)
    x, y, z = W.string_masks(cfg["strings"])
    assert np.array_equal(x, config1_golden["x"]) and np.array_equal(y, config1_golden["y"])
    assert np.array_equal(z, config1_golden["z"])
    assert np.array_equal(cfg["thetas"], config1_golden["thetas"])
    assert len(cfg["circuit"].gates) == int(config1_golden["n_gates"])
    psi = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    assert np.abs(psi - config1_golden["amplitudes"]).max() <= 1e-13
    e = O.expectation(psi, cfg["hamiltonian"], 12)
    assert abs(e - float(config1_golden["energy"])) <= 1e-12 * max(1.0, abs(e))


def test_numpy_twins_match_c_oracle():
    rng = np.random.default_rng(5)
    n = 8
    st = random_state(n, rng)
    m1 = O.gate_matrix("U3", (0.3, 1.2, -0.7))
    m2 = O.gate_matrix("CU3", (1.3, -0.2, 0.4))
    for q in range(n):
        a, b = st.copy(), st.copy()
        O.apply_1q(a, m1, q)
        O.np_apply_1q(b, m1, q)
        assert np.abs(a - b).max() <= 1e-15
    for q0, q1 in [(0, 1), (5, 2), (7, 0), (3, 6)]:
        a, b = st.copy(), st.copy()
        O.apply_2q(a, m2, q0, q1)
        O.np_apply_2q(b, m2, q0, q1)
        assert np.abs(a - b).max() <= 1e-15


@pytest.mark.parametrize("case,n", [("ucc", 8), ("mixed", 7)])
def test_oracle_reverse_gradient_golden(case, n):
    """oracle.reverse_gradient (restating statevector.py:153-211) vs the
    reference's own gradients (tests/golden/make_gradient_golden.py)."""
    from conftest import parse_h
    from paper_2208_10978_b200.circuit import circuit_from_json

    g = np.load(os.path.join(GOLDEN, "gradient_golden.npz"))
    circ = circuit_from_json(str(g[f"{case}_circuit"]))
    h = parse_h(g[f"{case}_h"])
    s0 = O.init_state(str(g[f"{case}_ref"]))
    grad = O.reverse_gradient(circ, g[f"{case}_theta"], h, s0, n)
    assert np.abs(grad - g[f"{case}_grad"]).max() <= 1e-12


def test_oracle_sample_golden():
    """oracle.sample (statevector.py:124-147) reproduces the reference's own
    shot estimates (tests/golden/make_sample_golden.py) exactly."""
    from paper_2208_10978_b200.pauli import PauliString

    g = np.load(os.path.join(GOLDEN, "sample_golden.npz"))
    for k in range(3):
        p = PauliString.from_label(str(g[f"c{k}_label"]))
        m = O.sample(g[f"c{k}_amps"], p, int(g[f"c{k}_shots"]), int(g[f"c{k}_seed"]))
        assert m == float(g[f"c{k}_mean"])
