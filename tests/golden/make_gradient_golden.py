"""Golden reverse-mode gradients from the REFERENCE (vqekit.statevector.reverse_gradient).

    make -C oracle ref
    PYTHONPATH=oracle/_ref python tests/golden/make_gradient_golden.py

Cases: the reference's own UCCSD ansatz (circuit.uccsd_ansatz: Affine-parametrised
pauli_evolution blocks, RZ slots) on 4 spatial orbitals / 4 electrons (8 qubits),
and a random circuit with Affine-parametrised RY / U3 / CU3 / RZ gates, each
against a random sparse Hermitian H.  Writes tests/golden/gradient_golden.npz.
"""

import io
import os

import numpy as np

from vqekit import circuit as C
from vqekit import kernels as K
from vqekit import pauli as P
from vqekit import statevector as SV

assert K.IMPLEMENTATION == "cython", K.IMPLEMENTATION
HERE = os.path.dirname(os.path.abspath(__file__))


def sparse_h(n, n_terms, rng):
    terms = []
    for _ in range(n_terms):
        w = int(rng.integers(1, 5))
        pos = rng.choice(n, size=w, replace=False)
        axes = rng.choice(list("XYZ"), size=w)
        s = P.PauliString(tuple(sorted(zip((int(p) for p in pos), axes))))
        terms.append(P.PauliTerm(complex(rng.standard_normal()), s))
    return P.PauliSum(tuple(terms))


def text(h):
    buf = io.StringIO()
    P.write_pauli_sum(h, buf)
    return buf.getvalue()


def random_param_circuit(n, n_gates, n_params, rng):
    gates = []
    for _ in range(n_gates):
        k = ["H", "CNOT", "RZ", "RY", "U3", "CU3", "X"][rng.integers(7)]
        qs = tuple(int(q) for q in rng.choice(n, size=C.GATE_QUBITS[k], replace=False))
        ps = []
        for _ in range(C.GATE_PARAMS[k]):
            if rng.random() < 0.7:
                ps.append(C.Affine(int(rng.integers(n_params)), float(rng.uniform(0.5, 2.0)) * (1 if rng.random() < .5 else -1),
                                   float(rng.uniform(-1, 1))))
            else:
                ps.append(C.Constant(float(rng.uniform(-3, 3))))
        gates.append(C.Gate(k, qs, tuple(ps)))
    return C.Circuit(n, tuple(gates), n_params)


def main():
    rng = np.random.default_rng(2024)
    out = {}
    ucc = C.uccsd_ansatz(4, 4)
    n = ucc.n_qubits
    theta = rng.uniform(-0.3, 0.3, ucc.n_params)
    h = sparse_h(n, 60, rng)
    s0 = SV.init_state("1" * 4 + "0" * (n - 4))
    out["ucc_circuit"] = C.circuit_to_json(ucc)
    out["ucc_theta"] = theta
    out["ucc_h"] = text(h)
    out["ucc_ref"] = "1" * 4 + "0" * (n - 4)
    out["ucc_grad"] = SV.reverse_gradient(ucc, theta, h, s0)
    out["ucc_energy"] = SV.expectation(SV.evolve(s0, C.bind(ucc, theta)), h)

    rc = random_param_circuit(7, 60, 9, rng)
    theta = rng.uniform(-2, 2, rc.n_params)
    h = sparse_h(7, 40, rng)
    s0 = SV.init_state("0110100")
    out["mixed_circuit"] = C.circuit_to_json(rc)
    out["mixed_theta"] = theta
    out["mixed_h"] = text(h)
    out["mixed_ref"] = "0110100"
    out["mixed_grad"] = SV.reverse_gradient(rc, theta, h, s0)
    np.savez(os.path.join(HERE, "gradient_golden.npz"), **out)
    print("ucc params", len(out["ucc_theta"]), "mixed params", len(out["mixed_theta"]))


if __name__ == "__main__":
    main()
