"""Generate golden fixtures from the REFERENCE implementation (vqekit).

Run in the build container, where the reference exists:
    make -C oracle ref          # builds /root/reference/pkg into oracle/_ref
    PYTHONPATH=oracle/_ref python tests/golden/make_golden.py

Everything written here comes from calling the unmodified reference
(vqekit.statevector / vqekit.circuit / vqekit.fermion / vqekit.engine with
its Cython kernels).  The fixtures pin both the CPU oracle (oracle/) and the
CUDA engine; the GPU box never needs the reference itself.
"""

from __future__ import annotations

import io
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_FIXTURES = "/root/reference/pkg/tests/fixtures"

import vqekit  # noqa: E402  (the reference)
from vqekit import circuit as C  # noqa: E402
from vqekit import engine as E  # noqa: E402
from vqekit import fermion as F  # noqa: E402
from vqekit import pauli as P  # noqa: E402
from vqekit import statevector as SV  # noqa: E402
from vqekit import kernels as K  # noqa: E402

assert K.IMPLEMENTATION == "cython", K.IMPLEMENTATION


def _pauli_text(h) -> str:
    buf = io.StringIO()
    P.write_pauli_sum(h, buf)
    return buf.getvalue()


def random_state(n, rng):
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    return a / np.linalg.norm(a)


def random_mixed_circuit(n, n_gates, rng):
    kinds = ["H", "HY", "X", "CNOT", "SWAP", "RZ", "RY", "U3", "CU3"]
    gates = []
    for _ in range(n_gates):
        k = kinds[rng.integers(len(kinds))]
        nq = C.GATE_QUBITS[k]
        qs = tuple(int(q) for q in rng.choice(n, size=nq, replace=False))
        ps = tuple(C.Constant(float(v)) for v in rng.uniform(-np.pi, np.pi, size=C.GATE_PARAMS[k]))
        gates.append(C.Gate(k, qs, ps))
    return C.Circuit(n, tuple(gates), 0)


def random_sparse_h(n, n_terms, rng, with_identity=True):
    terms = []
    if with_identity:
        terms.append(P.PauliTerm(0.37, P.PauliString()))
    for t in range(n_terms):
        w = int(rng.integers(1, min(n, 6) + 1))
        pos = rng.choice(n, size=w, replace=False)
        axes = ["XYZ"[k] for k in rng.integers(0, 3, size=w)]
        if t % 4 == 0:
            axes = ["Z"] * w
        terms.append(P.PauliTerm(float(rng.standard_normal()),
                                 P.PauliString(tuple(zip((int(p) for p in pos), axes)))))
    return P.PauliSum(tuple(terms))


def main():
    out = {}
    rng = np.random.default_rng(20221978)

    # 1. mixed-gate circuits (every gate kind), amplitudes after evolve
    for n, g in [(5, 60), (9, 200)]:
        circ = random_mixed_circuit(n, g, rng)
        s0 = SV.StateVector(n, random_state(n, rng))
        s1 = SV.evolve(s0, circ)
        out[f"mixed_n{n}_circuit"] = np.array(C.circuit_to_json(circ))
        out[f"mixed_n{n}_in"] = s0.amplitudes
        out[f"mixed_n{n}_out"] = s1.amplitudes

    # 2. brickwork (config-2 family) at small n, from |0...0>
    for n, layers in [(6, 4), (10, 6)]:
        gates = []
        r2 = np.random.default_rng(n)
        for layer in range(layers):
            for q in range(n):
                u, ph, la = r2.random(), r2.uniform(0, 2 * np.pi), r2.uniform(0, 2 * np.pi)
                gates.append(C.Gate("U3", (q,), (C.Constant(float(np.arccos(1 - 2 * u))),
                                                 C.Constant(float(ph)), C.Constant(float(la)))))
            for q in range(layer % 2, n - 1, 2):
                gates.append(C.Gate("CNOT", (q, q + 1)))
        circ = C.Circuit(n, tuple(gates), 0)
        out[f"brick_n{n}_circuit"] = np.array(C.circuit_to_json(circ))
        out[f"brick_n{n}_out"] = SV.evolve(SV.init_state("0" * n), circ).amplitudes

    # 3. apply_pauli on a random 7-qubit state
    n = 7
    st = random_state(n, rng)
    masks = []
    outs = []
    for _ in range(12):
        sel = rng.integers(0, 4, size=n)
        x = sum(1 << q for q in range(n) if sel[q] == 1)
        y = sum(1 << q for q in range(n) if sel[q] == 2)
        z = sum(1 << q for q in range(n) if sel[q] == 3)
        o = np.empty_like(st)
        K.apply_pauli(st, x, y, z, o)
        masks.append((x, y, z))
        outs.append(o)
    out["pauli_in"] = st
    out["pauli_masks"] = np.array(masks, dtype=np.uint64)
    out["pauli_out"] = np.array(outs)

    # 4. expectation of a sparse Hamiltonian on a random 10-qubit state
    n = 10
    st = random_state(n, rng)
    h = random_sparse_h(n, 300, rng)
    s = SV.StateVector(n, st)
    out["expect_state"] = st
    out["expect_h"] = np.array(_pauli_text(h))
    out["expect_value"] = np.array(SV.expectation(s, h))
    per = []
    for term in h.terms:
        per.append(np.vdot(st, SV.apply_pauli_string(s, term.string).amplitudes))
    out["expect_per_term"] = np.array(per)
    out["apply_operator_out"] = SV.apply_operator(s, h).amplitudes

    # 5. reference UCCSD ansatz (4 spatial orbitals, 4 electrons = 8 qubits), bound at random theta
    ans = C.uccsd_ansatz(4, 4)
    theta = rng.uniform(-0.3, 0.3, size=ans.n_params)
    bound = C.bind(ans, theta)
    hf = F.hf_reference(4, 8)
    psi = SV.evolve(SV.init_state(hf), bound)
    h8 = random_sparse_h(8, 120, rng)
    out["uccsd8_circuit"] = np.array(C.circuit_to_json(bound))
    out["uccsd8_reference"] = np.array(hf)
    out["uccsd8_out"] = psi.amplitudes
    out["uccsd8_h"] = np.array(_pauli_text(h8))
    out["uccsd8_energy"] = np.array(SV.expectation(psi, h8))

    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **out)

    # 6. H2 / STO-3G fixtures: JW Hamiltonians, HF energies, VQE optimum
    with open(os.path.join(REF_FIXTURES, "reference.json")) as fh:
        refjson = json.load(fh)
    h2 = {}
    for name in sorted(refjson):
        with open(os.path.join(REF_FIXTURES, name)) as fh:
            integrals = F.load_fcidump(fh)
        ham = F.jordan_wigner(F.build_hamiltonian(integrals))
        ref = F.hf_reference(integrals.n_electrons, integrals.n_qubits)
        ansatz = C.uccsd_ansatz(integrals.n_spatial, integrals.n_electrons)
        backend = E.StateVectorBackend()
        res = E.vqe_minimize(ham, ansatz, ref, backend, E.OptimizerOptions(tol_e=1e-12, tol_g=1e-9))
        hf_e = SV.expectation(SV.init_state(ref), ham)
        h2[name] = {
            "hamiltonian": _pauli_text(ham),
            "reference": ref,
            "ansatz": C.circuit_to_json(ansatz),
            "theta_opt": [float(v) for v in res.theta],
            "hf_energy_ref": hf_e,
            "vqe_energy_ref": float(res.energy),
            "fixture_hf_energy": refjson[name]["hf_energy"],
            "fixture_fci_energy": refjson[name]["fci_energy"],
            "cnot_count": C.count_resources(ansatz).n_cnot,
        }
        print(name, hf_e - refjson[name]["hf_energy"], res.energy - refjson[name]["fci_energy"])
    with open(os.path.join(HERE, "h2_sto3g.json"), "w") as fh:
        json.dump(h2, fh, indent=1)

    # 7. config 1 (12q UCCSD-shaped, 1,872 rotations, 500-term H) computed by the reference.
    sys.path.insert(0, REPO)
    from paper_2208_10978_b200 import workloads as W  # generator only (pure Python IR)

    cfg = W.config1(seed=0)
    x, y, z = W.string_masks(cfg["strings"])
    # rebuild the identical gate list with reference objects
    rgates = []
    for g in cfg["circuit"].gates:
        rgates.append(C.Gate(g.kind, g.qubits, tuple(C.Constant(p.value) for p in g.params)))
    rcirc = C.Circuit(12, tuple(rgates), 0)
    psi = SV.evolve(SV.init_state(cfg["reference"]), rcirc)
    rh = P.PauliSum(tuple(P.PauliTerm(t.coefficient, P.PauliString(t.string.factors))
                          for t in cfg["hamiltonian"].terms))
    energy = SV.expectation(psi, rh)
    np.savez_compressed(os.path.join(HERE, "config1_seed0.npz"), x=x, y=y, z=z,
                        thetas=cfg["thetas"], n_gates=np.array(len(rgates)), amplitudes=psi.amplitudes,
                        energy=np.array(energy), h=np.array(_pauli_text(rh)))
    print("config1 energy", energy, "gates", len(rgates))


if __name__ == "__main__":
    main()
