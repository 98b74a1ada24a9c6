"""Index-parity reduction (symmetry.py) checked on the CPU oracle.

An evolve from a basis state by an even-flip rotation program (UCC) keeps
the basis state's index-parity class; the half program on n-1 qubits,
embedded back, must equal the full oracle evolve (oracle.evolve, the
reference's gate loop statevector.py:65-74), and the Hamiltonian's
transformed even-flip terms must give the oracle energy.  The flat half
gate list must be exactly what circuit.evolution_gates emits for the
transformed strings (the planner re-matches it into rotations)."""

import numpy as np

from oracle import oracle as O
from paper_2208_10978_b200 import symmetry as S
from paper_2208_10978_b200 import workloads as W
from paper_2208_10978_b200.circuit import flatten_bound
from paper_2208_10978_b200.pauli import PauliString, PauliSum, PauliTerm, term_arrays


def strings_of(n, x, y, z):
    out = []
    for xs, ys, zs in zip(x.tolist(), y.tolist(), z.tolist()):
        f = []
        for q in range(n):
            if (xs >> q) & 1:
                f.append((q, "X"))
            elif (ys >> q) & 1:
                f.append((q, "Y"))
            elif (zs >> q) & 1:
                f.append((q, "Z"))
        out.append(PauliString(tuple(f)))
    return out


def embed(n, half, parity):
    full = np.zeros(1 << n, dtype=complex)
    top = 1 << (n - 1)
    for j in range(1 << n):
        if bin(j).count("1") & 1 == parity:
            full[j] = half[j & (top - 1)]
    return full


def test_parity_reduction_matches_oracle():
    rng = np.random.default_rng(8)
    for n, ne, ndbl in ((8, 4, 12), (9, 4, 20), (10, 5, 25)):
        occ, vir = range(ne), range(ne, n)
        import itertools

        quads = [(ij, ab) for ij in itertools.combinations(occ, 2) for ab in itertools.combinations(vir, 2)]
        pick = rng.choice(len(quads), size=min(ndbl, len(quads)), replace=False)
        strings = W.ucc_rotation_strings(n, ne, [quads[k] for k in pick])
        thetas = rng.uniform(-0.4, 0.4, len(strings))
        circ = W.rotations_circuit(n, strings, thetas)
        kinds, qubits, values = flatten_bound(circ)
        red = S.Reduction(n, kinds, qubits)
        for ref in (W.hf_bitstring(ne, n), "0110100101"[:n]):
            b = int(ref[::-1], 2)
            parity = bin(b).count("1") & 1
            hv = red.half_values(values, parity)
            # the half program as a circuit: same strings as the flat list
            half_strings = strings_of(n - 1, red.x2, red.y2, red.z2)
            th2 = hv[3 * red.rz_at]
            half_circ = W.rotations_circuit(n - 1, half_strings, th2)
            hk, hq, _ = flatten_bound(half_circ)
            assert np.array_equal(hk, red.kinds) and np.array_equal(hq, red.qubits)
            b_low = b & ((1 << (n - 1)) - 1)
            half = O.evolve(O.init_state(format(b_low, f"0{n - 1}b")[::-1]), half_circ.gates)
            full = O.evolve(O.init_state(ref), circ.gates)
            assert np.abs(embed(n, half, parity) - full).max() <= 1e-12
            # energy: transformed even-flip terms on the half
            h = W.sparse_random_hamiltonian(n, 60, rng, z_only=10, require_flip=False)
            x, y, z, cr, ci = term_arrays(h, n)
            x2, y2, z2, cr2, ci2, keep, sign = S.half_terms(n, x, y, z, cr, ci, parity)
            h2 = PauliSum(tuple(PauliTerm(complex(c), p) for c, p in zip(cr2 + 1j * ci2,
                                                                        strings_of(n - 1, x2, y2, z2))))
            e_half = O.expectation(half, h2, n - 1)
            e_full = O.expectation(full, h, n)
            assert abs(e_half - e_full) <= 1e-12 * max(1.0, abs(e_full))


def test_ineligible_programs():
    rng = np.random.default_rng(1)
    n = 9
    odd = [PauliString(((0, "X"),)), PauliString(((1, "Y"), (2, "X")))]
    circ = W.rotations_circuit(n, odd, rng.uniform(-1, 1, 2))
    k, q, _ = flatten_bound(circ)
    assert S.reduction_for(n, k, q) is None
    from paper_2208_10978_b200.circuit import Circuit, Constant, Gate

    ucc = W.rotations_circuit(n, W.ucc_rotation_strings(n, 4)[:10], rng.uniform(-1, 1, 10))
    mixed = Circuit(n, ucc.gates + (Gate("U3", (0,), (Constant(0.1), Constant(0.2), Constant(0.3))),), 0)
    k, q, _ = flatten_bound(mixed)
    assert S.reduction_for(n, k, q) is None
    k, q, _ = flatten_bound(ucc)
    assert S.reduction_for(n, k, q) is not None
