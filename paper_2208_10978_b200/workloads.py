"""Seeded synthetic workloads for BASELINE.json's five configs.

The reference publishes no dataset for this path; every config is synthetic.
Draws use numpy.random.default_rng(seed) (PCG64) in the order documented per
function, and circuits are returned as bound gate-level circuits in the
reference's own gate pattern (pauli_evolution blocks, circuit.py:254-281), so
the CPU oracle and the engine consume identical gates.

UCC strings come from a Jordan-Wigner restatement (fermion.py:336-363): a+_p
-> (X_p - iY_p)/2 Z_{<p}, a_p -> (X_p + iY_p)/2 Z_{<p}; T - T^dagger is
multiplied out, simplified and kept in canonical (sorted-factor) order.
"""

from __future__ import annotations

import itertools
import math

import numpy as np

from .circuit import Affine, Circuit, Constant, Gate, evolution_gates
from .pauli import PauliString, PauliSum, PauliTerm, multiply

# ---------------------------------------------------------------------------
# Jordan-Wigner of excitation generators
# ---------------------------------------------------------------------------


def _ladder(mode: int, creation: bool) -> list[tuple[complex, PauliString]]:
    chain = tuple((k, "Z") for k in range(mode))
    return [(0.5, PauliString(chain + ((mode, "X"),))),
            (-0.5j if creation else 0.5j, PauliString(chain + ((mode, "Y"),)))]


def _jw_product(ops: list[tuple[int, bool]]) -> dict[PauliString, complex]:
    acc: dict[PauliString, complex] = {PauliString(): 1.0}
    for mode, creation in ops:
        nxt: dict[PauliString, complex] = {}
        for s, c in acc.items():
            for cf, f in _ladder(mode, creation):
                ph, prod = multiply(s, f)
                nxt[prod] = nxt.get(prod, 0) + c * cf * ph
        acc = nxt
    return acc


def excitation_strings(create: tuple[int, ...], annihilate: tuple[int, ...]) -> list[tuple[complex, PauliString]]:
    """JW image of T - T^dagger with T = a+_{create...} a_{annihilate...}
    (operators applied right to left), simplified, canonical order."""
    t_ops = [(m, True) for m in create] + [(m, False) for m in annihilate]
    dag_ops = [(m, True) for m in reversed(annihilate)] + [(m, False) for m in reversed(create)]
    acc = _jw_product(t_ops)
    for s, c in _jw_product(dag_ops).items():
        acc[s] = acc.get(s, 0) - c
    kept = [(c, s) for s, c in acc.items() if abs(c) >= 1e-12]
    kept.sort(key=lambda cs: cs[1].factors)
    return kept


def ucc_rotation_strings(n_qubits: int, n_electrons: int, doubles=None) -> list[PauliString]:
    """Pauli strings of all singles (i in occ, a in vir, ascending) then the
    given doubles ((i, j), (a, b)) (default: all, itertools.combinations order)."""
    occ = range(n_electrons)
    vir = range(n_electrons, n_qubits)
    strings: list[PauliString] = []
    for i in occ:
        for a in vir:
            strings.extend(s for _, s in excitation_strings((a,), (i,)))
    if doubles is None:
        doubles = [(ij, ab) for ij in itertools.combinations(occ, 2)
                   for ab in itertools.combinations(vir, 2)]
    for (i, j), (a, b) in doubles:
        strings.extend(s for _, s in excitation_strings((a, b), (j, i)))
    return strings


def rotations_circuit(n_qubits: int, strings, thetas) -> Circuit:
    """Bound circuit of exp(-i theta/2 P) blocks = pauli_evolution(P, -theta/2)."""
    gates: list[Gate] = []
    for s, th in zip(strings, thetas):
        gates.extend(evolution_gates(s, Constant(-0.5 * float(th))))
    return Circuit(n_qubits, tuple(gates), 0)


def parametric_rotations_circuit(n_qubits: int, strings) -> Circuit:
    """The same blocks with theta_k as parameter k (Affine(k, -1/2)): what a
    VQE loop binds every iteration (bind(c, thetas) == rotations_circuit)."""
    gates: list[Gate] = []
    for k, s in enumerate(strings):
        gates.extend(evolution_gates(s, Affine(k, -0.5)))
    return Circuit(n_qubits, tuple(gates), len(strings))


def hf_bitstring(n_electrons: int, n_qubits: int) -> str:
    """Aufbau occupation; character k is qubit k (fermion.py:366-372)."""
    return "1" * n_electrons + "0" * (n_qubits - n_electrons)


# ---------------------------------------------------------------------------
# Hamiltonians
# ---------------------------------------------------------------------------


def dense_random_hamiltonian(n_qubits: int, n_terms: int, rng) -> PauliSum:
    """Config 1: each qubit uniform in {I,X,Y,Z}; c ~ N(0,1).
    Draw order: axes (n_terms x n_qubits integers in [0,4)), then coefficients."""
    axes = rng.integers(0, 4, size=(n_terms, n_qubits))
    coefs = rng.standard_normal(n_terms)
    terms = []
    for t in range(n_terms):
        f = tuple((q, "XYZ"[a - 1]) for q, a in enumerate(axes[t]) if a)
        terms.append(PauliTerm(float(coefs[t]), PauliString(f)))
    return PauliSum(tuple(terms))


def sparse_random_hamiltonian(n_qubits: int, n_terms: int, rng, z_only: int = 0,
                              require_flip: bool = True) -> PauliSum:
    """Configs 3/4: weight w ~ U{1..4}; positions without replacement; the
    first ``z_only`` strings are Z-only; the others draw axes uniformly from
    {X,Y,Z} (resampled until one is X/Y when require_flip); c ~ N(0,1).
    Draw order per term: w, positions, axes (repeat), coefficient."""
    terms = []
    for t in range(n_terms):
        w = int(rng.integers(1, 5))
        pos = rng.choice(n_qubits, size=w, replace=False)
        if t < z_only:
            axes = ["Z"] * w
        else:
            while True:
                axes = ["XYZ"[k] for k in rng.integers(0, 3, size=w)]
                if not require_flip or any(a != "Z" for a in axes):
                    break
        c = float(rng.standard_normal())
        terms.append(PauliTerm(c, PauliString(tuple(zip((int(p) for p in pos), axes)))))
    return PauliSum(tuple(terms))


# ---------------------------------------------------------------------------
# The five configs
# ---------------------------------------------------------------------------


def config1(seed: int = 0, n_qubits: int = 12, n_electrons: int = 6, n_terms: int = 500):
    """12q UCCSD-shaped ansatz (1,872 rotations) on |111111000000> + 500-term H.
    Draw order: one theta ~ U(-0.1, 0.1) per string, then the Hamiltonian."""
    rng = np.random.default_rng(seed)
    strings = ucc_rotation_strings(n_qubits, n_electrons)
    thetas = rng.uniform(-0.1, 0.1, size=len(strings))
    circ = rotations_circuit(n_qubits, strings, thetas)
    h = dense_random_hamiltonian(n_qubits, n_terms, rng)
    return {"n_qubits": n_qubits, "reference": hf_bitstring(n_electrons, n_qubits),
            "circuit": circ, "hamiltonian": h, "strings": strings, "thetas": thetas}


def brickwork(n_qubits: int, layers: int, seed: int = 0) -> Circuit:
    """Configs 2/5: per layer, U3(arccos(1-2u), phi, lam) on every qubit
    ascending (draws u, phi, lam per gate), then CNOT(q, q+1) for q = layer mod 2,
    layer mod 2 + 2, ...  Haar on SU(2) up to a global phase."""
    rng = np.random.default_rng(seed)
    gates: list[Gate] = []
    for layer in range(layers):
        for q in range(n_qubits):
            u, phi, lam = rng.random(), rng.uniform(0, 2 * math.pi), rng.uniform(0, 2 * math.pi)
            theta = math.acos(1.0 - 2.0 * u)
            gates.append(Gate("U3", (q,), (Constant(theta), Constant(phi), Constant(lam))))
        for q in range(layer % 2, n_qubits - 1, 2):
            gates.append(Gate("CNOT", (q, q + 1)))
    return Circuit(n_qubits, tuple(gates), 0)


def config2(seed: int = 0, n_qubits: int = 28, layers: int = 20):
    return {"n_qubits": n_qubits, "reference": "0" * n_qubits,
            "circuit": brickwork(n_qubits, layers, seed)}


def config3_hamiltonian(seed: int = 0, n_qubits: int = 30, n_terms: int = 10_000,
                        z_fraction: float = 0.3) -> PauliSum:
    rng = np.random.default_rng(seed + 1)
    return sparse_random_hamiltonian(n_qubits, n_terms, rng, z_only=int(round(z_fraction * n_terms)))


def config3_state(seed: int = 0, n_qubits: int = 30, chunk_bits: int = 24) -> np.ndarray:
    """N(0,1) + i N(0,1) amplitudes, drawn re-then-im per 2^chunk_bits chunk, normalised."""
    rng = np.random.default_rng(seed)
    n = 1 << n_qubits
    chunk = min(n, 1 << chunk_bits)
    out = np.empty(n, dtype=np.complex128)
    for k in range(0, n, chunk):
        out.real[k:k + chunk] = rng.standard_normal(chunk)
        out.imag[k:k + chunk] = rng.standard_normal(chunk)
    out /= np.linalg.norm(out)
    return out


def config4(seed: int = 0, n_qubits: int = 32, n_electrons: int = 16, n_doubles: int = 2000,
            n_terms: int = 5000):
    """32q UCC: all singles + n_doubles quadruples sampled without replacement
    (sampled order), theta ~ U(-0.05, 0.05) per string; H as config 3 without
    the Z-only quota (axes uniform, no resampling).
    Draw order: quadruple sample, thetas, Hamiltonian."""
    rng = np.random.default_rng(seed)
    occ = range(n_electrons)
    vir = range(n_electrons, n_qubits)
    quads = [(ij, ab) for ij in itertools.combinations(occ, 2) for ab in itertools.combinations(vir, 2)]
    pick = rng.choice(len(quads), size=min(n_doubles, len(quads)), replace=False)
    doubles = [quads[k] for k in pick]
    strings = ucc_rotation_strings(n_qubits, n_electrons, doubles)
    thetas = rng.uniform(-0.05, 0.05, size=len(strings))
    circ = rotations_circuit(n_qubits, strings, thetas)
    h = sparse_random_hamiltonian(n_qubits, n_terms, rng, z_only=0, require_flip=False)
    return {"n_qubits": n_qubits, "reference": hf_bitstring(n_electrons, n_qubits),
            "circuit": circ, "hamiltonian": h, "strings": strings, "thetas": thetas}


def config5(seed: int = 0, n_qubits: int = 36, layers: int = 10):
    return {"n_qubits": n_qubits, "reference": "0" * n_qubits,
            "circuit": brickwork(n_qubits, layers, seed)}


def string_masks(strings) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    xs, ys, zs = [], [], []
    for s in strings:
        x, y, z = s.masks()
        xs.append(x), ys.append(y), zs.append(z)
    return (np.array(xs, dtype=np.uint64), np.array(ys, dtype=np.uint64),
            np.array(zs, dtype=np.uint64))
