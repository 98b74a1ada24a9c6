"""Small-state rotation programs (csrc/qsv_small.cu) vs the oracle.

A program made only of Pauli rotations on <= 12 qubits -- config 1 -- runs as
one CTA with the state in shared memory, walking same-flip rotation groups
whose fused 2x2 matrices are selected per pair by phase-mask parities.  Every
case compares with the CPU oracle's gate loop (oracle.evolve, the reference's
statevector.py:65-74 over the decomposed blocks of circuit.py:271-281) and
with the tile-pass path (QSV_SMALL=0) on the same circuit.  Config 1's full
circuit is pinned to the reference's own output in test_gpu_parity.py
(test_config1_full, tests/golden).

Tolerance (north_star): amplitudes 1e-10 max-abs.
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2208_10978_b200 import _lib
from paper_2208_10978_b200 import statevector as sv
from paper_2208_10978_b200 import workloads as W
from paper_2208_10978_b200.pauli import PauliString

pytestmark = pytest.mark.gpu

AMP_TOL = 1e-10


def grouped_strings(n, n_groups, rng, per_group=(1, 9), weights=(1, 4)):
    """Runs of strings sharing a flip mask (X/Y positions) whose Y/Z patterns
    vary -- groups of up to 9 strings, so some need a fourth phase-difference
    dimension and split."""
    out = []
    for _ in range(n_groups):
        w = int(rng.integers(weights[0], min(weights[1], n) + 1))
        flip = rng.choice(n, size=w, replace=False)
        rest = [q for q in range(n) if q not in set(flip.tolist())]
        for _ in range(int(rng.integers(per_group[0], per_group[1] + 1))):
            axes = {int(q): "XY"[int(rng.integers(0, 2))] for q in flip}
            for q in rng.choice(rest, size=min(len(rest), int(rng.integers(0, 3))), replace=False) if rest else []:
                axes[int(q)] = "Z"
            out.append(PauliString(tuple(sorted(axes.items()))))
    return out


def run_both(circ, start, monkeypatch):
    before = _lib.small_launches()
    out = sv.evolve(start, circ).amplitudes
    ran_small = _lib.small_launches() - before
    monkeypatch.setenv("QSV_SMALL", "0")
    try:
        out_passes = sv.evolve(start, circ).amplitudes
    finally:
        monkeypatch.delenv("QSV_SMALL")
    return out, out_passes, ran_small


@pytest.mark.parametrize("n", [2, 5, 8, 10, 12])
def test_random_grouped_rotations_vs_oracle(n, monkeypatch):
    """8-12 qubits run small (below 8 the pair space is too small for four
    pairs per thread to share a matrix: tile passes)."""
    rng = np.random.default_rng(100 + n)
    strings = grouped_strings(n, 30, rng, weights=(1, 4))
    thetas = rng.uniform(-np.pi, np.pi, size=len(strings))
    circ = W.rotations_circuit(n, strings, thetas)
    bits = "".join("01"[int(b)] for b in rng.integers(0, 2, size=n))
    out, out_passes, ran = run_both(circ, sv.init_state(bits), monkeypatch)
    assert ran == (1 if n >= 8 else 0)
    ref = O.evolve(O.init_state(bits), circ.gates)
    assert np.abs(out - ref).max() <= AMP_TOL
    assert np.abs(out_passes - ref).max() <= AMP_TOL


def test_non_basis_input_state(monkeypatch):
    """Input read from device memory (not synthesised from a basis index)."""
    from conftest import random_state

    n = 10
    rng = np.random.default_rng(7)
    st = random_state(n, rng)
    strings = grouped_strings(n, 40, rng)
    circ = W.rotations_circuit(n, strings, rng.uniform(-2, 2, size=len(strings)))
    out, out_passes, ran = run_both(circ, sv.from_amplitudes(st), monkeypatch)
    assert ran == 1
    ref = O.evolve(st.copy(), circ.gates)
    assert np.abs(out - ref).max() <= AMP_TOL
    assert np.abs(out_passes - ref).max() <= AMP_TOL


def test_multiple_chunks_and_ucc_shape(monkeypatch):
    """> 80 groups and > 2048 rotations: several shared-memory chunks; the
    UCC construction at 10 q (5 electrons) besides."""
    n = 9
    rng = np.random.default_rng(11)
    strings = grouped_strings(n, 420, rng, per_group=(4, 9))
    assert len(strings) > 2048
    circ = W.rotations_circuit(n, strings, rng.uniform(-1, 1, size=len(strings)))
    out, out_passes, ran = run_both(circ, sv.init_state("0" * n), monkeypatch)
    assert ran == 1
    ref = O.evolve(O.init_state("0" * n), circ.gates)
    assert np.abs(out - ref).max() <= AMP_TOL
    assert np.abs(out_passes - ref).max() <= AMP_TOL
    cfg = W.config1(seed=3, n_qubits=10, n_electrons=5, n_terms=50)
    out, out_passes, ran = run_both(cfg["circuit"], sv.init_state(cfg["reference"]), monkeypatch)
    assert ran == 1
    ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    assert np.abs(out - ref).max() <= AMP_TOL
    assert np.abs(out_passes - ref).max() <= AMP_TOL


def test_config1_runs_small_and_matches_passes(monkeypatch):
    cfg = W.config1(seed=0)
    out, out_passes, ran = run_both(cfg["circuit"], sv.init_state(cfg["reference"]), monkeypatch)
    assert ran == 1
    assert np.abs(out - out_passes).max() <= AMP_TOL
    # prepared-program path (a VQE loop's bind + evolve) takes it too
    from paper_2208_10978_b200.circuit import bind

    param = W.parametric_rotations_circuit(12, cfg["strings"])
    before = _lib.small_launches()
    psi = sv.evolve(sv.init_state(cfg["reference"]), bind(param, cfg["thetas"]))
    psi = sv.evolve(sv.init_state(cfg["reference"]), bind(param, cfg["thetas"]))
    assert _lib.small_launches() - before == 2
    assert np.abs(psi.amplitudes - out).max() <= 1e-12


def test_ineligible_programs_use_passes():
    """Mixed gates, diagonal strings or more than 12 qubits: tile passes."""
    from paper_2208_10978_b200.circuit import Circuit, Constant, Gate

    rng = np.random.default_rng(5)
    n = 8
    strings = grouped_strings(n, 10, rng)
    base = W.rotations_circuit(n, strings, rng.uniform(-1, 1, size=len(strings)))
    mixed = Circuit(n, base.gates + (Gate("U3", (0,), (Constant(0.3), Constant(0.2), Constant(0.1))),), 0)
    diag = W.rotations_circuit(n, [PauliString(((1, "Z"), (4, "Z")))] + strings,
                               rng.uniform(-1, 1, size=len(strings) + 1))
    for circ in (mixed, diag):
        before = _lib.small_launches()
        out = sv.evolve(sv.init_state("0" * n), circ).amplitudes
        assert _lib.small_launches() == before
        ref = O.evolve(O.init_state("0" * n), circ.gates)
        assert np.abs(out - ref).max() <= AMP_TOL
    n = 13
    strings = grouped_strings(n, 10, rng)
    circ = W.rotations_circuit(n, strings, rng.uniform(-1, 1, size=len(strings)))
    before = _lib.small_launches()
    out = sv.evolve(sv.init_state("0" * n), circ).amplitudes
    assert _lib.small_launches() == before
    assert np.abs(out - O.evolve(O.init_state("0" * n), circ.gates)).max() <= AMP_TOL


def test_full_chunk_single_group(monkeypatch):
    """One same-flip group of exactly 2048 rotations: a whole chunk's angle
    table (the largest a small program takes)."""
    n = 9
    rng = np.random.default_rng(13)
    one = PauliString(((0, "X"), (1, "Y"), (2, "Z"), (7, "Y")))
    circ = W.rotations_circuit(n, [one] * 2048, rng.uniform(-0.01, 0.01, 2048))
    out, out_passes, ran = run_both(circ, sv.init_state("101000000"), monkeypatch)
    assert ran == 1
    ref = O.evolve(O.init_state("101000000"), circ.gates)
    assert np.abs(out - ref).max() <= AMP_TOL
    assert np.abs(out_passes - ref).max() <= AMP_TOL


def test_non_finite_angle_rejected_on_small_path():
    """The small-program path reads only the rotation angles of the gate list,
    and a non-finite angle fails loudly (QSV_ERR_INVALID) instead of running."""
    from paper_2208_10978_b200.circuit import bind

    strings = W.ucc_rotation_strings(10, 5)[:40]
    param = W.parametric_rotations_circuit(10, strings)
    b = bind(param, np.full(len(strings), 0.1))
    pid = b._plan.program_id()
    k, q, vals = b.flat()
    spans, _ = _lib.match_rotations(10, k, q)
    s10 = sv.init_state("1111100000")
    L = _lib.lib()
    vals = vals.copy()
    before = _lib.small_launches()
    assert L.qsv_evolve_basis_prepared(s10.handle, 31, pid, _lib.dptr(vals), None) == 0
    assert _lib.small_launches() == before + 1
    vals[3 * int(spans[5][2])] = np.inf  # the angle of rotation 5
    assert L.qsv_evolve_basis_prepared(s10.handle, 31, pid, _lib.dptr(vals), None) != 0
    assert b"non-finite" in L.qsv_last_error()


@pytest.mark.parametrize("n", [1, 6, 10, 12])
def test_small_state_expectation_vs_oracle_and_sweeps(n, monkeypatch):
    """States of <= 12 qubits take the one-launch expectation (a warp per
    string, qsv_small.cu: expect_small_kernel): per-term <P_t> (every axis
    mix, so all four i^ny phases) equal the CPU oracle's and the general
    sweep path's (QSV_SMALL_EXPECT=0) on a random state.  Tolerance:
    relative 1e-10 on the energy, 1e-12 absolute per term."""
    rng = np.random.default_rng(n)
    amps = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    amps /= np.linalg.norm(amps)
    h = W.dense_random_hamiltonian(n, 300, rng)
    s = sv.StateVector(n, amps)
    re, im, per = sv.expectation_terms(s, h)
    e_ref, per_ref = O.expectation(amps, h, n, per_term=True)
    assert abs(re - e_ref) <= 1e-10 * max(1.0, abs(e_ref))
    assert np.abs(per - per_ref[:, 0]).max() <= 1e-12
    monkeypatch.setenv("QSV_SMALL_EXPECT", "0")
    re2, _, per2 = sv.expectation_terms(s, h)
    assert np.abs(per - per2).max() <= 1e-12 and abs(re - re2) <= 1e-10 * max(1.0, abs(re))
