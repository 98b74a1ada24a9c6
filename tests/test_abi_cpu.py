"""The C-ABI library loads without a GPU and exports every symbol that
include/qsv.h declares; the native planner (no device work) is exercised on
the BASELINE configs."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO
import sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from paper_2208_10978_b200 import _lib
from paper_2208_10978_b200 import workloads as W
from paper_2208_10978_b200.circuit import Circuit, Constant, Gate, evolution_gates, flatten_bound
from paper_2208_10978_b200.pauli import PauliString, term_arrays


def header_symbols():
    text = open(os.path.join(REPO, "include", "qsv.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(qsv_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert L.qsv_abi_version() == 1


def plan(circ):
    k, q, _ = flatten_bound(circ)
    st = _lib.PlanStats()
    _lib.check(_lib.lib().qsv_plan_gates(circ.n_qubits, len(k), _lib.i32ptr(k), _lib.i32ptr(q),
                                         ctypes.byref(st)))
    return st.as_dict()


def test_planner_config1_tile_passes():
    st = plan(W.config1()["circuit"])
    assert st["n_input_ops"] == 37824
    assert st["n_rotations"] == 1872
    assert st["n_items"] == 261  # same-flip groups
    # 12 qubits = one shared-memory tile; passes split only by the 8192-double
    # parameter budget of a specialised pass (64 KiB __constant__)
    assert st["n_passes"] == 4


def test_planner_config2_fuses_brickwork():
    st = plan(W.config2()["circuit"])
    assert st["n_input_ops"] == 830
    assert st["n_rotations"] == 0
    assert st["n_passes"] <= 60


def test_pattern_matcher_recognises_every_block():
    rng = np.random.default_rng(0)
    n = 20
    gates = []
    for _ in range(50):
        w = int(rng.integers(1, 8))
        pos = rng.choice(n, size=w, replace=False)
        axes = rng.choice(list("XYZ"), size=w)
        s = PauliString(tuple(zip((int(p) for p in pos), axes)))
        gates.extend(evolution_gates(s, Constant(float(rng.uniform(-1, 1)))))
        if rng.random() < 0.3:  # a stray gate between blocks must stay a gate
            gates.append(Gate("H", (int(rng.integers(n)),)))
    st = plan(Circuit(n, tuple(gates), 0))
    assert st["n_rotations"] == 50


def test_planner_rejects_bad_gates():
    k = np.array([3], dtype=np.int32)
    q = np.array([2, 2], dtype=np.int32)
    st = _lib.PlanStats()
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().qsv_plan_gates(4, 1, _lib.i32ptr(k), _lib.i32ptr(q), ctypes.byref(st)))
    q = np.array([1, 7], dtype=np.int32)
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().qsv_plan_gates(4, 1, _lib.i32ptr(k), _lib.i32ptr(q), ctypes.byref(st)))


def test_expectation_planner_config3():
    h = W.config3_hamiltonian()
    x, y, z, _, _ = term_arrays(h, 30)
    st = _lib.PlanStats()
    _lib.check(_lib.lib().qsv_plan_expectation(30, len(x), _lib.u64ptr(x), _lib.u64ptr(y),
                                               _lib.u64ptr(z), ctypes.byref(st)))
    assert st.n_fallback == 0
    assert 1 <= st.n_passes <= 300
    # a flip wider than a tile needs the global fallback sweep
    x2 = np.array([(1 << 20) - 1], dtype=np.uint64)
    zz = np.zeros(1, dtype=np.uint64)
    _lib.check(_lib.lib().qsv_plan_expectation(30, 1, _lib.u64ptr(x2), _lib.u64ptr(zz),
                                               _lib.u64ptr(zz), ctypes.byref(st)))
    assert st.n_fallback == 1


def test_no_gpu_compute_fails_loudly():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    with pytest.raises(_lib.QsvCudaError):
        _lib.check(_lib.lib().qsv_create(ctypes.byref(h), 4, 0))


# ---- planner + encoding checked on CPU through the kernel emulator ----

def _emulate(circ, psi0):
    import emulator
    k, q, v = flatten_bound(circ)
    prog = _lib.debug_plan(circ.n_qubits, k, q, v)
    return emulator.run_program(prog, psi0), prog


@pytest.mark.parametrize("n,layers", [(9, 5), (14, 4), (20, 6)])
def test_emulated_brickwork_matches_oracle(n, layers):
    from oracle import oracle as O
    circ = W.brickwork(n, layers, seed=5)
    psi0 = O.init_state("0" * n)
    out, prog = _emulate(circ, psi0)
    assert np.abs(out - O.evolve(psi0, circ.gates)).max() <= 1e-12


@pytest.mark.parametrize("n", [6, 13, 16])
def test_emulated_mixed_and_rotations_match_oracle(n):
    from oracle import oracle as O
    rng = np.random.default_rng(n)
    kinds = ["H", "HY", "X", "CNOT", "SWAP", "RZ", "RY", "U3", "CU3"]
    gates = []
    for _ in range(150):
        kd = kinds[rng.integers(len(kinds))]
        nq = 2 if kd in ("CNOT", "SWAP", "CU3") else 1
        qs = tuple(int(x) for x in rng.choice(n, size=nq, replace=False))
        npar = {"RZ": 1, "RY": 1, "U3": 3, "CU3": 3}.get(kd, 0)
        gates.append(Gate(kd, qs, tuple(Constant(float(x)) for x in rng.uniform(-3, 3, size=npar))))
        if rng.random() < 0.3:
            w = int(rng.integers(1, min(n, 7) + 1))
            pos = rng.choice(n, size=w, replace=False)
            s = PauliString(tuple(zip((int(p) for p in pos), rng.choice(list("XYZ"), size=w))))
            gates.extend(evolution_gates(s, Constant(float(rng.uniform(-1, 1)))))
    circ = Circuit(n, tuple(gates), 0)
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    psi0 = a / np.linalg.norm(a)
    out, _ = _emulate(circ, psi0)
    assert np.abs(out - O.evolve(psi0, circ.gates)).max() <= 1e-12


@pytest.mark.parametrize("n,ne,ndoubles", [(8, 4, None), (14, 6, 40)])
def test_emulated_ucc_groups_match_oracle(n, ne, ndoubles):
    """Same-flip UCC groups take the fused 2x2-table path (OP_GMAT)."""
    import itertools

    from oracle import oracle as O
    occ, vir = range(ne), range(ne, n)
    doubles = [(ij, ab) for ij in itertools.combinations(occ, 2) for ab in itertools.combinations(vir, 2)]
    if ndoubles is not None:
        rng = np.random.default_rng(1)
        doubles = [doubles[k] for k in rng.choice(len(doubles), size=ndoubles, replace=False)]
    strings = W.ucc_rotation_strings(n, ne, doubles)
    thetas = np.random.default_rng(2).uniform(-0.3, 0.3, size=len(strings))
    circ = W.rotations_circuit(n, strings, thetas)
    psi0 = O.init_state(W.hf_bitstring(ne, n))
    out, prog = _emulate(circ, psi0)
    assert any(op[0] == 9 for op in prog["ops"])  # fused groups present
    assert np.abs(out - O.evolve(psi0, circ.gates)).max() <= 1e-12


def test_pattern_matcher_relabelled_qubits():
    """A pauli_evolution block whose qubits were relabelled (non-ascending
    order, as in a shard's remapped segment) is still one direct rotation."""
    rng = np.random.default_rng(1)
    n = 16
    perm = rng.permutation(n)
    gates = []
    for _ in range(30):
        w = int(rng.integers(2, 7))
        pos = rng.choice(n, size=w, replace=False)
        axes = rng.choice(list("XYZ"), size=w)
        s = PauliString(tuple(zip((int(p) for p in pos), axes)))
        for g in evolution_gates(s, Constant(float(rng.uniform(-1, 1)))):
            gates.append(Gate(g.kind, tuple(int(perm[q]) for q in g.qubits), g.params))
    st = plan(Circuit(n, tuple(gates), 0))
    assert st["n_rotations"] == 30


@pytest.mark.parametrize("seed", [0, 1])
def test_emulated_relabelled_rotations_match_oracle(seed):
    from oracle import oracle as O

    rng = np.random.default_rng(40 + seed)
    n = 13
    perm = rng.permutation(n)
    gates = []
    for _ in range(40):
        w = int(rng.integers(1, 6))
        pos = rng.choice(n, size=w, replace=False)
        axes = rng.choice(list("XYZ"), size=w)
        s = PauliString(tuple(zip((int(p) for p in pos), axes)))
        for g in evolution_gates(s, Constant(float(rng.uniform(-1, 1)))):
            gates.append(Gate(g.kind, tuple(int(perm[q]) for q in g.qubits), g.params))
    circ = Circuit(n, tuple(gates), 0)
    a = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    st = a / np.linalg.norm(a)
    out, prog = _emulate(circ, st)
    assert np.abs(out - O.evolve(st, circ.gates)).max() <= 1e-12


def test_prepared_programs_host_side():
    """qsv_prepare_gates validates and plans on the host (no GPU needed);
    bind() results carry the plan whose program id the engine runs."""
    import ctypes

    from paper_2208_10978_b200 import _lib
    from paper_2208_10978_b200.circuit import bind

    strings = W.ucc_rotation_strings(8, 4)[:20]
    param = W.parametric_rotations_circuit(8, strings)
    b = bind(param, np.linspace(-0.1, 0.1, len(strings)))
    pid = b._plan.program_id()
    assert pid > 0 and b._plan.program_id() == pid  # prepared once
    bad = ctypes.c_int64()
    k = np.array([3], dtype=np.int32)            # CNOT with equal qubits
    q = np.array([1, 1], dtype=np.int32)
    rc = _lib.lib().qsv_prepare_gates(8, 1, _lib.i32ptr(k), _lib.i32ptr(q), ctypes.byref(bad))
    assert rc != 0 and bad.value == 0
    assert _lib.lib().qsv_release_program(pid) == 0
    b._plan._pid = None  # released above; a later use prepares again


def test_specialised_pass_sources_host_side():
    """The NVRTC sources are generated on the host: config 1's single-tile
    passes are straight-line by default and the compact data-driven block loop
    on request (QSV_COMPACT_GMAT=1); config 2's passes are straight-line;
    sweeps are specialised pair-bit sweeps."""
    import os

    cfg = W.config1(seed=0)
    k, q, _ = flatten_bound(cfg["circuit"])
    src0, npass = _lib.debug_pass_source(12, k, q, 0)
    assert npass >= 1 and "gm<" in src0 and "gm_run(a, tid, base" not in src0  # default: straight-line
    os.environ["QSV_COMPACT_GMAT"] = "1"
    try:
        src, _ = _lib.debug_pass_source(12, k, q, 0)
    finally:
        del os.environ["QSV_COMPACT_GMAT"]
    assert "gm_run(a, tid, base" in src and "__device__ const unsigned BD[" in src
    circ = W.brickwork(28, 4, seed=0)
    k2, q2, _ = flatten_bound(circ)
    src2, _ = _lib.debug_pass_source(28, k2, q2, 0)
    assert src2 and "gm_run(" not in src2.split("apply_tile")[-1] and "u1<" in src2
    from paper_2208_10978_b200.pauli import term_arrays

    h = W.sparse_random_hamiltonian(20, 200, np.random.default_rng(3), z_only=0)
    x, y, z, _, _ = term_arrays(h, 20)
    s3, nsw = _lib.debug_sweep_source(20, x, y, z, 0)
    assert nsw >= 1 and "qsv_sweep" in s3


def test_emulated_singular_u3_angles_take_the_plain_plan():
    """U3 angles whose cos(theta/2) vanishes (theta = pi: an X-like gate) or is
    tiny cannot take the normalised U3 forms (row 0 divided by cos(theta/2));
    the call is planned without them (set_plain_u3) and stays exact."""
    import emulator
    from oracle import oracle as O
    from paper_2208_10978_b200.circuit import Circuit, Constant, Gate

    n = 12
    base = W.brickwork(n, 6, seed=8)
    gates = list(base.gates)
    for i, g in enumerate(gates):  # a few U3s at theta = pi and pi - 1e-6
        if g.kind == "U3" and i % 7 == 3:
            th = np.pi if i % 2 else np.pi - 1e-6
            gates[i] = Gate("U3", g.qubits, (Constant(th),) + tuple(g.params[1:]))
    circ = Circuit(n, tuple(gates), 0)
    k, q, v = flatten_bound(circ)
    prog = _lib.debug_plan(n, k, q, v)
    psi0 = O.init_state("0" * n)
    out = emulator.run_program(prog, psi0)
    assert np.all(np.isfinite(out))
    assert np.abs(out - O.evolve(psi0, circ.gates)).max() <= 1e-12


def test_gate_pass_blocks_bank_conflict_free():
    """Every register block of config 2's plan puts three thread columns with
    independent 16-B granule vectors on lane bits 0-2, so its 128-bit LDS/STS
    are conflict-free (a block whose W-bit placement would leave rank 2 gives
    it up; ncu showed 2-way conflicts on two such blocks before)."""
    circ = W.brickwork(28, 20, seed=0)
    k, q, v = flatten_bound(circ)
    plan = _lib.debug_plan(28, k, q, v)

    def rank(vs):
        basis = []
        for x in vs:
            x &= 7
            for b in basis:
                x = min(x, x ^ b)
            if x:
                basis.append(x)
                basis.sort(reverse=True)
        return len(basis)

    blocks = [b for p in plan["passes"] for b in p.get("blocks", []) if b["kind"] == 0]
    assert len(blocks) > 100
    assert all(rank(b["cols"][:3]) == 3 for b in blocks)


def test_small_program_grouping_host_side():
    """Small-state rotation programs (csrc/qsv_small.cu) are built on the
    host: config 1 is 261 same-flip groups (36 singles of 2 strings, 225
    doubles of 8) in warp runs of <= 48 groups; mixed gates, diagonal strings,
    fewer than 8 or more than 12 qubits leave no small program (tile passes)."""
    import collections

    from paper_2208_10978_b200.circuit import Circuit, Constant, Gate
    from paper_2208_10978_b200.pauli import PauliString

    cfg = W.config1(seed=0)
    k, q, v = flatten_bound(cfg["circuit"])
    sm = _lib.debug_plan(12, k, q, v)["small"]
    assert sm["valid"] == 1 and len(sm["groups"]) == 261
    assert collections.Counter(g[2] - g[1] for g in sm["groups"]) == {8: 225, 2: 36}
    runs = sm["runs"]  # warp runs: contiguous, each <= 48 groups (one CTA barrier each)
    assert runs[0] == 0 and runs[-1] == 261 and all(runs[i] == runs[i + 1] for i in range(1, len(runs) - 1, 2))
    assert all(0 < runs[i + 1] - runs[i] <= 48 for i in range(0, len(runs), 2)) and len(runs) // 2 <= 30
    assert all(g[3] <= 3 for g in sm["groups"])  # <= 8 sign-pattern configs per group
    rng = np.random.default_rng(2)
    strings = W.ucc_rotation_strings(10, 5)[:60]
    base = W.rotations_circuit(10, strings, rng.uniform(-1, 1, len(strings)))

    def small_valid(circ, n):
        kk, qq, vv = flatten_bound(circ)
        return _lib.debug_plan(n, kk, qq, vv)["small"]["valid"]

    assert small_valid(base, 10) == 1
    mixed = Circuit(10, base.gates + (Gate("U3", (0,), (Constant(0.3), Constant(0.2), Constant(0.1))),), 0)
    assert small_valid(mixed, 10) == 0
    diag = W.rotations_circuit(10, [PauliString(((1, "Z"), (4, "Z")))] + strings,
                               rng.uniform(-1, 1, len(strings) + 1))
    assert small_valid(diag, 10) == 0
    for n in (6, 13):
        s_n = W.ucc_rotation_strings(n, n // 2)[:40]
        assert small_valid(W.rotations_circuit(n, s_n, rng.uniform(-1, 1, len(s_n))), n) == 0
    # one group of more than 2048 rotations does not fit a run's angle buffer
    one = PauliString(((0, "X"), (1, "Y"), (2, "Z")))
    assert small_valid(W.rotations_circuit(9, [one] * 2049, rng.uniform(-1, 1, 2049)), 9) == 0
    assert small_valid(W.rotations_circuit(9, [one] * 2048, rng.uniform(-1, 1, 2048)), 9) == 1


def _popc(v):
    return bin(int(v)).count("1") & 1


def _slot(v, swz=(8, 8, 8)):
    """slot3 (csrc/qsv_small.cu): the program's involution on 16-B shared-memory
    slots -- the low 3 bits XOR three parities of the higher bits."""
    return v ^ sum(_popc(v & m) << j for j, m in enumerate(swz))


def _emulate_small(n, circ, basis):
    """CPU mirror of small_rot_kernel: the host table (debug_plan's "small":
    per group and class, each thread's first pair slot | config << 16, the
    share / flip slot XORs and the run-end flag) decides which pairs each
    thread covers; the matrices are rebuilt here from the rotation list.
    Returns the evolved state and checks that every group covers each pair of
    the basis state's class exactly once with one config per thread, that the
    lanes of each quarter warp hit distinct 16-B granules, and that inside a
    warp run no two warps touch the same amplitude (so __syncwarp suffices)."""
    k, q, v = flatten_bound(circ)
    plan = _lib.debug_plan(n, k, q, v)
    sm = plan["small"]
    assert sm["valid"] == 1
    spans, masks = _lib.match_rotations(n, k, q)
    R = [(int(m[0]), int(m[1]), int(m[2]), float(v[3 * int(s[2])])) for s, m in zip(spans, masks)]
    ncls, W, nthr = sm["ncls"], sm["w"], sm["nthr"]
    tab, xo, swz = sm["tab"], sm["xo"], sm["swz"]
    assert len(tab) == len(sm["groups"]) * (nthr << ncls)
    cls = sum(_popc(basis & W[j]) << j for j in range(ncls))
    psi = np.zeros(1 << n, dtype=complex)
    psi[basis] = 1.0
    owner = {}  # amplitude -> warp, within the current run
    conflicts = []  # per quarter warp: lanes sharing a 16-B granule
    for gi, g in enumerate(sm["groups"]):
        xm, r0, r1, dimb, h = g[0:5]
        pm, lu = g[5:9], g[9:11]
        assert xo[4 * gi] >> 4 == _slot(lu[0], swz) and xo[4 * gi + 1] >> 4 == _slot(lu[1], swz)
        assert (xo[4 * gi + 3] & 0xFFFF) >> 4 == _slot(xm, swz)
        rots = R[r0:r1]
        pairs_seen = set()
        lowm = (1 << h) - 1
        for t in range(nthr):
            e = tab[((gi << ncls) | cls) * nthr + t]
            lo0 = _slot((e & 0xFFFF) >> 4, swz)
            cfg0 = (e >> 16) & 15
            if t % 8 == 0:
                granules = set()
            granules.add(_slot(lo0, swz) & 7)
            if t % 8 == 7:
                conflicts.append(8 - len(granules))
            for a in range(4):
                lo = lo0 ^ (lu[0] if a & 1 else 0) ^ (lu[1] if a & 2 else 0)
                p = (lo & lowm) | ((lo >> 1) & ~lowm)
                assert sum(_popc(p & m) << j for j, m in enumerate(pm)) == cfg0  # shared config
                assert (lo >> h) & 1 == 0 and lo not in pairs_seen
                pairs_seen.add(lo)
                hi = lo ^ xm
                for amp in (lo, hi):
                    assert owner.setdefault(amp, t // 32) == t // 32, "two warps in one run"
                M = np.eye(2, dtype=complex)
                for (x, y, z, th) in rots:
                    ny = bin(y).count("1")
                    s_lo = -1 if _popc(lo & (y | z)) else 1
                    c, s = np.cos(th / 2), np.sin(th / 2)
                    off = -1j * s * (1j) ** ny * s_lo
                    M = np.array([[c, off * (-1) ** ny], [off, c]]) @ M
                psi[lo], psi[hi] = M[0, 0] * psi[lo] + M[0, 1] * psi[hi], M[1, 0] * psi[lo] + M[1, 1] * psi[hi]
        want = {lo for lo in range(1 << n) if not (lo >> h) & 1
                and sum(_popc(lo & W[j]) << j for j in range(ncls)) == cls}
        assert pairs_seen == want
        if xo[4 * gi + 3] >> 31:  # a CTA barrier ends the run
            owner = {}
    sm["conflicts"] = conflicts
    return psi, sm


def test_small_program_enumeration_emulated():
    """Invariant classes: a number-conserving UCC ansatz has only even-weight
    flips, so the total parity of the index is conserved and an evolve from a
    basis state touches half of the pairs.  The CPU mirror of the kernel's
    enumeration covers exactly that class and matches the oracle."""
    from oracle import oracle as O

    rng0 = np.random.default_rng(5)
    ucc = W.ucc_rotation_strings(10, 5)
    strings = ucc[:40] + ucc[-80:]  # singles + the last ten doubles
    circ = W.rotations_circuit(10, strings, rng0.uniform(-0.5, 0.5, len(strings)))
    ref_bits = W.hf_bitstring(5, 10)
    b = int(ref_bits[::-1], 2)
    psi, sm = _emulate_small(10, circ, b)
    assert sm["ncls"] == 1 and sm["w"][0] == 1023 and sm["share"] == 2
    # the program's slot map lets every quarter warp hit 8 distinct granules
    assert sum(sm["conflicts"]) == 0
    ref = O.evolve(O.init_state(ref_bits), circ.gates)
    assert np.abs(psi - ref).max() <= 1e-12
    # a program with odd-weight flips has no conserved parity
    from paper_2208_10978_b200.pauli import PauliString

    rng = np.random.default_rng(4)
    strings = [PauliString(((0, "X"),)), PauliString(((1, "Y"), (3, "X"), (5, "Z")))] + W.ucc_rotation_strings(8, 4)[:20]
    c2 = W.rotations_circuit(8, strings, rng.uniform(-1, 1, len(strings)))
    psi2, sm2 = _emulate_small(8, c2, 0b1011)
    assert sm2["ncls"] == 0
    assert np.abs(psi2 - O.evolve(O.init_state("11010000"), c2.gates)).max() <= 1e-12
