"""Host logic of the sharded (multi-GPU) path -- distributed.py -- on CPU.

Local shard compute goes through a test double backed by the CPU oracle (the
oracle is test infrastructure: it stands in for libqsv here so the planner,
the qubit map, the pairwise relayout exchange and the ordered reduction can be
checked without a GPU).  The exchange runs both in-process (LoopbackComm)
and across 2 processes over gloo (ProcessGroupComm), as SURVEY.md 8(e)/4 ask.
"""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2208_10978_b200 import distributed as D
from paper_2208_10978_b200 import workloads as W
from paper_2208_10978_b200.circuit import flatten_bound

NAMES = ["H", "HY", "X", "CNOT", "SWAP", "RZ", "RY", "U3", "CU3"]
NPAR = {"H": 0, "HY": 0, "X": 0, "CNOT": 0, "SWAP": 0, "RZ": 1, "RY": 1, "U3": 3, "CU3": 3}


class _Shard:
    def __init__(self, amps):
        self.amps = amps


class OracleEngine:
    """LocalEngine test double: numpy shards, oracle kernels."""

    def zeros(self, n_local):
        return _Shard(np.zeros(1 << n_local, dtype=np.complex128))

    def basis(self, n_local, index):
        s = self.zeros(n_local)
        s.amps[index] = 1.0
        return s

    def copy(self, shard):
        return _Shard(shard.amps.copy())

    def apply_gates(self, shard, kinds, qubits, values):
        for i, k in enumerate(kinds):
            name = NAMES[int(k)]
            qs = (int(qubits[2 * i]),) if qubits[2 * i + 1] < 0 else (int(qubits[2 * i]),
                                                                      int(qubits[2 * i + 1]))
            O.apply_gate(shard.amps, name, qs, tuple(values[3 * i:3 * i + NPAR[name]]))

    def expectation_terms(self, shard, x, y, z):
        out = np.zeros(len(x))
        scratch = np.empty_like(shard.amps)
        for t in range(len(x)):
            O.apply_pauli(shard.amps, int(x[t]), int(y[t]), int(z[t]), scratch)
            out[t] = np.vdot(shard.amps, scratch).real
        return out

    def apply_pauli(self, src, dst, x, y, z):
        O.apply_pauli(src.amps, int(x), int(y), int(z), dst.amps)

    def apply_rotations(self, shard, x, y, z, theta):
        scratch = np.empty_like(shard.amps)
        for k in range(len(theta)):
            O.apply_pauli(shard.amps, int(x[k]), int(y[k]), int(z[k]), scratch)
            shard.amps[:] = np.cos(theta[k] / 2) * shard.amps - 1j * np.sin(theta[k] / 2) * scratch

    def vdot(self, a, b):
        return complex(np.vdot(a.amps, b.amps))

    def tensor(self, shard):
        return torch.from_numpy(shard.amps.view(np.float64).reshape(-1, 2))

    def synchronize(self, shard):
        pass

    def download(self, shard):
        return shard.amps.copy()


def _oracle_state(circ, bitstring):
    return O.evolve(O.init_state(bitstring), circ.gates)


def _random_mixed(n, G, seed):
    from paper_2208_10978_b200.circuit import Circuit, Constant, Gate

    rng = np.random.default_rng(seed)
    gates = []
    for _ in range(G):
        k = NAMES[rng.integers(len(NAMES))]
        if k in ("CNOT", "SWAP", "CU3"):
            a, b = rng.choice(n, 2, replace=False)
            qs = (int(a), int(b))
        else:
            qs = (int(rng.integers(n)),)
        ps = tuple(Constant(float(v)) for v in rng.uniform(-np.pi, np.pi, NPAR[k]))
        gates.append(Gate(k, qs, ps))
    return Circuit(n, tuple(gates), 0)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_plan_segments_only_local_gates(P):
    n = 9
    g = P.bit_length() - 1
    circ = W.brickwork(n, 6, seed=P)
    kinds, qubits, values = flatten_bound(circ)
    segs, perm = D.plan_segments(kinds, qubits, n, n - g, list(range(n)))
    assert sorted(perm) == list(range(n))
    seen = []
    for s in segs:
        assert np.all(s.qubits[s.qubits >= 0] < n - g)
        seen.extend(int(i) for i in s.src if i >= 0)
        if s.relayout is not None:
            assert 1 <= s.relayout.k <= g
    assert sorted(seen) == list(range(len(kinds)))  # every gate exactly once
    # gates sharing a qubit keep their relative order (only commuting gates move)
    last = {}
    for i in seen:
        qs = [int(qubits[2 * i])] + ([int(qubits[2 * i + 1])] if qubits[2 * i + 1] >= 0 else [])
        for q in qs:
            assert last.get(q, -1) < i
            last[q] = i
    # light-cone scheduling: one exchange serves the whole brickwork
    assert sum(s.relayout is not None for s in segs) <= 2


@pytest.mark.parametrize("P,n,layers", [(2, 8, 5), (4, 9, 6), (8, 10, 4)])
def test_loopback_brickwork_matches_oracle(P, n, layers):
    circ = W.brickwork(n, layers, seed=11 + P)
    ref = _oracle_state(circ, "0" * n)
    comm = D.LoopbackComm(P)
    s = D.evolve(D.init_state("0" * n, comm, OracleEngine()), circ)
    assert np.abs(s.amplitudes() - ref).max() < 1e-12


@pytest.mark.parametrize("P", [2, 4])
def test_loopback_mixed_gates_and_basis(P):
    n = 8
    circ = _random_mixed(n, 120, seed=P)
    bits = "10110010"
    ref = _oracle_state(circ, bits)
    comm = D.LoopbackComm(P)
    s0 = D.init_state(bits, comm, OracleEngine())
    s = D.evolve(s0, circ)
    assert np.abs(s.amplitudes() - ref).max() < 1e-12
    # evolve leaves its input untouched (statevector.py:71)
    e0 = np.zeros(1 << n, dtype=complex)
    e0[sum(1 << k for k, c in enumerate(bits) if c == "1")] = 1
    assert np.abs(s0.amplitudes() - e0).max() == 0


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_loopback_expectation_worker_invariant(P):
    n = 9
    cfg = W.config1(seed=5, n_qubits=n, n_electrons=4, n_terms=150)
    ref_state = _oracle_state(cfg["circuit"], cfg["reference"])
    e_ref = O.expectation(ref_state, cfg["hamiltonian"], n)
    comm = D.LoopbackComm(P)
    be = D.DistributedBackend(comm, OracleEngine())
    psi = be.evolve(be.prepare(cfg["reference"]), cfg["circuit"])
    e = be.expectation(psi, cfg["hamiltonian"])
    assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))
    # the relayouts expectation performs keep the logical state unchanged
    assert np.abs(psi.amplitudes() - ref_state).max() < 1e-12


def test_wide_string_rejected():
    # a flip wider than the local qubits of a shard cannot be localised
    with pytest.raises(ValueError):
        D.plan_localize([0b1111], 4, 2, list(range(4)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, world, port, n, layers, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = D.ProcessGroupComm(piece_bytes=1 << 10)  # small pieces: exercise chunking
        circ = W.brickwork(n, layers, seed=3)
        be = D.DistributedBackend(comm, OracleEngine())
        psi = be.evolve(be.prepare("0" * n), circ)
        amps = psi.amplitudes()
        rng = np.random.default_rng(7)
        h = W.dense_random_hamiltonian(n, 60, rng)  # strings up to n wide: pairwise path too
        e = be.expectation(psi, h)
        q.put((rank, amps, e))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_match_oracle():
    import torch.multiprocessing as mp

    n, layers, world = 8, 5, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, n, layers, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    circ = W.brickwork(n, layers, seed=3)
    ref = _oracle_state(circ, "0" * n)
    rng = np.random.default_rng(7)
    h = W.dense_random_hamiltonian(n, 60, rng)
    e_ref = O.expectation(ref, h, n)
    for rank, amps, e in res:
        assert np.abs(amps - ref).max() < 1e-12
        assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))
    assert res[0][2] == res[1][2]  # identical reduction on every rank


@pytest.mark.parametrize("P,n,seed", [(2, 7, 0), (4, 8, 1), (8, 9, 2), (8, 9, 3)])
def test_plan_align_random_layouts(P, n, seed):
    """Any physical layout can be realigned to any other by <= 2 relayouts +
    local SWAPs; the logical state is unchanged (oracle engine, loopback)."""
    rng = np.random.default_rng(seed)
    circ = _random_mixed(n, 60, seed)
    comm = D.LoopbackComm(P)
    be = D.DistributedBackend(comm, OracleEngine())
    psi = be.evolve(be.prepare("0" * n), circ)
    ref = _oracle_state(circ, "0" * n)
    for _ in range(3):
        target = [int(v) for v in rng.permutation(n)]
        steps = D.plan_align(psi.perm, target, n, psi.n_local)
        assert sum(1 for k, _ in steps if k == "relayout") <= 2
        psi.align_to(target)
        assert psi.perm == target
        assert np.abs(psi.amplitudes() - ref).max() < 1e-13


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_overlap_across_layouts(P):
    """DistributedBackend.overlap (engine.py:74-75: np.vdot(a, b)) between
    states whose layouts differ (different circuits -> different relayouts)."""
    n = 8
    comm = D.LoopbackComm(P)
    be = D.DistributedBackend(comm, OracleEngine())
    c1, c2 = _random_mixed(n, 50, 11), W.brickwork(n, 4, seed=12)
    a = be.evolve(be.prepare("0" * n), c1)
    b = be.evolve(be.prepare("1" + "0" * (n - 1)), c2)
    ra, rb = _oracle_state(c1, "0" * n), _oracle_state(c2, "1" + "0" * (n - 1))
    v = be.overlap(a, b)
    assert abs(v - np.vdot(ra, rb)) < 1e-13
    assert abs(be.overlap(a, a) - 1.0) < 1e-13
    assert np.abs(b.amplitudes() - rb).max() < 1e-13  # realigned, logically unchanged


def test_lazy_basis_evolve_allocates_one_state():
    """prepare() keeps |index> lazy: evolve materialises it straight into its
    output shards and the input never allocates (config 5: one 128 GiB shard
    per GPU, not two)."""
    n, P = 8, 4
    made = []

    class Counting(OracleEngine):
        def zeros(self, n_local):
            made.append(n_local)
            return super().zeros(n_local)

    comm = D.LoopbackComm(P)
    be = D.DistributedBackend(comm, Counting())
    s0 = be.prepare("0110" + "0" * (n - 4))
    assert s0.basis_index is not None and not made
    circ = W.brickwork(n, 3, seed=2)
    psi = be.evolve(s0, circ)
    assert s0.basis_index is not None  # input untouched and still lazy
    assert len(made) == P  # one shard per rank (the test engine's basis() goes through zeros())
    assert np.abs(psi.amplitudes() - _oracle_state(circ, "0110" + "0" * (n - 4))).max() < 1e-13


def _gloo_overlap_worker(rank, world, port, n, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = D.ProcessGroupComm(piece_bytes=1 << 9)
        be = D.DistributedBackend(comm, OracleEngine())
        a = be.evolve(be.prepare("0" * n), _random_mixed(n, 40, 21))
        b = be.evolve(be.prepare("1" * n), W.brickwork(n, 3, seed=22))
        v = be.overlap(a, b)  # realigns b over the process group (P2P relayouts)
        q.put((rank, v, a.perm == b.perm, b.amplitudes()))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_overlap_across_layouts():
    import torch.multiprocessing as mp

    n, world = 7, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_overlap_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ra = _oracle_state(_random_mixed(n, 40, 21), "0" * n)
    rb = _oracle_state(W.brickwork(n, 3, seed=22), "1" * n)
    for rank, v, same, amps in res:
        assert same
        assert abs(v - np.vdot(ra, rb)) < 1e-13
        assert np.abs(amps - rb).max() < 1e-13
    assert res[0][1] == res[1][1]
