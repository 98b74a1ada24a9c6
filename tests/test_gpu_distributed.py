"""Sharded path (distributed.py) on the GPU through libqsv: P logical shards
on one device (LoopbackComm, exchanges are device copies), checked against
the CPU oracle.  Tolerances: amplitudes 1e-10 max-abs, energies 1e-10
relative (BASELINE.json north_star)."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2208_10978_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def D():
    from paper_2208_10978_b200 import distributed

    return distributed


@pytest.mark.parametrize("P,n,layers", [(2, 14, 6), (4, 18, 5), (8, 20, 4)])
def test_sharded_brickwork_vs_oracle(D, P, n, layers):
    circ = W.brickwork(n, layers, seed=20 + P)
    ref = O.evolve(O.init_state("0" * n), circ.gates)
    comm = D.LoopbackComm(P)
    s = D.evolve(D.init_state("0" * n, comm), circ)
    assert np.abs(s.amplitudes() - ref).max() < 1e-10


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_ucc_energy_vs_oracle(D, P):
    cfg = W.config1(seed=2, n_qubits=12, n_electrons=6, n_terms=300)
    ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    e_ref = O.expectation(ref, cfg["hamiltonian"], 12)
    be = D.DistributedBackend(D.LoopbackComm(P))
    psi = be.evolve(be.prepare(cfg["reference"]), cfg["circuit"])
    assert np.abs(psi.amplitudes() - ref).max() < 1e-10
    e = be.expectation(psi, cfg["hamiltonian"])  # dense strings: relayout + pairwise paths
    assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))


def test_sharded_sparse_hamiltonian_20q(D):
    n, P = 20, 4
    circ = W.brickwork(n, 3, seed=9)
    ref = O.evolve(O.init_state("0" * n), circ.gates)
    rng = np.random.default_rng(4)
    h = W.sparse_random_hamiltonian(n, 400, rng, z_only=120)
    e_ref = O.expectation(ref, h, n)
    be = D.DistributedBackend(D.LoopbackComm(P))
    e = be.expectation(be.evolve(be.prepare("0" * n), circ), h)
    assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))


def _pg_worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    from paper_2208_10978_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = D.ProcessGroupComm(piece_bytes=1 << 16)
        be = D.DistributedBackend(comm, D.CudaEngine(0))
        n = 18
        circ = W.brickwork(n, 6, seed=31)
        psi = be.evolve(be.prepare("0" * n), circ)
        rng = np.random.default_rng(13)
        h = W.sparse_random_hamiltonian(n, 150, rng, z_only=40)
        e = be.expectation(psi, h)
        q.put((rank, psi.amplitudes(), e, psi.stats["relayouts"], psi.stats.get("ipc_swaps", 0)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ipc", ["1", "0", "fail"])
def test_process_group_sharded_on_device(D, ipc, monkeypatch):
    """ProcessGroupComm + CudaEngine across 2 processes (gloo plumbing, both
    on this GPU): the multi-process sharded path against the oracle, with the
    relayout chunks swapped in place over CUDA IPC peer memory (default) or,
    with QSV_DIST_IPC=0, sent through host staging; "fail": rank 1 cannot map
    its partner, so both ranks agree to fall back to the staged path."""
    import socket

    import torch.multiprocessing as mp

    if ipc == "fail":
        monkeypatch.setenv("QSV_DIST_IPC", "1")
        monkeypatch.setenv("QSV_DIST_IPC_FAIL", "1")
    else:
        monkeypatch.setenv("QSV_DIST_IPC", ipc)

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_pg_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 18
    circ = W.brickwork(n, 6, seed=31)
    ref = O.evolve(O.init_state("0" * n), circ.gates)
    rng = np.random.default_rng(13)
    h = W.sparse_random_hamiltonian(n, 150, rng, z_only=40)
    e_ref = O.expectation(ref, h, n)
    for rank, amps, e, nrel, nswap in res:
        assert np.abs(amps - ref).max() < 1e-10
        assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))
        assert nrel >= 1
        assert (nswap > 0) == (ipc == "1")  # "fail": no swap kernels, the staged path ran


@pytest.mark.parametrize("P", [2, 8])
def test_sharded_ucc_units_16q(D, P):
    """UCC rotations as units: flips off the global qubits run as direct
    rotations with a per-rank angle sign for global Z; others via relayouts."""
    cfg = W.config1(seed=4, n_qubits=16, n_electrons=8, n_terms=100)
    ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    be = D.DistributedBackend(D.LoopbackComm(P))
    psi = be.evolve(be.prepare(cfg["reference"]), cfg["circuit"])
    assert np.abs(psi.amplitudes() - ref).max() < 1e-10
    assert psi.stats["relayouts"] >= 1
    e = be.expectation(psi, cfg["hamiltonian"])
    e_ref = O.expectation(ref, cfg["hamiltonian"], 16)
    assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))


def test_sharded_bound_circuit_from_bind(D):
    """bind() results (BoundCircuit: arrays, lazily built gates) go through the
    sharded path like reference Circuit objects."""
    from paper_2208_10978_b200.circuit import bind

    n, ne, P = 14, 6, 4
    strings = W.ucc_rotation_strings(n, ne)[:120]
    param = W.parametric_rotations_circuit(n, strings)
    theta = np.random.default_rng(3).uniform(-0.4, 0.4, len(strings))
    ref = W.hf_bitstring(ne, n)
    be = D.DistributedBackend(D.LoopbackComm(P))
    psi = be.evolve(be.prepare(ref), bind(param, theta))
    exp = O.evolve(O.init_state(ref), W.rotations_circuit(n, strings, theta).gates)
    assert np.abs(psi.amplitudes() - exp).max() < 1e-10


def test_config5_structure_29q_one_state_of_memory(D):
    """Config-5 structure (brickwork depth 10, top 3 qubits global, P = 8) at
    29 q on one B200 (loopback shards): evolving the lazy |0...0> allocates
    the output shards only -- device memory in use afterwards (shards, the
    library workspace, relayout staging) <= 1.1 x the 8 GiB state -- and,
    realigned to the identity layout on the device, the shards equal the
    single-GPU engine's state (<= 1e-12)."""
    import torch

    from paper_2208_10978_b200 import statevector as sv

    n, P = 29, 8
    sv.release_pool()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    free0, _ = sv.mem_info(0)
    be = D.DistributedBackend(D.LoopbackComm(P), D.CudaEngine(0))
    circ = W.brickwork(n, 10, seed=5)
    s0 = be.prepare("0" * n)
    psi = be.evolve(s0, circ)
    for sh in psi.shards.values():
        sh.synchronize()
    torch.cuda.synchronize()
    free1, _ = sv.mem_info(0)
    state = 16 * (1 << n)
    assert free0 - free1 <= 1.1 * state, f"{(free0 - free1) / 2**30:.2f} GiB for an 8 GiB state"
    assert psi.stats["relayouts"] >= 1 and s0.basis_index == 0
    psi.align_to(list(range(n)))  # relayouts + local SWAPs on the device
    single = sv.evolve(sv.init_state("0" * n), circ)
    single.synchronize()
    for sh in psi.shards.values():
        sh.synchronize()
    ref = torch.as_tensor(single, device="cuda")
    chunk = 1 << (n - 3)
    worst = 0.0
    for r, sh in psi.shards.items():
        d = (torch.as_tensor(sh, device="cuda") - ref[r * chunk:(r + 1) * chunk]).abs().max()
        worst = max(worst, float(d))
    assert worst <= 1e-12


@pytest.mark.parametrize("P,n,layers", [(2, 14, 6), (4, 16, 5), (8, 18, 4)])
@pytest.mark.parametrize("p2p", ["1", "0"])
def test_native_multidevice_brickwork_vs_oracle(P, n, layers, p2p, monkeypatch):
    """qsv_dist (C++ planner + relayouts, P shards on device 0) vs the oracle;
    the 20-layer light cone needs few relayouts.  Relayouts run as in-place
    swap kernels over peer memory (event-ordered, each rank of a pair swapping
    one half) or, with QSV_DIST_P2P=0, as staged cudaMemcpyPeerAsync."""
    from paper_2208_10978_b200.multidevice import MultiDeviceState

    monkeypatch.setenv("QSV_DIST_P2P", p2p)
    circ = W.brickwork(n, layers, seed=40 + P)
    st = MultiDeviceState(n, [0] * P)
    st.set_basis(0)
    st.apply(circ)
    ref = O.evolve(O.init_state("0" * n), circ.gates)
    assert np.abs(st.amplitudes - ref).max() < 1e-10
    info = st.info()
    assert info["ranks"] == P and info["relayouts"] >= 1
    assert info["p2p"]  # shards sharing a device address each other
    assert (info["swap_launches"] > 0) == (p2p == "1")
    # the C++ scheduler is the Python one (distributed.plan_segments): same
    # relayouts and the same final qubit map
    from paper_2208_10978_b200 import distributed as Dm
    from paper_2208_10978_b200.circuit import flatten_bound

    k, q, _ = flatten_bound(circ)
    segs, perm = Dm.plan_segments(k, q, n, n - (P.bit_length() - 1), list(range(n)))
    assert info["relayouts"] == sum(1 for sg in segs if sg.relayout is not None)
    assert info["perm"] == list(perm)


@pytest.mark.parametrize("P", [2, 4, 8])
def test_native_multidevice_ucc_energy_vs_oracle(P):
    """UCC-shaped circuit + a config-3-style Hamiltonian (weights 1-4, flips
    localised by relayouts) through the native handle's backend protocol:
    energy within 1e-10 of the oracle and of the Python sharded path."""
    from paper_2208_10978_b200.multidevice import MultiDeviceBackend
    from paper_2208_10978_b200 import distributed as Dm

    cfg = W.config1(seed=7, n_qubits=12, n_electrons=6, n_terms=10)
    h = W.sparse_random_hamiltonian(12, 300, np.random.default_rng(12 + P), z_only=90)
    ref = O.evolve(O.init_state(cfg["reference"]), cfg["circuit"].gates)
    e_ref = O.expectation(ref, h, 12)
    be = MultiDeviceBackend([0] * P)
    psi = be.evolve(be.prepare(cfg["reference"]), cfg["circuit"])
    assert np.abs(psi.amplitudes - ref).max() < 1e-10
    e = be.expectation(psi, h)
    assert abs(e - e_ref) <= 1e-10 * max(1.0, abs(e_ref))
    assert np.abs(psi.amplitudes - ref).max() < 1e-10  # localising relayouts keep the state
    py = Dm.DistributedBackend(Dm.LoopbackComm(P))
    e_py = py.expectation(py.evolve(py.prepare(cfg["reference"]), cfg["circuit"]), h)
    assert abs(e - e_py) <= 1e-10 * max(1.0, abs(e_py))


def test_native_multidevice_errors():
    from paper_2208_10978_b200.multidevice import MultiDeviceState

    with pytest.raises(ValueError):
        MultiDeviceState(10, [0, 0, 0])  # not a power of two
    st = MultiDeviceState(8, [0, 0])
    with pytest.raises(ValueError):
        st.set_basis(1 << 8)
    h = W.sparse_random_hamiltonian(8, 20, np.random.default_rng(0), z_only=5)
    st.set_basis(3)
    re, im = st.expectation_terms(h)
    assert np.isfinite(re)
    from paper_2208_10978_b200.pauli import PauliString, PauliSum, PauliTerm

    wide = PauliSum((PauliTerm(1.0, PauliString(tuple((q, "X") for q in range(8)))),))
    with pytest.raises(ValueError):  # a flip wider than a shard's local qubits
        st.expectation_terms(wide)
