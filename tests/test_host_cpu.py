"""Host-side logic without a GPU: IR, interchange formats, JW generator,
workload determinism, LPT partition semantics."""

import io

import numpy as np
import pytest

from conftest import parse_h
from paper_2208_10978_b200 import engine
from paper_2208_10978_b200 import workloads as W
from paper_2208_10978_b200.circuit import (Affine, Circuit, Constant, Gate, bind, circuit_from_json,
                                           circuit_to_json, flatten_bound, gate_matrix,
                                           pauli_evolution)
from paper_2208_10978_b200.errors import FormatError
from paper_2208_10978_b200.pauli import PauliString, PauliSum, read_pauli_sum, write_pauli_sum


def test_pauli_text_roundtrip(golden):
    h = parse_h(golden["expect_h"])
    buf = io.StringIO()
    write_pauli_sum(h, buf)
    assert buf.getvalue() == str(golden["expect_h"])
    with pytest.raises(FormatError):
        read_pauli_sum(io.StringIO("1.0 X0 X0\n"))
    with pytest.raises(FormatError):
        read_pauli_sum(io.StringIO("abc X0\n"))


def test_circuit_json_roundtrip(golden):
    text = str(golden["uccsd8_circuit"])
    assert circuit_to_json(circuit_from_json(text)) == text


def test_gate_validation():
    with pytest.raises(ValueError):
        Gate("CNOT", (1, 1))
    with pytest.raises(ValueError):
        Gate("RZ", (0,))
    with pytest.raises(ValueError):
        Circuit(2, (Gate("H", (2,)),))
    c = Circuit(2, (Gate("RZ", (0,), (Affine(0, 2.0, 0.5),)),), 1)
    with pytest.raises(RuntimeError):
        flatten_bound(c)
    b = bind(c, [0.25])
    assert b.gates[0].bound_values() == (1.0,)
    with pytest.raises(ValueError):
        bind(c, [np.nan])


def test_gate_matrices_unitary():
    for kind, vals in [("H", ()), ("HY", ()), ("RZ", (0.3,)), ("RY", (1.1,)), ("U3", (0.4, 1.3, -2.0)),
                       ("CU3", (0.4, 1.3, -2.0)), ("CNOT", ()), ("SWAP", ()), ("X", ())]:
        m = gate_matrix(kind, vals)
        assert np.allclose(m.conj().T @ m, np.eye(m.shape[0]), atol=1e-14)
    hy = gate_matrix("HY")
    y = np.array([[0, -1j], [1j, 0]])
    z = np.diag([1, -1])
    assert np.allclose(hy @ z @ hy, y)  # HY rotates the Y eigenbasis onto Z


def test_pauli_evolution_gate_pattern():
    p = PauliString.from_label("X0 Z2 Y5")
    c = pauli_evolution(p, 0.3, 6)
    kinds = [g.kind for g in c.gates]
    assert kinds == ["H", "HY", "CNOT", "CNOT", "RZ", "CNOT", "CNOT", "H", "HY"]
    assert c.gates[4].bound_values() == (-0.6,)
    assert c.gates[4].qubits == (5,)


def test_workload_shapes():
    c1 = W.config1()
    assert len(c1["strings"]) == 1872 and c1["reference"] == "111111000000"
    assert len(c1["hamiltonian"]) == 500 and c1["hamiltonian"].is_hermitian()
    c2 = W.config2()
    assert len(c2["circuit"].gates) == 830
    assert sum(g.kind == "CNOT" for g in c2["circuit"].gates) == 270
    h3 = W.config3_hamiltonian()
    assert len(h3) == 10_000
    zonly = [all(a == "Z" for _, a in t.string.factors) for t in h3.terms]
    assert all(zonly[:3000]) and not any(zonly[3000:])
    assert all(1 <= t.string.weight <= 4 for t in h3.terms)


def test_workload_determinism():
    a = W.brickwork(8, 3, seed=7)
    b = W.brickwork(8, 3, seed=7)
    assert circuit_to_json(a) == circuit_to_json(b)
    s = W.config3_state(seed=1, n_qubits=12, chunk_bits=8)
    assert abs(np.linalg.norm(s) - 1) < 1e-12


def test_plan_partition_lpt():
    h = PauliSum.from_terms([(1.0, PauliString.from_label(lbl)) for lbl in
                             ["X0", "X0 X1 X2", "Z3", "Y1 Y2", "Z0 Z1 Z2 Z3", ""]])
    plan = engine.plan_partition(h, 2)
    seen = sorted(i for p in plan.partitions for i in p)
    assert seen == list(range(6))
    loads = [sum(plan.costs[i] for i in p) for p in plan.partitions]
    assert max(loads) <= sum(plan.costs) / 2 + max(plan.costs)
    assert plan.partitions == engine.plan_partition(h, 2).partitions  # deterministic


def test_vectorised_bind_matches_per_gate_evaluation():
    """bind's numpy gather + multiply-add gives the same bits as evaluating
    each Affine (circuit.py:145-156), and the lazily built gates match."""
    from paper_2208_10978_b200 import workloads as W
    from paper_2208_10978_b200.circuit import BoundCircuit, evolution_gates, flatten_bound

    cfg = W.config1(seed=3, n_qubits=8, n_electrons=4, n_terms=10)
    strings = W.ucc_rotation_strings(8, 4)
    gates = []
    for k, s in enumerate(strings):
        gates.extend(evolution_gates(s, Affine(k, -0.5, 0.125 * (k % 3))))
    gates.append(Gate("U3", (1,), (Affine(0, 2.0, 0.5), Constant(0.3), Affine(1, -1.5))))
    c = Circuit(8, tuple(gates), len(strings))
    theta = np.random.default_rng(0).uniform(-1, 1, len(strings))
    b = bind(c, theta)
    assert isinstance(b, BoundCircuit) and b.is_bound() and len(b) == len(gates)
    k, q, v = flatten_bound(b)
    for i, g in enumerate(c.gates):
        for j, p in enumerate(g.params):
            assert v[3 * i + j] == p.evaluate(theta)  # bit-identical
        assert b.gates[i].bound_values() == tuple(p.evaluate(theta) for p in g.params)
    assert b == Circuit(8, b.gates, 0)
    k2, q2, v2 = flatten_bound(Circuit(8, b.gates, 0))
    assert np.array_equal(k, k2) and np.array_equal(q, q2) and np.array_equal(v, v2)
    assert cfg["circuit"].n_qubits == 8


def test_lazy_bind_values_are_per_circuit():
    """bind evaluates only the Affine slots: each BoundCircuit keeps its own
    values (successive binds of one parametric circuit do not share a value
    array), the full array built on demand equals the engine-call buffer
    (call_values, the plan's reused scratch), and both equal per-gate
    evaluation."""
    from paper_2208_10978_b200.circuit import evolution_gates

    strings = W.ucc_rotation_strings(8, 4)
    gates = []
    for k, st in enumerate(strings):
        gates.extend(evolution_gates(st, Affine(k, -0.5, 0.1)))
    c = Circuit(8, tuple(gates), len(strings))
    rng = np.random.default_rng(1)
    t1, t2 = rng.uniform(-1, 1, len(strings)), rng.uniform(-1, 1, len(strings))
    b1, b2 = bind(c, t1), bind(c, t2)
    with b2.call_values() as v:  # fills the shared scratch with b2's slots
        v2_call = v.copy()
    with b1.call_values() as v:  # ... then with b1's
        v1_call = v.copy()
    v1, v2 = b1.flat()[2], b2.flat()[2]
    assert v1 is not v2 and np.array_equal(v1, v1_call) and np.array_equal(v2, v2_call)
    for i, g in enumerate(c.gates):
        for j, p in enumerate(g.params):
            assert v1[3 * i + j] == p.evaluate(t1) and v2[3 * i + j] == p.evaluate(t2)


def _ref_engine():
    import os
    import sys

    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
    if not os.path.isdir(os.path.join(ref, "vqekit")):
        pytest.skip("oracle/_ref (reference build) not built")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import vqekit.engine as RE
    import vqekit.pauli as RP

    return RE, RP


@pytest.mark.parametrize("workers", [1, 2, 3, 4, 8, 16])
def test_plan_partition_equals_reference(workers):
    """LPT split identical to the reference's plan_partition (engine.py:131-147)
    on a config-3-style Hamiltonian with many equal weights (tie rules)."""
    RE, RP = _ref_engine()
    from paper_2208_10978_b200 import workloads as W

    h = W.sparse_random_hamiltonian(12, 300, np.random.default_rng(workers), z_only=90)
    rh = RP.PauliSum(tuple(RP.PauliTerm(complex(t.coefficient), RP.PauliString(tuple(t.string.factors)))
                           for t in h.terms))
    ours = engine.plan_partition(h, workers)
    ref = RE.plan_partition(rh, workers)
    assert ours.partitions == ref.partitions
    assert ours.costs == ref.costs


class _HostState:
    def __init__(self, amps):
        self.amps = amps
        self.n_qubits = int(amps.size).bit_length() - 1


class _OraclePerTerm:
    """Per-term <P_t> from the C oracle (test stand-in for the CUDA engine)."""

    def expectation_terms(self, state, x, y, z):
        from oracle import oracle as O

        out = np.zeros(len(x))
        scratch = np.empty_like(state.amps)
        for k in range(len(x)):
            O.apply_pauli(state.amps, int(x[k]), int(y[k]), int(z[k]), scratch)
            out[k] = O.vdot(state.amps, scratch).real
        return out


def test_expectation_parallel_worker_invariant_and_equals_reference():
    """SPEC acceptance #8: W in {1,2,4,8} identical to 1e-12; equal to the
    reference's own expectation_parallel on the same state and plan."""
    RE, RP = _ref_engine()
    import vqekit.statevector as RSV

    from conftest import random_state
    from paper_2208_10978_b200 import workloads as W

    n = 10
    rng = np.random.default_rng(8)
    h = W.sparse_random_hamiltonian(n, 400, rng, z_only=120)
    st = random_state(n, rng)
    rh = RP.PauliSum(tuple(RP.PauliTerm(complex(t.coefficient), RP.PauliString(tuple(t.string.factors)))
                           for t in h.terms))
    vals = []
    for w in (1, 2, 4, 8):
        e = engine.expectation_parallel(_HostState(st), h, engine.plan_partition(h, w),
                                        engine=_OraclePerTerm())
        e_ref = RE.expectation_parallel(RSV.StateVector(n, st), rh, RE.plan_partition(rh, w))
        assert abs(e - e_ref) <= 1e-12 * max(1.0, abs(e_ref))
        vals.append(e)
    assert max(vals) - min(vals) <= 1e-12 * max(1.0, abs(vals[0]))


def _a16_worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    from conftest import random_state
    from paper_2208_10978_b200 import distributed as D
    from paper_2208_10978_b200 import workloads as W

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 9
        rng = np.random.default_rng(4)
        h = W.sparse_random_hamiltonian(n, 200, rng, z_only=60)
        st = random_state(n, rng)  # every rank holds the same replica
        comm = D.ProcessGroupComm()
        out = {w: engine.expectation_parallel(_HostState(st), h, engine.plan_partition(h, w),
                                              comm=comm, engine=_OraclePerTerm())
               for w in (1, 2, 4, 8)}
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_expectation_parallel_two_ranks_gloo():
    """Replicated state on 2 ranks: worker w evaluated on rank w % 2, partials
    gathered and summed in worker order -- same value on every rank, for
    every W, as the single-process sum."""
    import socket

    import torch.multiprocessing as mp

    from conftest import random_state
    from paper_2208_10978_b200 import workloads as W

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_a16_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 9
    rng = np.random.default_rng(4)
    h = W.sparse_random_hamiltonian(n, 200, rng, z_only=60)
    st = random_state(n, rng)
    for w in (1, 2, 4, 8):
        single = engine.expectation_parallel(_HostState(st), h, engine.plan_partition(h, w),
                                             engine=_OraclePerTerm())
        assert res[0][w] == res[1][w] == single


@pytest.mark.parametrize("create,annihilate", [((7,), (2,)), ((9,), (0,)), ((6, 11), (3, 1)),
                                               ((8, 10), (5, 4)), ((31, 16), (15, 0))])
def test_jw_excitation_strings_equal_reference_jordan_wigner(create, annihilate):
    """workloads.excitation_strings (the generator behind configs 1 and 4) vs
    the reference's own fermion.jordan_wigner of T - T^dagger (fermion.py:345):
    same strings, same coefficients (1e-15), and -- after the canonical sort
    -- the same order."""
    _ref_engine()  # puts oracle/_ref on sys.path (skips if absent)
    import vqekit.fermion as RF

    ops = [(m, True) for m in create] + [(m, False) for m in annihilate]
    t = RF.FermionSum.from_terms([(1.0, ops)])
    ref = RF.jordan_wigner(t - t.dagger())
    ref_terms = sorted(((tt.string.factors, complex(tt.coefficient)) for tt in ref.terms),
                       key=lambda kv: kv[0])
    ours = W.excitation_strings(create, annihilate)
    assert [s.factors for _, s in ours] == [f for f, _ in ref_terms]
    for (c, _), (_, rc) in zip(ours, ref_terms):
        assert abs(c - rc) <= 1e-15
    assert len(ours) == (2 if len(create) == 1 else 8)


def test_integration_install_dispatches_host_states_to_the_reference():
    """integration.install wraps exactly four reference attributes; host
    (reference) states still go to the reference's own functions, and
    uninstall restores the originals (no GPU needed)."""
    RE, RP = _ref_engine()
    import json
    import os

    import vqekit
    import vqekit.circuit as RC
    import vqekit.statevector as RSV

    from conftest import GOLDEN
    from paper_2208_10978_b200 import integration

    with open(os.path.join(GOLDEN, "h2_sto3g.json")) as fh:
        fx = json.load(fh)["h2_sto3g_d0735.fcidump"]
    h = RP.read_pauli_sum(io.StringIO(fx["hamiltonian"]))
    ansatz = RC.circuit_from_json(fx["ansatz"])
    s0 = RSV.init_state(fx["reference"])
    theta = np.array([0.1, -0.2])
    before = (RSV.reverse_gradient, RSV.reverse_gradient_general, RSV.apply_operator,
              RE.expectation_parallel)
    g0 = RSV.reverse_gradient(ansatz, theta, h, s0)
    integration.install(vqekit)
    try:
        assert integration.installed()
        assert RSV.reverse_gradient is not before[0] and RE.expectation_parallel is not before[3]
        assert np.array_equal(RSV.reverse_gradient(ansatz, theta, h, s0), g0)
        st = RSV.evolve(s0, RC.bind(ansatz, theta))
        plan = RE.plan_partition(h, 2)
        assert RE.expectation_parallel(st, h, plan) == before[3](st, h, plan)
        assert np.array_equal(RSV.apply_operator(st, h).amplitudes, before[2](st, h).amplitudes)
    finally:
        integration.uninstall()
    assert (RSV.reverse_gradient, RSV.reverse_gradient_general, RSV.apply_operator,
            RE.expectation_parallel) == before
    assert not integration.installed()
