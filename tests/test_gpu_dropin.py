"""Drop-in proof: the reference's OWN drivers run on the B200 backend.

The reference package (oracle/_ref: vqekit, built from /root/reference/pkg
by oracle/Makefile; travels to the GPU box) supplies the callers and the
objects -- ``vqe_minimize`` (engine.py:433-481), ``parameter_shift_gradient``
(:248-266), ``vqd_excited`` (:607-689), its ``Circuit``/``PauliSum`` built from
the H2 fixtures by its own JW + UCCSD code (tests/golden/h2_sto3g.json,
written by tests/golden/make_golden.py) and its ``bind``.  Each driver runs
twice, once with the reference's CPU ``StateVectorBackend`` and once with
``paper_2208_10978_b200.engine.StateVectorBackend`` (device states; the
gradient / operator / partitioned-expectation calls the drivers make on
``vqekit.statevector`` directly are registered by
``integration.install``).  Energies must agree within 1e-10 relative
(north_star), gradients within 1e-10."""

import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REPO

pytestmark = pytest.mark.gpu

REL = 1e-10


@pytest.fixture(scope="module")
def vq():
    ref = os.path.join(REPO, "oracle", "_ref")
    assert os.path.isdir(os.path.join(ref, "vqekit")), "oracle/_ref (reference build) missing"
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import io

    import vqekit
    import vqekit.circuit as RC
    import vqekit.engine as RE
    import vqekit.pauli as RP

    from paper_2208_10978_b200 import integration

    integration.install(vqekit)
    with open(os.path.join(GOLDEN, "h2_sto3g.json")) as fh:
        fx = json.load(fh)["h2_sto3g_d0735.fcidump"]
    h = RP.read_pauli_sum(io.StringIO(fx["hamiltonian"]))
    ansatz = RC.circuit_from_json(fx["ansatz"])
    yield {"RE": RE, "RC": RC, "h": h, "ansatz": ansatz, "ref": fx["reference"], "fx": fx}
    integration.uninstall()


def _b200():
    from paper_2208_10978_b200 import engine

    return engine.StateVectorBackend()


def test_backend_advertises_device_gradient(vq):
    be = _b200()
    assert be.supports_reverse_gradient  # routed to the device adjoint by install()


@pytest.mark.parametrize("method", ["gradient", "simplex"])
def test_vqe_minimize_matches_cpu_backend(vq, method):
    RE = vq["RE"]
    opts = RE.OptimizerOptions(method=method)
    cpu = RE.vqe_minimize(vq["h"], vq["ansatz"], vq["ref"], RE.StateVectorBackend(), opts)
    gpu = RE.vqe_minimize(vq["h"], vq["ansatz"], vq["ref"], _b200(), opts)
    assert abs(gpu.energy - cpu.energy) <= REL * abs(cpu.energy)
    assert gpu.n_iterations == cpu.n_iterations
    assert np.abs(np.asarray(gpu.theta) - np.asarray(cpu.theta)).max() <= 1e-7
    if method == "gradient":  # FCI of the fixture (pkg/tests/fixtures/reference.json)
        assert abs(gpu.energy - vq["fx"]["fixture_fci_energy"]) <= 1e-8


def test_vqe_minimize_workers_partitioned_expectation(vq):
    """workers > 1: vqe_minimize builds the reference's LPT plan and calls
    expectation_parallel (engine.py:454-459) -- on device states that is the
    term-partitioned device expectation (engine.expectation_parallel)."""
    RE = vq["RE"]
    opts = RE.OptimizerOptions(method="simplex", max_iter=40)
    cpu = RE.vqe_minimize(vq["h"], vq["ansatz"], vq["ref"], RE.StateVectorBackend(), opts)
    gpu = RE.vqe_minimize(vq["h"], vq["ansatz"], vq["ref"], _b200(), opts, workers=4)
    assert abs(gpu.energy - cpu.energy) <= REL * abs(cpu.energy)


def test_parameter_shift_gradient_matches(vq):
    RE = vq["RE"]
    theta = np.array([0.13, -0.21])
    cpu = RE.parameter_shift_gradient(vq["ansatz"], theta, vq["h"], RE.StateVectorBackend(), vq["ref"])
    gpu = RE.parameter_shift_gradient(vq["ansatz"], theta, vq["h"], _b200(), vq["ref"])
    assert np.abs(np.asarray(gpu.values) - np.asarray(cpu.values)).max() <= 1e-10
    # and the device adjoint the drivers now get agrees with the shift rule
    import vqekit.statevector as RSV

    be = _b200()
    adj = RSV.reverse_gradient(vq["ansatz"], theta, vq["h"], be.prepare(vq["ref"]))
    assert np.abs(adj - np.asarray(cpu.values)).max() <= 1e-10


def test_vqd_excited_matches_cpu_backend(vq):
    """VQD with the deflated gradient: apply_operator + reverse_gradient_general
    on device states, the deflation's host StateVector round trip included."""
    RE = vq["RE"]
    opts = RE.OptimizerOptions(method="gradient", max_iter=60)
    cpu = RE.vqd_excited(vq["h"], vq["ansatz"], vq["ref"], RE.StateVectorBackend(), k=1,
                         options=opts, restarts=1)
    gpu = RE.vqd_excited(vq["h"], vq["ansatz"], vq["ref"], _b200(), k=1, options=opts, restarts=1)
    for a, b in zip(gpu.energies, cpu.energies):
        assert abs(a - b) <= 1e-9 * max(1.0, abs(b))


def test_fresh_reference_bind_every_evaluation(vq):
    """The reference's bind() returns new Circuit objects every evaluation
    (engine.py:457): the engine recognises the structure and pulls values."""
    RC = vq["RC"]
    be = _b200()
    s0 = be.prepare(vq["ref"])
    rng = np.random.default_rng(3)
    import vqekit.statevector as RSV

    cpu0 = RSV.init_state(vq["ref"])
    for _ in range(3):
        th = rng.uniform(-1, 1, vq["ansatz"].n_params)
        bound = RC.bind(vq["ansatz"], th)
        e = be.expectation(be.evolve(s0, bound), vq["h"])
        e_ref = RSV.expectation(RSV.evolve(cpu0, bound), vq["h"])
        assert abs(e - e_ref) <= REL * max(1.0, abs(e_ref))
    with pytest.raises(RuntimeError):
        be.evolve(s0, vq["ansatz"])  # unbound (statevector.py:69-70)


def test_device_expectation_parallel_worker_invariant():
    """a16 on a device state: LPT partitions of a 16-qubit, 600-string
    Hamiltonian evaluated by the batched device sweeps and reduced in worker
    order -- W in {1, 2, 4, 8} identical to 1e-12 (SPEC acceptance #8) and
    equal to the oracle within 1e-10."""
    from conftest import random_state
    from oracle import oracle as O
    from paper_2208_10978_b200 import engine
    from paper_2208_10978_b200 import statevector as sv
    from paper_2208_10978_b200 import workloads as W

    n = 16
    rng = np.random.default_rng(16)
    h = W.sparse_random_hamiltonian(n, 600, rng, z_only=180)
    st = random_state(n, rng)
    s = sv.from_amplitudes(st)
    vals = [engine.expectation_parallel(s, h, engine.plan_partition(h, w)) for w in (1, 2, 4, 8)]
    assert max(vals) - min(vals) <= 1e-12 * max(1.0, abs(vals[0]))
    e_ref = O.expectation(st, h, n)
    assert abs(vals[0] - e_ref) <= REL * max(1.0, abs(e_ref))
    assert abs(sv.expectation(s, h) - e_ref) <= REL * max(1.0, abs(e_ref))
