"""Backend adapter and term-partitioned expectation -- the drop-in boundary.

``StateVectorBackend`` implements the reference's duck-typed backend protocol
(engine.py:59-75: ``name``, ``supports_reverse_gradient``, ``prepare``,
``evolve``, ``expectation``, ``overlap``), so ``vqe_minimize``,
``parameter_shift_gradient``, ``adapt_vqe`` and ``vqd_excited`` accept it
unchanged.  ``supports_reverse_gradient`` is True once ``integration.install``
has registered the device gradient with the reference's ``statevector``
module: ``vqe_minimize`` calls ``statevector.reverse_gradient`` directly on
the backend's states (engine.py:463-464), and without the registration that
would be the CPU function.

``plan_partition`` / ``expectation_parallel`` are the reference's
Hamiltonian-term data parallelism (engine.py:106-199) on
device states: an LPT split of the terms by Pauli weight, per-partition
partial sums in ascending term order, reduced in ascending worker order
(engine.py:199).  On P GPUs (one process per GPU, every rank holding a
replica of the state -- the zero-swap route for states that fit one GPU,
SURVEY.md 8(e)) worker w's partition is evaluated on rank w mod P and the
partials are gathered; a single GPU evaluates every partition itself.  Either
way the per-term values come from the batched expectation sweeps, so the
energy is W- and P-invariant up to the order of the final float sums.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass

import numpy as np

from . import statevector as sv


class StateVectorBackend:
    name = "sv-b200"

    def __init__(self, device: int = 0):
        self.device = device

    @property
    def supports_reverse_gradient(self) -> bool:
        from . import integration

        return integration.installed()

    def prepare(self, bitstring: str) -> sv.StateVector:
        return sv.init_state(bitstring, self.device)

    def evolve(self, state: sv.StateVector, bound) -> sv.StateVector:
        return sv.evolve(state, bound)

    def expectation(self, state: sv.StateVector, h) -> float:
        return sv.expectation(state, h)

    def overlap(self, a: sv.StateVector, b: sv.StateVector) -> complex:
        return sv.vdot(a, b)

    def reverse_gradient(self, circuit, theta, h, state0: sv.StateVector):
        """Device reverse-mode gradient (statevector.py:153-163 semantics)."""
        return sv.reverse_gradient(circuit, theta, h, state0)


@dataclass(frozen=True)
class ExpectationPlan:
    """LPT assignment of term indices to workers (engine.py:106-128)."""

    n_workers: int
    partitions: tuple[tuple[int, ...], ...]
    costs: tuple[int, ...]

    def __post_init__(self):
        flat = sorted(i for part in self.partitions for i in part)
        if flat != list(range(len(self.costs))):
            raise ValueError("partitions must cover every term exactly once")
        if self.costs:
            bound = sum(self.costs) / self.n_workers + max(self.costs)
            if max(sum(self.costs[i] for i in p) for p in self.partitions) > bound + 1e-9:
                raise ValueError("partition exceeds the LPT balance bound")


def plan_partition(h, workers: int) -> ExpectationPlan:
    """Greedy longest-processing-time split (engine.py:131-147): terms by
    decreasing Pauli weight (ties: lower index first), each to the least
    loaded worker (ties: lower worker)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    costs = tuple(len(t.string.factors) for t in h.terms)
    order = np.lexsort((np.arange(len(costs)), -np.asarray(costs, dtype=np.int64)))
    heap = [(0, w) for w in range(workers)]  # (load, worker): min-heap order = the tie rule
    parts: list[list[int]] = [[] for _ in range(workers)]
    for idx in order.tolist():
        load, w = heapq.heappop(heap)
        parts[w].append(idx)
        heapq.heappush(heap, (load + costs[idx], w))
    return ExpectationPlan(workers, tuple(tuple(sorted(p)) for p in parts), costs)


def _rank_world(comm) -> tuple[int, int]:
    if comm is None or getattr(comm, "rank", None) is None:
        return 0, 1  # single process (LoopbackComm owns every worker)
    return comm.rank, comm.world


def expectation_parallel(state, h, plan, comm=None, engine=None) -> float:
    """<state|H|state> split over the plan's workers (engine.py:177-199).

    state: a device StateVector (the rank's replica when comm is a
    ProcessGroupComm; every rank passes the same state and plan).  Worker w
    sums coef_t.real * Re<P_t> over its partition in ascending term order
    (engine.py:150-159); partials are summed in ascending worker order
    (engine.py:199).  engine: local per-term evaluator (default: the CUDA
    engine on the state's device; tests pass the oracle engine)."""
    if not sv._is_hermitian(h):
        raise ValueError("expectation requires a Hermitian operator")
    if not h.terms:
        return 0.0
    if engine is None:
        from .distributed import CudaEngine

        engine = CudaEngine(state.device)
    n = state.n_qubits
    x, y, z, cr, _ = sv._hamiltonian(h, n)
    rank, world = _rank_world(comm)
    W = plan.n_workers
    mine = [w for w in range(W) if w % world == rank]
    idx = np.asarray(sorted(i for w in mine for i in plan.partitions[w]), dtype=np.int64)
    per = np.zeros(len(cr), dtype=np.float64)
    if len(idx):
        per[idx] = engine.expectation_terms(state, np.ascontiguousarray(x[idx]),
                                            np.ascontiguousarray(y[idx]),
                                            np.ascontiguousarray(z[idx]))
    partials = np.zeros(W, dtype=np.float64)
    for w in mine:
        acc = 0.0
        for i in plan.partitions[w]:
            acc += float(cr[i]) * float(per[i])
        partials[w] = acc
    if world > 1:
        gathered = comm.gather_partials({rank: partials})
        partials = np.array([gathered[w % world][w] for w in range(W)])
    return float(sum(partials.tolist()))
