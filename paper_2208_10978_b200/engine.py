"""Backend adapter -- the drop-in boundary.

``StateVectorBackend`` implements the reference's duck-typed backend protocol
(engine.py:59-75: ``name``, ``supports_reverse_gradient``, ``prepare``,
``evolve``, ``expectation``, ``overlap``), so ``vqe_minimize``,
``parameter_shift_gradient``, ``adapt_vqe`` and ``vqd_excited`` accept it
unchanged.  ``supports_reverse_gradient`` stays False: ``vqe_minimize`` would
otherwise call the reference's CPU ``reverse_gradient`` on device states
(engine.py:463-464).  Use it with ``workers=1`` -- the engine parallelises on
the GPU, and CUDA is not fork-safe (engine.py:189-196 forks).

``plan_partition`` restates the reference's LPT term split (engine.py:131-147)
for the multi-GPU expectation in distributed.py; partial sums are reduced in
ascending worker order like engine.py:199.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import statevector as sv


class StateVectorBackend:
    name = "sv-b200"
    supports_reverse_gradient = False

    def __init__(self, device: int = 0):
        self.device = device

    def prepare(self, bitstring: str) -> sv.StateVector:
        return sv.init_state(bitstring, self.device)

    def evolve(self, state: sv.StateVector, bound) -> sv.StateVector:
        return sv.evolve(state, bound)

    def expectation(self, state: sv.StateVector, h) -> float:
        return sv.expectation(state, h)

    def overlap(self, a: sv.StateVector, b: sv.StateVector) -> complex:
        return sv.vdot(a, b)

    def reverse_gradient(self, circuit, theta, h, state0: sv.StateVector):
        """Device reverse-mode gradient (statevector.py:153-163 semantics).
        Callers that want it use this method explicitly: the reference's
        vqe_minimize would route supports_reverse_gradient=True to its own CPU
        statevector.reverse_gradient (engine.py:463-464)."""
        return sv.reverse_gradient(circuit, theta, h, state0)


@dataclass(frozen=True)
class ExpectationPlan:
    n_workers: int
    partitions: tuple[tuple[int, ...], ...]
    costs: tuple[int, ...]


def plan_partition(h, workers: int) -> ExpectationPlan:
    """Greedy longest-processing-time split by Pauli weight, ties by index
    (engine.py:131-147)."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    costs = tuple(len(t.string.factors) for t in h.terms)
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    loads = [0] * workers
    parts: list[list[int]] = [[] for _ in range(workers)]
    for idx in order:
        w = min(range(workers), key=lambda j: (loads[j], j))
        parts[w].append(idx)
        loads[w] += costs[idx]
    return ExpectationPlan(workers, tuple(tuple(sorted(p)) for p in parts), costs)
