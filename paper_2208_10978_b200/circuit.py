"""Gate-level circuit IR consumed by the engine.

Mirrors the input contract of the reference's circuit module
(circuit.py:27-156): the closed gate set {H, HY, X, CNOT, SWAP, RZ, RY, U3,
CU3}; the first qubit of a two-qubit gate is the control and the
most-significant bit of its 4x4 matrix (circuit.py:5-6); parameters are
``Constant`` or ``Affine`` (scale * theta[index] + offset) and ``bind``
evaluates them.  The engine consumes circuits duck-typed (``gate.kind``,
``gate.qubits``, ``gate.params``/``gate.bound_values()``), so reference
``Circuit`` objects work unchanged; these classes let the engine run without
the reference.  ``pauli_evolution`` reproduces the gate pattern of
circuit.py:254-281 exactly -- that pattern is what the native planner
recognises and turns back into one direct Pauli rotation.
"""

from __future__ import annotations

import contextlib
import json
import math
from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

from . import _lib

GATE_QUBITS = {"H": 1, "HY": 1, "X": 1, "RZ": 1, "RY": 1, "U3": 1, "CNOT": 2, "SWAP": 2, "CU3": 2}
GATE_PARAMS = {"H": 0, "HY": 0, "X": 0, "CNOT": 0, "SWAP": 0, "RZ": 1, "RY": 1, "U3": 3, "CU3": 3}


@dataclass(frozen=True)
class Constant:
    value: float

    def evaluate(self, theta) -> float:
        return self.value


@dataclass(frozen=True)
class Affine:
    index: int
    scale: float
    offset: float = 0.0

    def __post_init__(self):
        if self.index < 0:
            raise ValueError("negative parameter index")
        if not math.isfinite(self.scale) or self.scale == 0.0:
            raise ValueError("affine scale must be finite and non-zero")

    def evaluate(self, theta) -> float:
        return self.scale * theta[self.index] + self.offset


@dataclass(frozen=True)
class Gate:
    kind: str
    qubits: tuple[int, ...]
    params: tuple = ()

    def __post_init__(self):
        if self.kind not in GATE_QUBITS:
            raise ValueError(f"unknown gate kind {self.kind!r}")
        object.__setattr__(self, "qubits", tuple(self.qubits))
        object.__setattr__(self, "params", tuple(self.params))
        if len(self.qubits) != GATE_QUBITS[self.kind]:
            raise ValueError(f"{self.kind} expects {GATE_QUBITS[self.kind]} qubits")
        if len(set(self.qubits)) != len(self.qubits):
            raise ValueError("gate qubit indices must be distinct")
        if any(q < 0 for q in self.qubits):
            raise ValueError("negative qubit index")
        if len(self.params) != GATE_PARAMS[self.kind]:
            raise ValueError(f"{self.kind} expects {GATE_PARAMS[self.kind]} parameters")

    def is_bound(self) -> bool:
        return all(isinstance(p, Constant) for p in self.params)

    def bound_values(self) -> tuple[float, ...]:
        if not self.is_bound():
            raise RuntimeError(f"gate {self.kind} has unbound parameters")
        return tuple(p.value for p in self.params)


@dataclass(frozen=True)
class Circuit:
    n_qubits: int
    gates: tuple[Gate, ...] = ()
    n_params: int = 0

    def __post_init__(self):
        object.__setattr__(self, "gates", tuple(self.gates))
        for g in self.gates:
            if any(q >= self.n_qubits for q in g.qubits):
                raise ValueError(f"gate {g.kind} addresses qubit outside 0..{self.n_qubits - 1}")
            for p in g.params:
                if isinstance(p, Affine) and p.index >= self.n_params:
                    raise ValueError(f"parameter index {p.index} out of range")

    def is_bound(self) -> bool:
        return all(g.is_bound() for g in self.gates)

    def __len__(self) -> int:
        return len(self.gates)


class _BindPlan:
    """Flattened parametric structure of a circuit: kinds / qubits as in
    flatten_bound, constant parameter values, and the (slot, index, scale,
    offset) of every Affine parameter -- so bind is O(#params) numpy work."""

    __slots__ = ("n_qubits", "kinds", "qubits", "const", "slot", "index", "scale", "offset", "_pid",
                 "_scratch", "_lock", "__weakref__")

    def __init__(self, c):
        import threading

        self.n_qubits = c.n_qubits
        self._pid = None
        self._scratch = None  # const with one bound circuit's Affine slots, reused per call
        self._lock = threading.Lock()
        gates = c.gates
        G = len(gates)
        codes = _lib.KIND_CODES
        self.kinds = np.empty(G, dtype=np.int32)
        self.qubits = np.full(2 * G, -1, dtype=np.int32)
        self.const = np.zeros(3 * G, dtype=np.float64)
        slot, index, scale, offset = [], [], [], []
        for i, g in enumerate(gates):
            self.kinds[i] = codes[g.kind]
            qs = g.qubits
            self.qubits[2 * i] = qs[0]
            if len(qs) == 2:
                self.qubits[2 * i + 1] = qs[1]
            for k, p in enumerate(g.params):
                if not hasattr(p, "value"):  # Affine (ours or the reference's: duck-typed)
                    slot.append(3 * i + k)
                    index.append(p.index)
                    scale.append(p.scale)
                    offset.append(p.offset)
                else:
                    self.const[3 * i + k] = p.value
        self.slot = np.asarray(slot, dtype=np.int64)
        self.index = np.asarray(index, dtype=np.int64)
        self.scale = np.asarray(scale, dtype=np.float64)
        self.offset = np.asarray(offset, dtype=np.float64)

    @contextlib.contextmanager
    def values_with(self, slot_values):
        """The full 3 x gates value array for these Affine slot values, in a
        buffer reused across calls (held under a lock for the duration of the
        caller's synchronous library call) -- so an energy evaluation at new
        angles does not allocate and fill a fresh 3 x gates array."""
        with self._lock:
            if self._scratch is None:
                self._scratch = self.const.copy()
            if len(self.slot):
                self._scratch[self.slot] = slot_values
            yield self._scratch

    def program_id(self) -> int:
        """Id of this structure prepared in the library (qsv_prepare_gates):
        validated and planned once, released with the plan."""
        if self._pid is None:
            import ctypes
            import weakref

            pid = ctypes.c_int64()
            _lib.check(_lib.lib().qsv_prepare_gates(self.n_qubits, len(self.kinds),
                                                    _lib.i32ptr(self.kinds), _lib.i32ptr(self.qubits),
                                                    ctypes.byref(pid)))
            self._pid = pid.value
            weakref.finalize(self, _release_program, pid.value)
        return self._pid


def _release_program(pid: int) -> None:
    L = _lib._lib
    if L is not None:
        L.qsv_release_program(pid)


_BIND_PLANS: dict = {}  # id(parametric circuit) -> (circuit, plan); small LRU


def _bind_plan(c) -> _BindPlan:
    hit = _BIND_PLANS.get(id(c))
    if hit is not None and hit[0] is c:
        return hit[1]
    plan = _BindPlan(c)
    if len(_BIND_PLANS) >= 8:
        _BIND_PLANS.pop(next(iter(_BIND_PLANS)))
    _BIND_PLANS[id(c)] = (c, plan)
    return plan


class BoundCircuit:
    """Result of ``bind``: a bound circuit whose flattened arrays are computed
    up front (vectorised Affine evaluation, bit-identical to evaluating each
    parameter: scale * theta[index] + offset in float64) and whose Gate
    objects are only built if someone reads ``gates``.  Duck-types Circuit
    (n_qubits, gates, n_params = 0, is_bound, len)."""

    __slots__ = ("n_qubits", "n_params", "_kinds", "_qubits", "_values", "_slot_values", "_src", "_gates",
                 "_plan", "__weakref__")

    def __init__(self, src, kinds, qubits, values, plan=None, slot_values=None):
        self.n_qubits = src.n_qubits
        self.n_params = 0
        self._src = src
        self._plan = plan
        self._kinds, self._qubits, self._values = kinds, qubits, values
        self._slot_values = slot_values  # Affine slots only; the full array on demand
        self._gates = None

    def call_values(self):
        """Context manager yielding the full value array for ONE synchronous
        library call: the materialised array if there is one, else the
        plan's reused scratch filled with this circuit's slot values."""
        if self._values is not None or self._plan is None:
            return contextlib.nullcontext(self.flat()[2])
        return self._plan.values_with(self._slot_values)

    @property
    def gates(self) -> tuple:
        if self._gates is None:
            v = self.flat()[2]
            self._gates = tuple(
                Gate(g.kind, g.qubits, tuple(Constant(float(v[3 * i + k])) for k in range(len(g.params))))
                for i, g in enumerate(self._src.gates))
        return self._gates

    def flat(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        if self._values is None:
            v = self._plan.const.copy()
            if len(self._plan.slot):
                v[self._plan.slot] = self._slot_values
            self._values = v
        return self._kinds, self._qubits, self._values

    def is_bound(self) -> bool:
        return True

    def __len__(self) -> int:
        return len(self._kinds)

    def __eq__(self, other) -> bool:
        if isinstance(other, BoundCircuit):
            other = Circuit(other.n_qubits, other.gates, 0)
        return Circuit(self.n_qubits, self.gates, 0) == other

    __hash__ = None


def bind(c, theta: Sequence[float]) -> BoundCircuit:
    """Evaluate every parameter at theta (circuit.py:145-156).  The parametric
    structure is flattened once per circuit object; each call is then a
    vectorised gather + multiply-add over the Affine slots (~us instead of
    ~ms per 10k gates) and the engine consumes the arrays directly."""
    theta = np.asarray(theta, dtype=float)
    if theta.shape != (c.n_params,):
        raise ValueError(f"expected {c.n_params} parameter values, got {theta.shape}")
    if not np.all(np.isfinite(theta)):
        raise ValueError("parameter values must be finite")
    plan = _bind_plan(c)
    # only the Affine slots are evaluated here; the full value array is built
    # on demand (BoundCircuit.flat) or filled into the plan's scratch for one
    # engine call (BoundCircuit.call_values)
    slot_values = plan.scale * theta[plan.index] + plan.offset if len(plan.slot) else plan.scale[:0]
    return BoundCircuit(c, plan.kinds, plan.qubits, None, plan, slot_values)


def gate_matrix(kind: str, values: Sequence[float] = ()) -> np.ndarray:
    """Dense gate matrix (row-major complex128); same convention as the native
    planner's restatement of circuit.py:198-223."""
    code = _lib.KIND_CODES[kind]
    if kind in ("X", "CNOT", "SWAP"):
        return {
            "X": np.array([[0, 1], [1, 0]], dtype=complex),
            "CNOT": np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=complex),
            "SWAP": np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=complex),
        }[kind]
    v = list(values) + [0.0] * (3 - len(values))
    r = math.sqrt(0.5)
    if code == 0:
        return np.array([[r, r], [r, -r]], dtype=complex)
    if code == 1:
        return np.array([[r, -1j * r], [1j * r, -r]], dtype=complex)
    if kind == "RZ":
        return np.diag([np.exp(-0.5j * v[0]), np.exp(0.5j * v[0])])
    if kind == "RY":
        c, s = math.cos(v[0] / 2), math.sin(v[0] / 2)
        return np.array([[c, -s], [s, c]], dtype=complex)
    c, s = math.cos(v[0] / 2), math.sin(v[0] / 2)
    u = np.array([[c, -np.exp(1j * v[2]) * s], [np.exp(1j * v[1]) * s, np.exp(1j * (v[1] + v[2])) * c]])
    if kind == "U3":
        return u
    out = np.eye(4, dtype=complex)
    out[2:, 2:] = u
    return out


def _u3_derivative(theta: float, phi: float, lam: float, slot: int) -> np.ndarray:
    c, s = math.cos(theta / 2), math.sin(theta / 2)
    if slot == 0:
        return 0.5 * np.array([[-s, -np.exp(1j * lam) * c],
                               [np.exp(1j * phi) * c, -np.exp(1j * (phi + lam)) * s]])
    if slot == 1:
        return np.array([[0, 0], [1j * np.exp(1j * phi) * s, 1j * np.exp(1j * (phi + lam)) * c]])
    return np.array([[0, -1j * np.exp(1j * lam) * s], [0, 1j * np.exp(1j * (phi + lam)) * c]])


def gate_derivative(kind: str, values: Sequence[float], slot: int) -> np.ndarray:
    """d(gate matrix)/d(angle in parameter slot) (circuit.py:226-243); generally non-unitary."""
    if kind == "RZ":
        lam = values[0]
        return np.array([[-0.5j * np.exp(-0.5j * lam), 0], [0, 0.5j * np.exp(0.5j * lam)]])
    if kind == "RY":
        c, s = math.cos(values[0] / 2), math.sin(values[0] / 2)
        return 0.5 * np.array([[-s, -c], [c, -s]], dtype=complex)
    if kind == "U3":
        return _u3_derivative(*values, slot)
    if kind == "CU3":
        out = np.zeros((4, 4), dtype=complex)
        out[2:, 2:] = _u3_derivative(*values, slot)
        return out
    raise ValueError(f"gate kind {kind!r} is not differentiable")


def dagger_gate(g: Gate) -> Gate:
    """Bound gate implementing g^dagger: H, HY, X, CNOT, SWAP are Hermitian;
    RZ/RY negate the angle; U3(t, p, l)^dagger = U3(-t, -l, -p) (same for CU3)."""
    if g.kind in ("H", "HY", "X", "CNOT", "SWAP"):
        return g
    v = g.bound_values()
    if g.kind in ("RZ", "RY"):
        return Gate(g.kind, g.qubits, (Constant(-v[0]),))
    return Gate(g.kind, g.qubits, (Constant(-v[0]), Constant(-v[2]), Constant(-v[1])))


# ---------------------------------------------------------------------------
# Pauli exponentials (gate pattern of circuit.py:254-281)
# ---------------------------------------------------------------------------


def _scaled(expr, factor: float):
    if isinstance(expr, (int, float)):
        return Constant(float(expr) * factor)
    if isinstance(expr, Constant):
        return Constant(expr.value * factor)
    return Affine(expr.index, expr.scale * factor, expr.offset * factor)


def evolution_gates(string, angle) -> list[Gate]:
    """Gates of exp(i * angle * P): basis layer (H for X, HY for Y, ascending
    qubit order), CNOT ladder down the support, RZ(-2 angle) on the last
    support qubit, then the mirror image."""
    support = tuple(q for q, _ in string.factors)
    if not support:
        raise ValueError("cannot build an evolution circuit for the identity string")
    basis = [Gate("H" if a == "X" else "HY", (q,)) for q, a in string.factors if a in ("X", "Y")]
    ladder = [Gate("CNOT", (support[k], support[k + 1])) for k in range(len(support) - 1)]
    rz = Gate("RZ", (support[-1],), (_scaled(angle, -2.0),))
    return basis + ladder + [rz] + ladder[::-1] + basis


def pauli_evolution(string, angle, n_qubits: int) -> Circuit:
    if string.max_index() >= n_qubits:
        raise ValueError("string support exceeds qubit count")
    if isinstance(angle, (int, float)):
        angle = Constant(float(angle))
    n_params = angle.index + 1 if isinstance(angle, Affine) else 0
    return Circuit(n_qubits, tuple(evolution_gates(string, angle)), n_params)


def rotation_circuit(n_qubits: int, rotations: Iterable[tuple[object, float]]) -> Circuit:
    """Bound circuit applying exp(-i theta/2 P) for each (P, theta) in order
    (pauli_evolution(P, -theta/2))."""
    gates: list[Gate] = []
    for string, theta in rotations:
        gates.extend(evolution_gates(string, Constant(-0.5 * float(theta))))
    return Circuit(n_qubits, tuple(gates), 0)


# ---------------------------------------------------------------------------
# Flattening for the C ABI, and the reference's JSON interchange
# (circuit.py:539-579)
# ---------------------------------------------------------------------------


class _FlatStructure:
    """Flattened structure of a gate list (kinds, qubits, parameter slots),
    kept so a fresh circuit object with the same structure -- what the
    reference's bind() returns every evaluation (engine.py:457) -- only needs
    its parameter values pulled."""

    __slots__ = ("kind_list", "qubit_list", "kinds", "qubits", "slots", "n_values")

    def __init__(self, kind_list, qubit_list, param_counts):
        G = len(kind_list)
        codes = _lib.KIND_CODES
        self.kind_list, self.qubit_list = kind_list, qubit_list
        self.kinds = np.fromiter((codes[k] for k in kind_list), dtype=np.int32, count=G)
        q = np.full(2 * G, -1, dtype=np.int32)
        q0 = np.fromiter((qs[0] for qs in qubit_list), dtype=np.int32, count=G)
        q1 = np.fromiter((qs[1] if len(qs) == 2 else -1 for qs in qubit_list), dtype=np.int32, count=G)
        q[0::2], q[1::2] = q0, q1
        self.qubits = q
        pc = np.asarray(param_counts, dtype=np.int64)
        gate_of = np.repeat(np.arange(G, dtype=np.int64), pc)
        first = np.repeat(np.cumsum(pc) - pc, pc)
        self.slots = 3 * gate_of + (np.arange(len(gate_of), dtype=np.int64) - first)
        self.n_values = 3 * G


_FLAT_STRUCTS: list = []  # most recent first


def _unbound() -> RuntimeError:
    return RuntimeError("circuit must be bound before evolution")


def flatten_bound(c) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Bound circuit -> (kinds int32[G], qubits int32[2G], values float64[3G]).
    Raises RuntimeError (statevector.py:69-70) if a parameter is unbound.

    The gate walk is three list comprehensions (kinds, qubits, parameter
    values): a structure seen before is recognised by list equality and its
    arrays reused; only the values are scattered into place."""
    if isinstance(c, BoundCircuit):
        return c.flat()
    gates = c.gates
    kind_list = [g.kind for g in gates]
    qubit_list = [g.qubits for g in gates]
    try:
        pv = [p.value for g in gates for p in g.params]
    except AttributeError:
        raise _unbound() from None
    st = None
    for k, cand in enumerate(_FLAT_STRUCTS):
        if cand.kind_list == kind_list and cand.qubit_list == qubit_list:
            st = cand
            if k:
                _FLAT_STRUCTS.insert(0, _FLAT_STRUCTS.pop(k))
            break
    if st is None:
        st = _FlatStructure(kind_list, qubit_list, [len(g.params) for g in gates])
        _FLAT_STRUCTS.insert(0, st)
        del _FLAT_STRUCTS[4:]
    values = np.zeros(st.n_values, dtype=np.float64)
    if pv:
        if len(pv) != len(st.slots):
            st = _FlatStructure(kind_list, qubit_list, [len(g.params) for g in gates])
        try:
            values[st.slots] = pv
        except (TypeError, ValueError):
            raise _unbound() from None
    return st.kinds, st.qubits, values


def _expr_json(e) -> dict:
    if isinstance(e, Constant):
        return {"type": "const", "value": e.value}
    return {"type": "affine", "index": e.index, "scale": e.scale, "offset": e.offset}


def circuit_to_json(c) -> str:
    return json.dumps({
        "n_qubits": c.n_qubits,
        "n_params": c.n_params,
        "gates": [{"kind": g.kind, "qubits": list(g.qubits), "params": [_expr_json(p) for p in g.params]}
                  for g in c.gates],
    }, separators=(",", ":"))


def circuit_from_json(text: str) -> Circuit:
    d = json.loads(text)

    def expr(o):
        if o["type"] == "const":
            return Constant(float(o["value"]))
        if o["type"] == "affine":
            return Affine(int(o["index"]), float(o["scale"]), float(o.get("offset", 0.0)))
        raise ValueError(f"unknown parameter expression type {o['type']!r}")

    gates = tuple(Gate(g["kind"], tuple(g["qubits"]), tuple(expr(p) for p in g["params"]))
                  for g in d["gates"])
    return Circuit(int(d["n_qubits"]), gates, int(d["n_params"]))
