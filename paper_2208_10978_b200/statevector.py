"""Device-resident dense state-vector simulation on B200 (sm_100a).

Mirror of the reference's statevector module (statevector.py:26-216) for the
hot path: the same names, argument meaning and error behaviour, with the
amplitudes living in HBM behind a libqsv handle instead of a NumPy array.

* ``StateVector`` -- (n_qubits, device amplitudes); ``.amplitudes`` downloads
  a NumPy copy (the reference's attribute), ``.norm()`` / ``.copy()`` run on
  the GPU.  A state made by ``init_state`` stays a lazy basis state until it
  is first needed, so ``evolve`` writes |index> straight into its output
  instead of copying 16 * 2^n bytes (hard part 1).
* ``evolve`` returns a new state and leaves the input untouched
  (statevector.py:65-74); gates run as fused shared-memory tile passes.
* ``expectation`` keeps the Hermitian check and the 1e-10 imaginary-residue
  check (statevector.py:98-110).

Layout: basis-index bit k is qubit k (statevector.py:4-5).
"""

from __future__ import annotations

import ctypes
import os
import weakref
from typing import Optional

import numpy as np

from . import _lib
from . import symmetry as _symmetry
from .circuit import BoundCircuit, flatten_bound
from .errors import ResourceLimitError
from .pauli import term_arrays

# One B200 holds 2^33 complex128 amplitudes (128 GiB) next to its workspace:
# enough for init_state -> evolve (|index> is synthesised in the output, no
# copy) -> expectation at 33 qubits.  Calls that hold a second state (see
# _alloc) need <= 32 qubits and raise ResourceLimitError, with the sizes, when
# the second state does not fit.  Larger states: distributed.py.
QUBIT_CAP = 33

_POOL: dict[tuple[int, int], list[int]] = {}
_POOL_MAX = 2


def _alloc(n: int, device: int) -> int:
    key = (n, device)
    bucket = _POOL.get(key)
    if bucket:
        return bucket.pop()
    h = ctypes.c_void_p()
    try:
        _lib.check(_lib.lib().qsv_create(ctypes.byref(h), n, device))
    except ResourceLimitError:
        release_pool()  # pooled buffers of other sizes may be what is in the way
        try:
            _lib.check(_lib.lib().qsv_create(ctypes.byref(h), n, device))
        except ResourceLimitError as e:
            free, total = mem_info(device)
            raise ResourceLimitError(
                f"a {n}-qubit state needs {(16 << n) / 2**30:.1f} GiB but device {device} has "
                f"{free / 2**30:.1f} of {total / 2**30:.1f} GiB free; evolve of a non-basis "
                f"state, copy(), apply_rotations, apply_operator, apply_pauli_string, sample and "
                f"reverse_gradient each hold a second state (one B200 fits one 33-qubit state, "
                f"or two 32-qubit states); larger problems shard over GPUs (distributed.py)"
            ) from e
    return h.value


def mem_info(device: int = 0) -> tuple[int, int]:
    """(free, total) device memory in bytes."""
    f, t = ctypes.c_uint64(), ctypes.c_uint64()
    _lib.check(_lib.lib().qsv_mem_info(device, ctypes.byref(f), ctypes.byref(t)))
    return f.value, t.value


def _release(n: int, device: int, h: int) -> None:
    if not h:
        return
    L = _lib._lib
    if L is None:
        return
    L.qsv_download_wait(ctypes.c_void_p(h))  # no copy may outlive its host buffer
    bucket = _POOL.setdefault((n, device), [])
    if len(bucket) < _POOL_MAX and n < 30:
        bucket.append(h)
    else:
        L.qsv_destroy(ctypes.c_void_p(h))


def release_pool() -> None:
    """Free every pooled device buffer."""
    L = _lib._lib
    for bucket in _POOL.values():
        while bucket:
            h = bucket.pop()
            if L is not None:
                L.qsv_destroy(ctypes.c_void_p(h))


class _Handle:
    __slots__ = ("value", "n", "device", "__weakref__")

    def __init__(self, n: int, device: int, value: int):
        self.value = value
        self.n = n
        self.device = device
        weakref.finalize(self, _release, n, device, value)


class StateVector:
    """Dense 2^n complex128 state in device memory (statevector.py:26-39)."""

    __slots__ = ("n_qubits", "device", "_h", "_basis", "_dl_buf")

    def __init__(self, n_qubits: int, amplitudes=None, device: int = 0):
        self.n_qubits = int(n_qubits)
        self.device = device
        self._h: Optional[_Handle] = None
        self._basis: Optional[int] = None
        if amplitudes is not None:
            amps = np.ascontiguousarray(amplitudes, dtype=np.complex128)
            if amps.shape != (1 << self.n_qubits,):
                raise ValueError("amplitude vector length must be 2^n_qubits")
            self._ensure()
            _lib.check(_lib.lib().qsv_upload(self.handle, amps.ctypes.data_as(ctypes.c_void_p)))

    # -- handle management ---------------------------------------------------
    @classmethod
    def _empty(cls, n: int, device: int = 0) -> "StateVector":
        s = cls.__new__(cls)
        s.n_qubits = n
        s.device = device
        s._h = None
        s._basis = None
        s._ensure()
        return s

    @classmethod
    def _basis_state(cls, n: int, index: int, device: int = 0) -> "StateVector":
        s = cls.__new__(cls)
        s.n_qubits = n
        s.device = device
        s._h = None
        s._basis = index
        return s

    def _ensure(self) -> None:
        if self._h is None:
            self._h = _Handle(self.n_qubits, self.device, _alloc(self.n_qubits, self.device))
            if self._basis is not None:
                _lib.check(_lib.lib().qsv_set_basis(self.handle, self._basis))

    @property
    def handle(self) -> ctypes.c_void_p:
        self._ensure()
        return ctypes.c_void_p(self._h.value)

    @property
    def basis_index(self) -> Optional[int]:
        """Index of the basis state if this is an untouched init_state() result."""
        return self._basis if self._h is None else None

    # -- reference attributes -----------------------------------------------
    @property
    def amplitudes(self) -> np.ndarray:
        """Host copy of the amplitudes (NumPy complex128, index order)."""
        out = np.empty(1 << self.n_qubits, dtype=np.complex128)
        self.download_into(out)
        return out

    def download_into(self, out: np.ndarray) -> None:
        if out.dtype != np.complex128 or out.size != (1 << self.n_qubits) or not out.flags.c_contiguous:
            raise ValueError("output must be a contiguous complex128 array of length 2^n")
        _lib.check(_lib.lib().qsv_download(self.handle, out.ctypes.data_as(ctypes.c_void_p)))

    def download_async(self, out: np.ndarray) -> None:
        """Start copying the amplitudes into `out` (pinned memory for a truly
        asynchronous copy) on the device's copy stream; work queued afterwards
        on other states overlaps it.  `wait_download()` completes it; the next
        call that modifies this state waits for it on the device."""
        if out.dtype != np.complex128 or out.size != (1 << self.n_qubits) or not out.flags.c_contiguous:
            raise ValueError("output must be a contiguous complex128 array of length 2^n")
        _lib.check(_lib.lib().qsv_download_async(self.handle, out.ctypes.data_as(ctypes.c_void_p)))
        self._dl_buf = out  # keep the host buffer alive while the copy is in flight

    def wait_download(self) -> None:
        if self._h is not None:
            _lib.check(_lib.lib().qsv_download_wait(self.handle))
        self._dl_buf = None

    def norm(self) -> float:
        if self.basis_index is not None:
            return 1.0
        v = ctypes.c_double()
        _lib.check(_lib.lib().qsv_norm(self.handle, ctypes.byref(v)))
        return v.value

    def copy(self) -> "StateVector":
        if self.basis_index is not None:
            return StateVector._basis_state(self.n_qubits, self._basis, self.device)
        out = StateVector._empty(self.n_qubits, self.device)
        _lib.check(_lib.lib().qsv_copy(out.handle, self.handle))
        return out

    def device_ptr(self) -> int:
        p = ctypes.c_void_p()
        _lib.check(_lib.lib().qsv_device_ptr(self.handle, ctypes.byref(p)))
        return p.value

    @property
    def __cuda_array_interface__(self) -> dict:
        """Zero-copy view as (2^n, 2) float64 for torch.as_tensor / CuPy."""
        return {"shape": (1 << self.n_qubits, 2), "typestr": "<f8",
                "data": (self.device_ptr(), False), "version": 3, "strides": None}

    def synchronize(self) -> None:
        _lib.check(_lib.lib().qsv_synchronize(self.handle))


def _check_cap(n: int) -> None:
    if n > QUBIT_CAP:
        raise ResourceLimitError(
            f"{n} qubits exceeds the single-GPU dense cap of {QUBIT_CAP}; use distributed.py"
        )


def init_state(bitstring: str, device: int = 0) -> StateVector:
    """Computational basis state; character k of the bitstring is qubit k
    (statevector.py:42-54)."""
    n = len(bitstring)
    if n == 0 or any(c not in "01" for c in bitstring):
        raise ValueError(f"invalid bitstring {bitstring!r}")
    _check_cap(n)
    index = sum(1 << k for k, c in enumerate(bitstring) if c == "1")
    return StateVector._basis_state(n, index, device)


def from_amplitudes(amplitudes, device: int = 0) -> StateVector:
    amps = np.ascontiguousarray(amplitudes, dtype=np.complex128)
    n = int(amps.size).bit_length() - 1
    if amps.ndim != 1 or (1 << n) != amps.size:
        raise ValueError("amplitude vector length must be a power of two")
    return StateVector(n, amps, device)


# Per-circuit flattening cache: bound circuits are immutable, so repeated
# evolutions of the same object skip the Python walk over its gates.  Keyed by
# object identity (checked through a weak reference): hashing a frozen
# dataclass circuit hashes every gate -- 12 ms for config 1's 37,824 gates.
_FLAT_CACHE: dict = {}
_FLAT_MAX = 64
_last_stats = _lib.PlanStats()


def _id_cache_get(cache: dict, obj):
    hit = cache.get(id(obj))
    if hit is not None and hit[0]() is obj:
        return hit[1]
    return None


def _id_cache_put(cache: dict, obj, value, limit: int) -> None:
    key = id(obj)

    def _drop(r, cache=cache, key=key):
        # the object died: drop its entry (and with it a prepared program's
        # library-side plan) now instead of at FIFO eviction
        hit = cache.get(key)
        if hit is not None and hit[0] is r:
            del cache[key]

    try:
        ref = weakref.ref(obj, _drop)
    except TypeError:
        return
    if len(cache) >= limit:
        cache.pop(next(iter(cache)))
    cache[key] = (ref, value)


def _flat(c):
    flat = getattr(c, "flat", None)
    if flat is not None and callable(flat):  # BoundCircuit: arrays computed by bind
        return flat()
    hit = _id_cache_get(_FLAT_CACHE, c)
    if hit is not None:
        return hit
    flat = flatten_bound(c)
    _id_cache_put(_FLAT_CACHE, c, flat, _FLAT_MAX)
    return flat


class _Program:
    """A gate structure prepared in the library (qsv_prepare_gates) for one
    circuit object: re-running that object skips the per-call lookup."""

    __slots__ = ("n_qubits", "pid", "__weakref__")

    def __init__(self, n_qubits: int, kinds, qubits):
        pid = ctypes.c_int64()
        _lib.check(_lib.lib().qsv_prepare_gates(n_qubits, len(kinds), _lib.i32ptr(kinds),
                                                _lib.i32ptr(qubits), ctypes.byref(pid)))
        self.n_qubits = n_qubits
        self.pid = pid.value
        weakref.finalize(self, _release_program, pid.value)

    def program_id(self) -> int:
        return self.pid


def _release_program(pid: int) -> None:
    L = _lib._lib
    if L is not None:
        L.qsv_release_program(pid)


_PROG_CACHE: dict = {}


def apply_circuit_inplace(s: StateVector, c, basis: Optional[int] = None) -> None:
    """Apply a bound circuit to s in place (the loop of statevector.py:72-73).
    With basis: s is first set to |basis> (fused into the first pass).  The
    circuit's structure runs as a prepared program (bind() results carry
    theirs; other circuit objects get one on first use); the values are read
    from the circuit every call."""
    L = _lib.lib()
    plan = getattr(c, "_plan", None)
    if plan is not None and plan.n_qubits == s.n_qubits:
        # a bind() result: its values go down for this one synchronous call
        # (the plan's reused buffer -- no fresh 3 x gates array per evaluation)
        with c.call_values() as values:
            if basis is None:
                _lib.check(L.qsv_apply_prepared(s.handle, plan.program_id(), _lib.dptr(values),
                                                ctypes.byref(_last_stats)))
            else:
                _lib.check(L.qsv_evolve_basis_prepared(s.handle, basis, plan.program_id(),
                                                       _lib.dptr(values), ctypes.byref(_last_stats)))
        return
    else:
        kinds, qubits, values = _flat(c)
        plan = _id_cache_get(_PROG_CACHE, c)
        if not isinstance(plan, _Program) or plan.n_qubits != s.n_qubits:
            if plan is None:
                # first run of this object: the library's structure cache
                # (shared by equal structures in different objects)
                _id_cache_put(_PROG_CACHE, c, "seen", _FLAT_MAX)
                if basis is None:
                    _lib.check(L.qsv_apply_gates(s.handle, len(kinds), _lib.i32ptr(kinds),
                                                 _lib.i32ptr(qubits), _lib.dptr(values),
                                                 ctypes.byref(_last_stats)))
                else:
                    _lib.check(L.qsv_evolve_basis(s.handle, basis, len(kinds), _lib.i32ptr(kinds),
                                                  _lib.i32ptr(qubits), _lib.dptr(values),
                                                  ctypes.byref(_last_stats)))
                return
            plan = _Program(s.n_qubits, kinds, qubits)  # re-run: prepare (reuses the cached plan)
            _id_cache_put(_PROG_CACHE, c, plan, _FLAT_MAX)
    if basis is None:
        _lib.check(L.qsv_apply_prepared(s.handle, plan.program_id(), _lib.dptr(values),
                                        ctypes.byref(_last_stats)))
    else:
        _lib.check(L.qsv_evolve_basis_prepared(s.handle, basis, plan.program_id(),
                                               _lib.dptr(values), ctypes.byref(_last_stats)))


class ParityReduced(StateVector):
    """The result of an evolve from a basis state by an even-flip rotation
    program (symmetry.py): only the basis state's index-parity class is
    non-zero, held as an (n-1)-qubit half.  expectation() runs on the half;
    anything else materialises the full state on first use of `handle`
    (qsv_embed_parity), after which it behaves as a plain StateVector."""

    __slots__ = ("_half", "_cls")

    @classmethod
    def _wrap(cls, n: int, half: StateVector, parity: int) -> "ParityReduced":
        s = cls.__new__(cls)
        s.n_qubits = n
        s.device = half.device
        s._h = None
        s._basis = None
        s._half = half
        s._cls = int(parity)
        return s

    @property
    def reduced(self) -> bool:
        return self._h is None

    def _ensure(self) -> None:
        if self._h is None:
            h = _Handle(self.n_qubits, self.device, _alloc(self.n_qubits, self.device))
            wlow = (1 << (self.n_qubits - 1)) - 1
            _lib.check(_lib.lib().qsv_embed_parity(ctypes.c_void_p(h.value), self._half.handle, wlow, self._cls))
            self._h = h
            self._half = None

    @property
    def basis_index(self) -> Optional[int]:
        return None

    def norm(self) -> float:
        return self._half.norm() if self._h is None else StateVector.norm(self)

    def synchronize(self) -> None:
        (self._half if self._h is None else super()).synchronize()


_last_reduction = {"n_eff": None}


def last_reduction() -> dict:
    """{'n_eff': qubits actually evolved} of the last evolve (None: full size)."""
    return dict(_last_reduction)


def evolve(s: StateVector, c) -> StateVector:
    """Apply a bound circuit; returns a new state (statevector.py:65-74)."""
    if c.n_qubits != s.n_qubits:
        raise ValueError("circuit and state qubit counts differ")
    # boundness (statevector.py:69-70) is checked by the flattening itself
    # (RuntimeError on an unbound parameter), before any device work; a
    # bind() result is bound by construction and its value array is only
    # built when a path below needs it
    if isinstance(c, BoundCircuit):
        kinds, qubits = c._kinds, c._qubits
    else:
        kinds, qubits, _ = _flat(c)
    _last_reduction["n_eff"] = None
    if s.basis_index is not None and s.n_qubits > 12 and _symmetry.enabled():
        red = _symmetry.reduction_for(s.n_qubits, kinds, qubits)
        if red is not None:  # the basis state's parity class, as an (n-1)-qubit state
            values = _flat(c)[2]
            b = s.basis_index
            parity = bin(b).count("1") & 1
            half = StateVector._empty(s.n_qubits - 1, s.device)
            _lib.check(_lib.lib().qsv_evolve_basis_prepared(
                half.handle, b & ((1 << (s.n_qubits - 1)) - 1), red.program().program_id(),
                _lib.dptr(red.half_values(values, parity)), ctypes.byref(_last_stats)))
            _last_reduction["n_eff"] = s.n_qubits - 1
            return ParityReduced._wrap(s.n_qubits, half, parity)
    out = StateVector._empty(s.n_qubits, s.device)
    if s.basis_index is not None:  # |index> is synthesised by the first pass
        apply_circuit_inplace(out, c, s.basis_index)
    else:
        _lib.check(_lib.lib().qsv_copy(out.handle, s.handle))
        apply_circuit_inplace(out, c)
    return out


def apply_rotations(s: StateVector, x, y, z, theta) -> StateVector:
    """New state = prod_r exp(-i theta_r/2 P_r) s (direct Pauli-rotation path)."""
    x = np.ascontiguousarray(x, dtype=np.uint64)
    y = np.ascontiguousarray(y, dtype=np.uint64)
    z = np.ascontiguousarray(z, dtype=np.uint64)
    theta = np.ascontiguousarray(theta, dtype=np.float64)
    out = s.copy()
    _lib.check(_lib.lib().qsv_apply_pauli_rotations(out.handle, len(theta), _lib.u64ptr(x),
                                                    _lib.u64ptr(y), _lib.u64ptr(z),
                                                    _lib.dptr(theta), ctypes.byref(_last_stats)))
    return out


def last_plan_stats() -> dict:
    """Planner statistics of the last evolve / apply_rotations / expectation."""
    st = _lib.PlanStats()
    _lib.check(_lib.lib().qsv_last_plan_stats(ctypes.byref(st)))
    return st.as_dict()


_H_CACHE: dict = {}


def _hamiltonian(h, n: int):
    return _hamiltonian_entry(h, n)[0]


def _hamiltonian_entry(h, n: int):
    """(term arrays, their ctypes pointers) of a PauliSum, cached per object:
    an energy loop re-evaluates the same Hamiltonian."""
    hit = _id_cache_get(_H_CACHE, h)
    if hit is not None and hit[0] == n:
        return hit[1]
    arrays = term_arrays(h, n)
    x, y, z, cr, ci = arrays
    ptrs = (_lib.u64ptr(x), _lib.u64ptr(y), _lib.u64ptr(z), _lib.dptr(cr), _lib.dptr(ci))
    _id_cache_put(_H_CACHE, h, (n, (arrays, ptrs)), _FLAT_MAX)
    return arrays, ptrs


def expectation_terms(s: StateVector, h) -> tuple[float, float, np.ndarray]:
    """(Re, Im residue, per-term <P_t>) of <s|H|s>; no Hermitian checks."""
    (x, y, z, cr, ci), ptrs = _hamiltonian_entry(h, s.n_qubits)
    re, im = ctypes.c_double(), ctypes.c_double()
    per = np.zeros(len(cr), dtype=np.float64)
    if isinstance(s, ParityReduced) and s.reduced:
        # even-flip terms on the half (sigma folded into the coefficients);
        # odd-flip terms map the class onto the empty one: exactly 0
        x2, y2, z2, cr2, ci2, keep, sign = _symmetry.half_terms(s.n_qubits, x, y, z, cr, ci, s._cls)
        per2 = np.zeros(len(cr2), dtype=np.float64)
        if len(cr2):
            _lib.check(_lib.lib().qsv_expectation(s._half.handle, len(cr2), _lib.u64ptr(x2), _lib.u64ptr(y2),
                                                  _lib.u64ptr(z2), _lib.dptr(cr2), _lib.dptr(ci2),
                                                  ctypes.byref(re), ctypes.byref(im), _lib.dptr(per2),
                                                  None))
        per[keep] = per2 * sign
        return re.value, im.value, per
    if len(cr):
        _lib.check(_lib.lib().qsv_expectation(s.handle, len(cr), *ptrs, ctypes.byref(re), ctypes.byref(im),
                                              _lib.dptr(per), None))
    return re.value, im.value, per


def _is_hermitian(h) -> bool:
    hit = _id_cache_get(_HERM_CACHE, h)
    if hit is None:
        hit = bool(h.is_hermitian())
        _id_cache_put(_HERM_CACHE, h, hit, _FLAT_MAX)
    return hit


_HERM_CACHE: dict = {}


def expectation(s: StateVector, h) -> float:
    """<s|H|s> (statevector.py:98-110)."""
    if not _is_hermitian(h):
        raise ValueError("expectation requires a Hermitian operator (real coefficients)")
    re, im, _ = expectation_terms(s, h)
    if abs(im) > 1e-10:
        raise ArithmeticError(f"expectation has imaginary residue {im:.3e}")
    return float(re)


def apply_pauli_string(s: StateVector, p) -> StateVector:
    """P|s> (statevector.py:91-95)."""
    x, y, z = _masks(p, s.n_qubits)
    out = StateVector._empty(s.n_qubits, s.device)
    _lib.check(_lib.lib().qsv_apply_pauli(s.handle, out.handle, x, y, z))
    return out


def _masks(p, n: int) -> tuple[int, int, int]:
    x = y = zm = 0
    for q, axis in p.factors:
        if q >= n:
            raise ValueError(f"string index {q} out of range for {n} qubits")
        if axis == "X":
            x |= 1 << q
        elif axis == "Y":
            y |= 1 << q
        else:
            zm |= 1 << q
    return x, y, zm


def apply_operator(s: StateVector, h) -> StateVector:
    """H|s> as a dense (unnormalised) vector (statevector.py:113-121)."""
    x, y, z, cr, ci = _hamiltonian(h, s.n_qubits)
    out = StateVector._empty(s.n_qubits, s.device)
    _lib.check(_lib.lib().qsv_apply_operator(s.handle, out.handle, len(cr), _lib.u64ptr(x),
                                             _lib.u64ptr(y), _lib.u64ptr(z), _lib.dptr(cr),
                                             _lib.dptr(ci)))
    return out


def vdot(a: StateVector, b: StateVector) -> complex:
    """np.vdot(a, b) = sum conj(a) b (engine.py:74-75)."""
    if a.n_qubits != b.n_qubits:
        raise ValueError("state qubit counts differ")
    out = np.zeros(2, dtype=np.float64)
    _lib.check(_lib.lib().qsv_vdot(a.handle, b.handle, _lib.dptr(out)))
    return complex(out[0], out[1])


def sample(s: StateVector, p, shots: int, seed: int) -> float:
    """Shot-based estimate of <P> (statevector.py:124-147): the support is
    rotated into the Z basis (H for X, HY for Y) on a device copy, then the
    kernel draws `shots` outcomes from |psi|^2 with the reference's exact
    Philox4x64-10 stream (numpy seeds the key) and returns the mean parity."""
    from .circuit import Circuit, Gate

    if shots < 1:
        raise ValueError("shots must be >= 1")
    gates = []
    support = 0
    for q, axis in p.factors:
        if q >= s.n_qubits:
            raise ValueError(f"string index {q} out of range for {s.n_qubits} qubits")
        support |= 1 << q
        if axis == "X":
            gates.append(Gate("H", (q,)))
        elif axis == "Y":
            gates.append(Gate("HY", (q,)))
    rotated = evolve(s, Circuit(s.n_qubits, tuple(gates), 0)) if gates else s.copy()
    key = np.ascontiguousarray(np.random.Philox(seed).state["state"]["key"], dtype=np.uint64)
    mean = ctypes.c_double()
    _lib.check(_lib.lib().qsv_sample_parity(rotated.handle, support, int(shots), _lib.u64ptr(key),
                                            ctypes.byref(mean), None))
    return float(mean.value)


def reverse_gradient(c, theta, h, s0: StateVector) -> np.ndarray:
    """Gradient of <psi(theta)|H|psi(theta)> over all parameters in one
    backward sweep with a single application of H (statevector.py:153-163)."""
    if not _is_hermitian(h):
        raise ValueError("reverse-mode gradient requires a Hermitian operator")
    return reverse_gradient_general(c, theta, lambda s: apply_operator(s, h), s0)


_ROT_PROG_CACHE: dict = {}


def _rotation_program(c):
    """If every gate of c sits in a recognised pauli_evolution block
    (circuit.py:271-281) and the only parameters are the blocks' RZ angles,
    return (x, y, z masks, rz gate index per block); else None."""
    from .circuit import _bind_plan

    plan = _bind_plan(c)
    G = len(plan.kinds)
    if G == 0:
        return None
    spans, masks = _lib.match_rotations(c.n_qubits, plan.kinds, plan.qubits)
    if len(spans) == 0 or spans[0, 0] != 0 or int(spans[:, 1].sum()) != G:
        return None
    if np.any(spans[1:, 0] != spans[:-1, 0] + spans[:-1, 1]):
        return None
    rz = spans[:, 2]
    if not np.all(np.isin(plan.slot, 3 * rz)):
        return None
    return (np.ascontiguousarray(masks[:, 0]), np.ascontiguousarray(masks[:, 1]),
            np.ascontiguousarray(masks[:, 2]), rz)


def _rotation_gradient(c, theta, apply_h, s0: StateVector, prog) -> np.ndarray:
    """Device adjoint sweep over the rotations (qsv_rotation_adjoint): the
    block angle is its RZ value, dE/dtheta_k = sum over blocks of
    scale * Im <lam_r|P_r|phi_r>."""
    from .circuit import _bind_plan, bind

    x, y, z, rz = prog
    bound = bind(c, theta)
    plan = _bind_plan(c)
    block_of_slot = np.searchsorted(3 * rz, plan.slot)
    # the block angles straight from the bound Affine slots (no 3 x gates array)
    angles = np.ascontiguousarray(plan.const[3 * rz])
    if len(plan.slot):
        angles[block_of_slot] = bound._slot_values
    psi = evolve(s0, bound)
    lam = apply_h(psi)
    g = np.zeros(len(rz), dtype=np.float64)
    _lib.check(_lib.lib().qsv_rotation_adjoint(psi.handle, lam.handle, len(rz), _lib.u64ptr(x),
                                               _lib.u64ptr(y), _lib.u64ptr(z), _lib.dptr(angles),
                                               _lib.dptr(g)))
    grad = np.zeros(c.n_params, dtype=np.float64)
    np.add.at(grad, plan.index, plan.scale * g[block_of_slot])
    return grad


def reverse_gradient_general(c, theta, apply_h, s0: StateVector) -> np.ndarray:
    """Reverse-mode sweep (Algorithm 1, statevector.py:166-211) on device states.

    Forward evolve to |psi>, |psi_l> = H|psi>, |psi_r> = |psi>; walking the
    gates backwards, each Affine slot contributes scale * 2 Re <psi_l| dU |psi_r>
    with psi_r the state before the gate and psi_l the back-propagated H|psi>
    after it (psi_l is not renormalised).  B200 form: runs of gates without
    Affine parameters are un-applied as ONE fused gate list per state (the
    planner's tile passes), and RZ / RY slots use dU = -i/2 P U with U, P
    commuting, i.e. 2 Re <psi_l|dU|psi_before> = Im <U^dag psi_l| P |psi_before>:
    one apply_pauli + one vdot instead of a copy, a derivative pass and a vdot.
    """
    from .circuit import Circuit, bind, dagger_gate, gate_derivative
    from . import kernels

    theta = np.asarray(theta, dtype=float)
    if theta.shape != (c.n_params,):
        raise ValueError(f"expected {c.n_params} parameter values, got {theta.shape}")
    # circuits made of pauli_evolution blocks (UCC ansatze; only RZ angles
    # are parameters): one device-side adjoint sweep over the rotations
    if os.environ.get("QSV_ROTATION_ADJOINT", "1") != "0":
        prog = _id_cache_get(_ROT_PROG_CACHE, c)
        if prog is None:
            prog = (_rotation_program(c),)
            _id_cache_put(_ROT_PROG_CACHE, c, prog, _FLAT_MAX)
        if prog[0] is not None:
            return _rotation_gradient(c, theta, apply_h, s0, prog[0])
    for gate in c.gates:
        if gate.params and gate.kind not in ("RZ", "RY", "U3", "CU3"):
            raise ValueError(f"gate kind {gate.kind} is not differentiable")
    n = c.n_qubits
    bound = bind(c, theta)
    psi = evolve(s0, bound)
    psi_l = apply_h(psi)
    psi_r = psi
    grad = np.zeros(c.n_params)
    pend_r: list = []
    pend_l: list = []
    scratch = None

    def flush(state, pend):
        if pend:
            apply_circuit_inplace(state, Circuit(n, tuple(pend), 0))
            pend.clear()

    for gate, bg in zip(reversed(c.gates), reversed(bound.gates)):
        # Affine slots (ours or the reference's: duck-typed, no .value)
        slots = [(k, e) for k, e in enumerate(gate.params) if not hasattr(e, "value")]
        d = dagger_gate(bg)
        if not slots:
            pend_r.append(d)
            pend_l.append(d)
            continue
        pend_r.append(d)  # psi_r -> state before the gate
        if gate.kind in ("RZ", "RY"):
            pend_l.append(d)  # psi_l -> U^dag psi_l (U commutes with its generator)
            flush(psi_r, pend_r)
            flush(psi_l, pend_l)
            if scratch is None:
                scratch = StateVector._empty(n, psi_r.device)
            q = gate.qubits[0]
            pm = (0, 0, 1 << q) if gate.kind == "RZ" else (0, 1 << q, 0)
            _lib.check(_lib.lib().qsv_apply_pauli(psi_r.handle, scratch.handle, *pm))
            v = vdot(psi_l, scratch)
            for k, e in slots:
                grad[e.index] += e.scale * v.imag
        else:
            flush(psi_r, pend_r)
            flush(psi_l, pend_l)
            values = bg.bound_values()
            for k, e in slots:
                work = psi_r.copy()
                dm = np.ascontiguousarray(gate_derivative(gate.kind, values, k))
                if len(gate.qubits) == 1:
                    kernels.apply_1q(work, dm, gate.qubits[0])
                else:
                    kernels.apply_2q(work, dm, gate.qubits[0], gate.qubits[1])
                grad[e.index] += e.scale * 2.0 * vdot(psi_l, work).real
            pend_l.append(d)
    return grad


def dump_state(s: StateVector) -> bytes:
    """Little-endian complex-double amplitude dump (statevector.py:214-216)."""
    return s.amplitudes.astype("<c16").tobytes()
