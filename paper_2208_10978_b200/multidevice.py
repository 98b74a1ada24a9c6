"""Single-process multi-device state over the native C-ABI handle (qsv_dist_*).

One process drives P = 2^g shards on the listed devices (ids may repeat, so P
shards can share one GPU): the layout, light-cone relayout scheduling and
ascending-rank reduction of distributed.py, but planned and executed in C++
(csrc/qsv_dist.cpp) with cudaMemcpyPeerAsync chunk swaps between devices.
The reference runs its parallel expectation as one process with forked
workers (engine.py:169-199); this is the B200 equivalent for callers that do
not run one process per GPU.  ``MultiDeviceBackend`` implements the backend
protocol (engine.py:59-75).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .circuit import flatten_bound
from .pauli import term_arrays


class MultiDeviceState:
    """Logical n-qubit state sharded over P = len(devices) ranks."""

    def __init__(self, n_qubits: int, devices):
        devs = (ctypes.c_int * len(devices))(*[int(d) for d in devices])
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().qsv_dist_create(ctypes.byref(h), int(n_qubits), len(devices), devs))
        self._h = h
        self.n_qubits = int(n_qubits)
        self.devices = list(devices)

    def __del__(self):
        L = _lib._lib
        h = getattr(self, "_h", None)
        if L is not None and h is not None and h.value:
            L.qsv_dist_destroy(h)
            self._h = None

    def set_basis(self, index: int) -> None:
        _lib.check(_lib.lib().qsv_dist_set_basis(self._h, int(index)))

    def apply(self, circuit) -> None:
        """Apply a bound circuit in place (statevector.py:72-73's gate loop)."""
        if circuit.n_qubits != self.n_qubits:
            raise ValueError("circuit and state qubit counts differ")
        kinds, qubits, values = flatten_bound(circuit)
        _lib.check(_lib.lib().qsv_dist_apply_gates(self._h, len(kinds), _lib.i32ptr(kinds),
                                                   _lib.i32ptr(qubits), _lib.dptr(values)))

    def expectation_terms(self, h) -> tuple[float, float]:
        x, y, z, cr, ci = term_arrays(h, self.n_qubits)
        re, im = ctypes.c_double(), ctypes.c_double()
        _lib.check(_lib.lib().qsv_dist_expectation(self._h, len(cr), _lib.u64ptr(x), _lib.u64ptr(y),
                                                   _lib.u64ptr(z), _lib.dptr(cr), _lib.dptr(ci),
                                                   ctypes.byref(re), ctypes.byref(im)))
        return re.value, im.value

    @property
    def amplitudes(self) -> np.ndarray:
        out = np.empty(1 << self.n_qubits, dtype=np.complex128)
        _lib.check(_lib.lib().qsv_dist_download(self._h, out.ctypes.data_as(ctypes.c_void_p)))
        return out

    def info(self) -> dict:
        P, nl = ctypes.c_int(), ctypes.c_int()
        rel, sent = ctypes.c_int64(), ctypes.c_int64()
        perm = np.zeros(self.n_qubits, dtype=np.int32)
        _lib.check(_lib.lib().qsv_dist_info(self._h, ctypes.byref(P), ctypes.byref(nl), ctypes.byref(rel),
                                            ctypes.byref(sent), _lib.i32ptr(perm)))
        p2p, swaps = ctypes.c_int(), ctypes.c_int64()
        _lib.check(_lib.lib().qsv_dist_p2p_info(self._h, ctypes.byref(p2p), ctypes.byref(swaps)))
        return {"ranks": P.value, "local_qubits": nl.value, "relayouts": rel.value,
                "bytes_sent_per_rank": sent.value, "perm": perm.tolist(),
                "p2p": bool(p2p.value), "swap_launches": swaps.value}


class MultiDeviceBackend:
    """Backend protocol (engine.py:59-75) over the native multi-device state.
    prepare() is lazy; evolve() returns a new state (statevector.py:71)."""

    name = "sv-b200-multidevice"
    supports_reverse_gradient = False

    def __init__(self, devices):
        self.devices = list(devices)

    def prepare(self, bitstring: str):
        n = len(bitstring)
        if n == 0 or any(c not in "01" for c in bitstring):
            raise ValueError(f"invalid bitstring {bitstring!r}")
        return ("basis", n, sum(1 << k for k, c in enumerate(bitstring) if c == "1"))

    def evolve(self, state, bound) -> MultiDeviceState:
        if not isinstance(state, tuple):
            raise NotImplementedError("evolve of a non-basis multi-device state: use apply() in place")
        _, n, index = state
        out = MultiDeviceState(n, self.devices)
        out.set_basis(index)
        out.apply(bound)
        return out

    def expectation(self, state: MultiDeviceState, h) -> float:
        if not h.is_hermitian():
            raise ValueError("expectation requires a Hermitian operator (real coefficients)")
        re, im = state.expectation_terms(h)
        if abs(im) > 1e-10:
            raise ArithmeticError(f"expectation has imaginary residue {im:.3e}")
        return re

    def overlap(self, a: MultiDeviceState, b: MultiDeviceState) -> complex:
        """np.vdot (engine.py:74-75) of the logical amplitudes (host copies:
        for the sizes VQD deflation uses)."""
        return complex(np.vdot(a.amplitudes, b.amplitudes))
