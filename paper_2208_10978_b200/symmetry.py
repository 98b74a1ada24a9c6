"""Index-parity reduction of rotation programs (exact).

A Pauli rotation exp(-i theta/2 P) moves amplitude only between the indices i
and i ^ x of a pair, x = the X/Y positions of P.  When every rotation of a
circuit has an even-weight x -- a particle-number-conserving ansatz: UCC
singles flip (i, a), doubles (i, j, a, b) -- the parity of popcount(i) is
conserved, so an evolve from a basis state |b> (every energy evaluation,
statevector.py:65-74 from init_state) never leaves b's parity class: the other
half of the 2^n amplitudes stays exactly zero.  Here that class is evolved as
an (n-1)-qubit state: index i of the class <-> i without its top bit, the top
bit being a function of the rest (top = cls ^ parity(low bits)).

Each string P = i^ny X^x Z^zm (zm = Y|Z positions, ny = |Y|) acts on the
half as sigma * P'' with P'' the (n-1)-qubit string of X-part x_low and
Z-part zm'' = zm_low ^ (zm_top ? all ones : 0), and sigma = i^(ny - ny'')
(-1)^(zm_top * cls) = +-1 (ny'' = |x_low & zm''|; P restricted to the class is
Hermitian, so sigma is real).  So the half program is the same rotations with
new strings and angles sigma * theta, and <psi|P|psi> = sigma <half|P''|half>
for the Hamiltonian's even-flip terms; odd-flip terms map the class to the
other one and contribute exactly 0.  `QSV_PARITY=0` turns the reduction off.
"""

from __future__ import annotations

import os
import zlib

import numpy as np

from . import _lib


def enabled() -> bool:
    return os.environ.get("QSV_PARITY", "1") != "0"


def _popc(v: np.ndarray) -> np.ndarray:
    v = v.astype(np.uint64)
    c = np.zeros(v.shape, dtype=np.int64)
    while np.any(v):
        c += (v & np.uint64(1)).astype(np.int64)
        v >>= np.uint64(1)
    return c


def transform_strings(n: int, x, y, z):
    """(x'', y'', z'', sigma0, zm_top) of the (n-1)-qubit strings; sigma0 = i^(ny - ny'')
    (+-1) and the class sign (-1)^(zm_top * cls) stays separate.  Requires even flips."""
    x = np.asarray(x, dtype=np.uint64)
    y = np.asarray(y, dtype=np.uint64)
    z = np.asarray(z, dtype=np.uint64)
    top = np.uint64(n - 1)
    topbit = np.uint64(1) << top
    wlow = topbit - np.uint64(1)
    xm, zm = x | y, y | z
    x_low = xm & wlow
    zm_top = ((zm >> top) & np.uint64(1)).astype(np.int64)
    zmm = (zm & wlow) ^ (wlow * zm_top.astype(np.uint64))
    y2 = x_low & zmm
    x2 = x_low & ~zmm & wlow
    z2 = zmm & ~x_low & wlow
    dny = (_popc(y) - _popc(y2)) % 4
    if np.any(dny % 2):
        raise AssertionError("odd phase difference: not an even-flip string")
    sigma0 = np.where(dny == 0, 1.0, -1.0)
    return x2, y2, z2, sigma0, zm_top


def _flat_evolution(n: int, x2, y2, z2):
    """Flat gate list of the half program: circuit.py:271-281's pattern
    (basis layer ascending, CNOT ladder, RZ on the last support qubit,
    mirror) per string; returns kinds, qubits and each rotation's RZ index."""
    codes = _lib.KIND_CODES
    kH, kHY, kCX, kRZ = codes["H"], codes["HY"], codes["CNOT"], codes["RZ"]
    kinds, qubits, rz_at = [], [], []
    for xs, ys, zs in zip(x2.tolist(), y2.tolist(), z2.tolist()):
        supp = [q for q in range(n) if ((xs | ys | zs) >> q) & 1]
        basis = [(kH if (xs >> q) & 1 else kHY, q) for q in supp if ((xs | ys) >> q) & 1]
        for k, q in basis:
            kinds.append(k)
            qubits += [q, -1]
        for a, b in zip(supp[:-1], supp[1:]):
            kinds.append(kCX)
            qubits += [a, b]
        rz_at.append(len(kinds))
        kinds.append(kRZ)
        qubits += [supp[-1], -1]
        for a, b in reversed(list(zip(supp[:-1], supp[1:]))):
            kinds.append(kCX)
            qubits += [a, b]
        for k, q in basis:
            kinds.append(k)
            qubits += [q, -1]
    return (np.asarray(kinds, dtype=np.int32), np.asarray(qubits, dtype=np.int32),
            np.asarray(rz_at, dtype=np.int64))


class Reduction:
    """The half program of one circuit structure (angles come per call)."""

    def __init__(self, n: int, kinds, qubits):
        spans, masks = _lib.match_rotations(n, kinds, qubits)
        if len(spans) == 0 or int(spans[:, 1].sum()) != len(kinds):
            raise ValueError("not a rotation-only program")
        x, y, z = masks[:, 0], masks[:, 1], masks[:, 2]
        if np.any(_popc(x | y) % 2) or np.any((x | y) == 0):
            raise ValueError("odd or empty flips: index parity not conserved")
        self.n = n
        src = spans[:, 2].astype(np.int64)  # RZ gate of each rotation (angle = values[3 * src])
        x2, y2, z2, sigma0, zm_top = transform_strings(n, x, y, z)
        if np.any((x2 | y2) == 0):
            raise ValueError("a string reduces to a diagonal one")
        # A string with Z (or Y) on the eliminated qubit gets the complemented
        # Z-chain, so the strings of one excitation no longer share their sign
        # bits off the flip and would fuse into one table per run.  Within a
        # run of same-flip strings that all commute (the 8 strings of a UCC
        # double do) group equal Z masks together: two fused tables instead
        # of up to eight.
        order = np.arange(len(src))
        fl = x2 | y2
        i = 0
        while i < len(src):
            j = i + 1
            while j < len(src) and fl[j] == fl[i]:
                j += 1
            if j - i > 2:
                zm = (y2 | z2)[i:j]
                d = zm[:, None] ^ zm[None, :]
                if not np.any(_popc((d & fl[i]).ravel()) % 2):
                    zk = z2[i:j]
                    first = {}
                    for k, v in enumerate(zk.tolist()):
                        first.setdefault(v, k)
                    order[i:j] = i + np.array(sorted(range(j - i), key=lambda k: (first[zk[k]], k)))
            i = j
        self.src, self.sigma0, self.zm_top = src[order], sigma0[order], zm_top[order]
        x2, y2, z2 = x2[order], y2[order], z2[order]
        self.kinds, self.qubits, self.rz_at = _flat_evolution(n - 1, x2, y2, z2)
        self.x2, self.y2, self.z2 = x2, y2, z2
        self._prog = None

    def half_values(self, values, cls: int) -> np.ndarray:
        v = np.zeros(3 * len(self.kinds), dtype=np.float64)
        sign = self.sigma0 * np.where(self.zm_top * cls % 2 == 1, -1.0, 1.0)
        v[3 * self.rz_at] = sign * np.asarray(values, dtype=np.float64)[3 * self.src]
        return v

    def program(self):
        if self._prog is None:
            from .statevector import _Program
            self._prog = _Program(self.n - 1, self.kinds, self.qubits)
        return self._prog


_CACHE: dict = {}
_CACHE_MAX = 16


def reduction_for(n: int, kinds, qubits):
    """The Reduction of a structure, or None when the program is not an
    even-flip rotation program (cached per structure, misses too)."""
    key = (n, len(kinds), zlib.crc32(np.ascontiguousarray(kinds).view(np.uint8)),
           zlib.crc32(np.ascontiguousarray(qubits).view(np.uint8)))
    if key in _CACHE:
        return _CACHE[key]
    try:
        red = Reduction(n, kinds, qubits)
    except ValueError:
        red = None
    if len(_CACHE) >= _CACHE_MAX:
        _CACHE.pop(next(iter(_CACHE)))
    _CACHE[key] = red
    return red


_TERMS: dict = {}


def half_terms(n: int, x, y, z, cr, ci, cls: int):
    """Hamiltonian arrays on the half: the even-flip terms, transformed, with
    coefficients times sigma; and the indices of the kept terms."""
    key = (n, cls, x.ctypes.data, len(x), zlib.crc32(np.ascontiguousarray(x).view(np.uint8)),
           zlib.crc32(np.ascontiguousarray(z).view(np.uint8)), zlib.crc32(np.ascontiguousarray(cr).view(np.uint8)))
    hit = _TERMS.get(key)
    if hit is not None:
        return hit
    keep = np.nonzero(_popc(np.asarray(x | y, dtype=np.uint64)) % 2 == 0)[0]
    x2, y2, z2, s0, ztop = transform_strings(n, x[keep], y[keep], z[keep])
    sign = s0 * np.where(ztop * cls % 2 == 1, -1.0, 1.0)
    out = (np.ascontiguousarray(x2), np.ascontiguousarray(y2), np.ascontiguousarray(z2),
           np.ascontiguousarray(cr[keep] * sign), np.ascontiguousarray(ci[keep] * sign), keep, sign)
    if len(_TERMS) >= 8:
        _TERMS.pop(next(iter(_TERMS)))
    _TERMS[key] = out
    return out
