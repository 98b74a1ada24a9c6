"""Kernel plugin seam -- mirror of the reference's vqekit.kernels
(kernels/__init__.py:20-23) with the same three entry points, operating on
device-resident ``StateVector`` objects instead of NumPy buffers.

Unlike the reference (kernels/__init__.py:12-18) there is no fallback: the
CUDA library is the implementation, and importing it fails loudly when
libqsv.so has not been built.
"""

from __future__ import annotations

import numpy as np

from . import _lib

_lib.lib()  # fail at import time if the CUDA extension is missing

IMPLEMENTATION = "cuda-sm_100a"


def apply_1q(state, matrix, qubit: int) -> None:
    """In-place 2x2 gate (_cykernels.pyx:19-38)."""
    m = np.ascontiguousarray(matrix, dtype=np.complex128)
    if m.shape != (2, 2):
        raise ValueError("apply_1q expects a 2x2 matrix")
    _lib.check(_lib.lib().qsv_apply_1q(state.handle, _lib.dptr(m.view(np.float64)), int(qubit)))


def apply_2q(state, matrix, q0: int, q1: int) -> None:
    """In-place 4x4 gate, rows indexed by (bit q0, bit q1) (_cykernels.pyx:41-73)."""
    m = np.ascontiguousarray(matrix, dtype=np.complex128)
    if m.shape != (4, 4):
        raise ValueError("apply_2q expects a 4x4 matrix")
    _lib.check(_lib.lib().qsv_apply_2q(state.handle, _lib.dptr(m.view(np.float64)), int(q0), int(q1)))


def apply_matrix(state, matrix, qubits) -> None:
    """In-place dense k-qubit gate (k = 1..5); rows indexed by the target bits
    with qubits[0] as the most significant (the apply_2q convention,
    _cykernels.pyx:41-73, extended to k qubits)."""
    qs = np.ascontiguousarray([int(q) for q in qubits], dtype=np.int32)
    k = len(qs)
    m = np.ascontiguousarray(matrix, dtype=np.complex128)
    if m.shape != (1 << k, 1 << k):
        raise ValueError(f"apply_matrix expects a {1 << k}x{1 << k} matrix for {k} qubits")
    _lib.check(_lib.lib().qsv_apply_matrix(state.handle, k, _lib.i32ptr(qs), _lib.dptr(m.view(np.float64))))


def apply_pauli(state, x_mask: int, y_mask: int, z_mask: int, out) -> None:
    """Fill ``out`` with P|state> (_cykernels.pyx:76-102)."""
    _lib.check(_lib.lib().qsv_apply_pauli(state.handle, out.handle, int(x_mask), int(y_mask),
                                          int(z_mask)))
