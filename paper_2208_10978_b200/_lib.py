"""ctypes binding of libqsv.so (include/qsv.h).

The CUDA library is the only compute path of this package: if it is missing
or no sm_100 device is visible, the first call raises -- there is no CPU
fallback.  ctypes releases the GIL for the duration of each call.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ResourceLimitError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libqsv.so")

QSV_OK = 0
QSV_ERR_INVALID = 1
QSV_ERR_CUDA = 2
QSV_ERR_NOMEM = 3
QSV_ERR_RESOURCE = 4

# Gate kind codes of the C ABI (reference gate set, circuit.py:27-34).
KIND_CODES = {"H": 0, "HY": 1, "X": 2, "CNOT": 3, "SWAP": 4, "RZ": 5, "RY": 6, "U3": 7, "CU3": 8}


class QsvCudaError(RuntimeError):
    """The CUDA runtime failed (no device, launch failure, ...)."""


class PlanStats(ctypes.Structure):
    _fields_ = [
        ("n_input_ops", ctypes.c_int64),
        ("n_rotations", ctypes.c_int64),
        ("n_items", ctypes.c_int64),
        ("n_passes", ctypes.c_int64),
        ("n_fallback", ctypes.c_int64),
        ("tile_bits", ctypes.c_int32),
        ("cache_hit", ctypes.c_int32),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


# Every symbol include/qsv.h declares (checked by tests/test_abi_cpu.py).
EXPORTED = (
    "qsv_abi_version", "qsv_last_error", "qsv_device_count", "qsv_mem_info", "qsv_create", "qsv_destroy",
    "qsv_n_qubits", "qsv_set_stream", "qsv_get_stream", "qsv_device_ptr", "qsv_synchronize",
    "qsv_copy", "qsv_set_basis", "qsv_upload", "qsv_download", "qsv_download_async",
    "qsv_download_wait", "qsv_apply_1q", "qsv_apply_2q", "qsv_apply_matrix",
    "qsv_apply_pauli", "qsv_apply_gates", "qsv_apply_pauli_rotations", "qsv_expectation",
    "qsv_apply_operator", "qsv_vdot", "qsv_norm", "qsv_axpby", "qsv_plan_gates",
    "qsv_plan_expectation", "qsv_match_rotations", "qsv_debug_plan_json", "qsv_debug_sweep_source", "qsv_debug_pass_source", "qsv_sample_parity",
    "qsv_jit_info", "qsv_small_info", "qsv_embed_parity", "qsv_rotation_adjoint", "qsv_prepare_gates", "qsv_apply_prepared",
    "qsv_release_program", "qsv_evolve_basis", "qsv_evolve_basis_prepared",
    "qsv_last_plan_stats", "qsv_dist_create", "qsv_dist_destroy", "qsv_dist_set_basis",
    "qsv_dist_apply_gates", "qsv_dist_expectation", "qsv_dist_download", "qsv_dist_info", "qsv_dist_p2p_info", "qsv_ipc_get_handle",
    "qsv_ipc_open", "qsv_ipc_close", "qsv_swap_peer", "qsv_swap_info",
)

_lib = None


def _declare(L):
    vp, dp, i64 = ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64
    u64, u64p = ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64)
    i32p = ctypes.POINTER(ctypes.c_int32)
    sp = ctypes.POINTER(PlanStats)
    sig = {
        "qsv_abi_version": ([], ctypes.c_int),
        "qsv_last_error": ([], ctypes.c_char_p),
        "qsv_device_count": ([ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
        "qsv_mem_info": ([ctypes.c_int, u64p, u64p], ctypes.c_int),
        "qsv_dist_create": ([ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int)],
                            ctypes.c_int),
        "qsv_dist_destroy": ([vp], ctypes.c_int),
        "qsv_dist_set_basis": ([vp, u64], ctypes.c_int),
        "qsv_dist_apply_gates": ([vp, i64, i32p, i32p, dp], ctypes.c_int),
        "qsv_dist_expectation": ([vp, i64, u64p, u64p, u64p, dp, dp, dp, dp], ctypes.c_int),
        "qsv_dist_download": ([vp, vp], ctypes.c_int),
        "qsv_ipc_get_handle": ([vp, ctypes.c_void_p], ctypes.c_int),
        "qsv_ipc_open": ([ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)], ctypes.c_int),
        "qsv_ipc_close": ([ctypes.c_int, ctypes.c_void_p], ctypes.c_int),
        "qsv_swap_peer": ([vp, u64, ctypes.c_void_p, u64, u64], ctypes.c_int),
        "qsv_swap_info": ([ctypes.POINTER(i64)], ctypes.c_int),
        "qsv_dist_p2p_info": ([vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(i64)], ctypes.c_int),
        "qsv_dist_info": ([vp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                           ctypes.POINTER(i64), ctypes.POINTER(i64), i32p], ctypes.c_int),
        "qsv_create": ([ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "qsv_destroy": ([vp], ctypes.c_int),
        "qsv_n_qubits": ([vp, ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
        "qsv_set_stream": ([vp, vp], ctypes.c_int),
        "qsv_get_stream": ([vp, ctypes.POINTER(vp)], ctypes.c_int),
        "qsv_device_ptr": ([vp, ctypes.POINTER(vp)], ctypes.c_int),
        "qsv_synchronize": ([vp], ctypes.c_int),
        "qsv_copy": ([vp, vp], ctypes.c_int),
        "qsv_set_basis": ([vp, u64], ctypes.c_int),
        "qsv_upload": ([vp, vp], ctypes.c_int),
        "qsv_download": ([vp, vp], ctypes.c_int),
        "qsv_download_async": ([vp, vp], ctypes.c_int),
        "qsv_download_wait": ([vp], ctypes.c_int),
        "qsv_apply_1q": ([vp, dp, ctypes.c_int], ctypes.c_int),
        "qsv_apply_2q": ([vp, dp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "qsv_apply_matrix": ([vp, ctypes.c_int, i32p, dp], ctypes.c_int),
        "qsv_apply_pauli": ([vp, vp, u64, u64, u64], ctypes.c_int),
        "qsv_apply_gates": ([vp, i64, i32p, i32p, dp, sp], ctypes.c_int),
        "qsv_apply_pauli_rotations": ([vp, i64, u64p, u64p, u64p, dp, sp], ctypes.c_int),
        "qsv_expectation": ([vp, i64, u64p, u64p, u64p, dp, dp, dp, dp, dp, sp], ctypes.c_int),
        "qsv_apply_operator": ([vp, vp, i64, u64p, u64p, u64p, dp, dp], ctypes.c_int),
        "qsv_vdot": ([vp, vp, dp], ctypes.c_int),
        "qsv_norm": ([vp, dp], ctypes.c_int),
        "qsv_axpby": ([vp, vp, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                       ctypes.c_double], ctypes.c_int),
        "qsv_plan_gates": ([ctypes.c_int, i64, i32p, i32p, sp], ctypes.c_int),
        "qsv_plan_expectation": ([ctypes.c_int, i64, u64p, u64p, u64p, sp], ctypes.c_int),
        "qsv_debug_plan_json": ([ctypes.c_int, i64, i32p, i32p, dp, ctypes.c_char_p, i64,
                                 ctypes.POINTER(i64)], ctypes.c_int),
        "qsv_debug_pass_source": ([ctypes.c_int, i64, i32p, i32p, i64, ctypes.c_char_p, i64,
                                   ctypes.POINTER(i64), ctypes.POINTER(i64)], ctypes.c_int),
        "qsv_debug_sweep_source": ([ctypes.c_int, i64, u64p, u64p, u64p, i64, ctypes.c_char_p, i64,
                                    ctypes.POINTER(i64), ctypes.POINTER(i64)], ctypes.c_int),
        "qsv_sample_parity": ([vp, u64, i64, u64p, dp, ctypes.POINTER(i64)], ctypes.c_int),
        "qsv_match_rotations": ([ctypes.c_int, i64, i32p, i32p, i64, ctypes.POINTER(i64), u64p,
                                 ctypes.POINTER(i64)], ctypes.c_int),
        "qsv_jit_info": ([ctypes.POINTER(ctypes.c_int), ctypes.POINTER(i64)], ctypes.c_int),
        "qsv_small_info": ([ctypes.POINTER(i64)], ctypes.c_int),
        "qsv_embed_parity": ([vp, vp, u64, ctypes.c_int], ctypes.c_int),
        "qsv_rotation_adjoint": ([vp, vp, i64, u64p, u64p, u64p, dp, dp], ctypes.c_int),
        "qsv_prepare_gates": ([ctypes.c_int, i64, i32p, i32p, ctypes.POINTER(i64)], ctypes.c_int),
        "qsv_apply_prepared": ([vp, i64, dp, sp], ctypes.c_int),
        "qsv_release_program": ([i64], ctypes.c_int),
        "qsv_evolve_basis": ([vp, u64, i64, i32p, i32p, dp, sp], ctypes.c_int),
        "qsv_evolve_basis_prepared": ([vp, u64, i64, dp, sp], ctypes.c_int),
        "qsv_last_plan_stats": ([sp], ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def lib():
    """Load libqsv.so; raises ImportError if the extension was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback"
            )
        L = ctypes.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == QSV_OK:
        return
    msg = lib().qsv_last_error().decode("utf-8", "replace")
    if rc == QSV_ERR_INVALID:
        raise ValueError(msg)
    if rc in (QSV_ERR_RESOURCE, QSV_ERR_NOMEM):
        raise ResourceLimitError(msg)
    raise QsvCudaError(msg)


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = lib().qsv_device_count(ctypes.byref(n))
    return n.value if rc == QSV_OK else 0


def debug_plan(n_qubits: int, kinds, qubits, values) -> dict:
    """Compiled tile program of a flattened gate list (planner debug export)."""
    import json

    need = ctypes.c_int64(0)
    check(lib().qsv_debug_plan_json(n_qubits, len(kinds), i32ptr(kinds), i32ptr(qubits),
                                    dptr(values), None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    check(lib().qsv_debug_plan_json(n_qubits, len(kinds), i32ptr(kinds), i32ptr(qubits),
                                    dptr(values), buf, need.value, ctypes.byref(need)))
    return json.loads(buf.value.decode())


def debug_sweep_source(n_qubits: int, x, y, z, k: int) -> tuple[str, int]:
    """(specialised source of sweep k of the expectation plan, number of sweeps)."""
    need, ns = ctypes.c_int64(0), ctypes.c_int64(0)
    check(lib().qsv_debug_sweep_source(n_qubits, len(x), u64ptr(x), u64ptr(y), u64ptr(z), k, None, 0,
                                       ctypes.byref(need), ctypes.byref(ns)))
    buf = ctypes.create_string_buffer(need.value)
    check(lib().qsv_debug_sweep_source(n_qubits, len(x), u64ptr(x), u64ptr(y), u64ptr(z), k, buf,
                                       need.value, ctypes.byref(need), ctypes.byref(ns)))
    return buf.value.decode(), ns.value


def debug_pass_source(n_qubits: int, kinds, qubits, k: int) -> tuple[str, int]:
    """(specialised source of tile pass k of the plan, number of passes)."""
    need, npass = ctypes.c_int64(0), ctypes.c_int64(0)
    check(lib().qsv_debug_pass_source(n_qubits, len(kinds), i32ptr(kinds), i32ptr(qubits), k, None, 0,
                                      ctypes.byref(need), ctypes.byref(npass)))
    buf = ctypes.create_string_buffer(need.value)
    check(lib().qsv_debug_pass_source(n_qubits, len(kinds), i32ptr(kinds), i32ptr(qubits), k, buf,
                                      need.value, ctypes.byref(need), ctypes.byref(npass)))
    return buf.value.decode(), npass.value


def small_launches() -> int:
    """Small-state rotation program launches so far (qsv_small.cu)."""
    n = ctypes.c_int64(0)
    check(lib().qsv_small_info(ctypes.byref(n)))
    return int(n.value)


def jit_info() -> tuple[bool, int]:
    """(specialised passes available, specialised pass launches so far)."""
    av, n = ctypes.c_int(0), ctypes.c_int64(0)
    check(lib().qsv_jit_info(ctypes.byref(av), ctypes.byref(n)))
    return bool(av.value), int(n.value)


def match_rotations(n_qubits: int, kinds, qubits):
    """Recognised pauli_evolution blocks: (spans int64[R, 3] = start, length,
    rz gate; masks uint64[R, 3] = x, y, z)."""
    import numpy as np

    cnt = ctypes.c_int64(0)
    check(lib().qsv_match_rotations(n_qubits, len(kinds), i32ptr(kinds), i32ptr(qubits), 0, None,
                                    None, ctypes.byref(cnt)))
    spans = np.zeros((cnt.value, 3), dtype=np.int64)
    masks = np.zeros((cnt.value, 3), dtype=np.uint64)
    if cnt.value:
        check(lib().qsv_match_rotations(n_qubits, len(kinds), i32ptr(kinds), i32ptr(qubits), cnt.value,
                                        spans.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                        u64ptr(masks), ctypes.byref(cnt)))
    return spans, masks


def dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def u64ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


def i32ptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
