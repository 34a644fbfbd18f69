"""ctypes binding of libqsv.so (include/qsv.h).

Loading is strict: if the library is missing or a CUDA call fails, the
caller gets an exception - there is no eager/CPU substitute anywhere in the
package.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from .errors import NativeLibraryMissing, raise_for_status

LIB_PATH = Path(__file__).resolve().parent / "libqsv.so"

QSV_OP_MAT1, QSV_OP_MAT2, QSV_OP_DIAG1, QSV_OP_DIAG2 = 1, 2, 3, 4
QSV_E_UNSUPPORTED = -6  # qsv.h

# numpy mirror of `qsv_gate` (C layout: int32 n_targets, int32 targets[2],
# uint64 control_mask, double u[32]) - built in bulk from a Program
GATE_DTYPE = np.dtype([("n_targets", "<i4"), ("targets", "<i4", (2,)),
                       ("control_mask", "<u8"), ("u", "<f8", (32,))], align=True)


# one Pauli error before gate record `gate` (qsv.h qsv_pauli): kind 1 X, 2 Y, 3 Z
PAULI_DTYPE = np.dtype([("gate", "<i8"), ("qubit", "<i4"), ("kind", "<i4")], align=True)


class qsv_exchange(C.Structure):
    _fields_ = [("positions", C.c_uint64), ("self_bits", C.c_uint64), ("dst", C.c_uint64 * 8)]


class qsv_options(C.Structure):
    _fields_ = [("fuse", C.c_int32), ("tile_qubits", C.c_int32), ("reg_qubits", C.c_int32),
                ("low_qubits", C.c_int32), ("profile", C.c_int32), ("n_global", C.c_int32),
                ("jit", C.c_int32), ("super_qubits", C.c_int32), ("product_start", C.c_int32),
                ("plan_objective", C.c_int32)]


class qsv_run_stats(C.Structure):
    _fields_ = [("gates", C.c_int64), ("passes", C.c_int64), ("stages", C.c_int64),
                ("inner_passes", C.c_int64), ("launches", C.c_int64), ("kernel_ms", C.c_double), ("max_launch_ms", C.c_double),
                ("algorithmic_bytes", C.c_double), ("plan_ms", C.c_double), ("jit_ms", C.c_double),
                ("compiled_passes", C.c_int64)]

    def as_dict(self) -> dict:
        return {f: getattr(self, f) for f, _ in self._fields_}


class qsv_plan_info(C.Structure):
    _fields_ = [("n_qubits", C.c_int32), ("tile_qubits", C.c_int32), ("reg_qubits", C.c_int32),
                ("low_qubits", C.c_int32), ("gates", C.c_int64), ("passes", C.c_int64),
                ("stages", C.c_int64), ("ops", C.c_int64), ("super_qubits", C.c_int32),
                ("product_start", C.c_int32), ("super_passes", C.c_int64)]


class qsv_pass_info(C.Structure):
    _fields_ = [("tile_mask", C.c_uint64), ("m", C.c_int32), ("n_stages", C.c_int32),
                ("n_ops", C.c_int64), ("super_mask", C.c_uint64), ("super_index", C.c_int64)]


class qsv_op_info(C.Structure):
    _fields_ = [("stage", C.c_int32), ("kind", C.c_int32), ("qa", C.c_int32), ("qb", C.c_int32),
                ("control_mask", C.c_uint64), ("stage_regs", C.c_uint64), ("m", C.c_double * 32)]


_P = C.c_void_p
_SIGNATURES = {
    "qsv_version": ([], C.c_char_p),
    "qsv_last_error": ([], C.c_char_p),
    "qsv_state_last_error": ([C.c_void_p], C.c_char_p),
    "qsv_last_launches": ([_P, _P, _P, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
    "qsv_jit_wait": ([], C.c_int),
    "qsv_plan_product_tables": ([_P, C.c_uint64, _P, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
    "qsv_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "qsv_create": ([C.c_int, C.c_int, _P, C.POINTER(_P)], C.c_int),
    "qsv_create_on": ([C.c_int, C.c_int, _P, _P, C.POINTER(_P)], C.c_int),
    "qsv_destroy": ([_P], C.c_int),
    "qsv_device_ptr": ([_P, C.POINTER(_P)], C.c_int),
    "qsv_set_basis": ([_P, C.c_uint64], C.c_int),
    "qsv_upload": ([_P, _P, C.c_uint64, C.c_uint64], C.c_int),
    "qsv_download": ([_P, _P, C.c_uint64, C.c_uint64], C.c_int),
    "qsv_download_async": ([_P, _P, C.c_uint64, C.c_uint64], C.c_int),
    "qsv_synchronize": ([_P], C.c_int),
    "qsv_apply_gate": ([_P, _P], C.c_int),
    "qsv_run": ([_P, _P, C.c_int64, C.POINTER(qsv_options), C.POINTER(qsv_run_stats)], C.c_int),
    "qsv_plan_create": ([_P, C.c_int64, C.c_int, C.POINTER(qsv_options), C.POINTER(_P)], C.c_int),
    "qsv_plan_destroy": ([_P], C.c_int),
    "qsv_plan_summary": ([_P, C.POINTER(qsv_plan_info)], C.c_int),
    "qsv_plan_pass": ([_P, C.c_int64, C.POINTER(qsv_pass_info)], C.c_int),
    "qsv_plan_op": ([_P, C.c_int64, C.c_int64, C.POINTER(qsv_op_info)], C.c_int),
    "qsv_plan_execute": ([_P, _P, C.POINTER(qsv_options), C.POINTER(qsv_run_stats)], C.c_int),
    "qsv_norm_sq": ([_P, C.POINTER(C.c_double)], C.c_int),
    "qsv_prob_bit0": ([_P, C.c_int, C.POINTER(C.c_double)], C.c_int),
    "qsv_collapse": ([_P, C.c_int, C.c_int, C.c_double], C.c_int),
    "qsv_scale": ([_P, C.c_double], C.c_int),
    "qsv_pmeasure": ([_P, _P, C.c_int, _P], C.c_int),
    "qsv_pmeasure_async": ([_P, _P, C.c_int, _P], C.c_int),
    "qsv_inner": ([_P, _P, C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
    "qsv_max_abs_diff": ([_P, _P, C.POINTER(C.c_double)], C.c_int),
    "qsv_reduced_density": ([_P, C.c_int, _P, _P], C.c_int),
    "qsv_upload_strided": ([_P, _P, C.c_uint64, C.c_uint64, C.c_uint64], C.c_int),
    "qsv_gather_rows": ([_P, _P, C.c_int, C.c_uint64, _P], C.c_int),
    "qsv_noisy_batch_step_async": ([_P, C.c_int, C.c_int, _P, _P, C.c_int, _P], C.c_int),
    "qsv_noisy_batch_wait": ([_P, C.c_int, _P], C.c_int),
    "qsv_noisy_batch_step": ([_P, C.c_int, C.c_int, _P, _P, C.c_int, _P, _P], C.c_int),
    "qsv_plan_kernel_source": ([_P, C.c_int64, C.c_int, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
    "qsv_plan_exchange_source": ([_P, C.c_int64, C.c_int, C.c_uint64, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)],
                                 C.c_int),
    "qsv_plan_super_source": ([_P, C.c_int64, C.c_int, C.c_char_p, C.c_int64, C.POINTER(C.c_int64)], C.c_int),
    "qsv_plan_pass_cost": ([_P, C.c_int64, C.POINTER(C.c_double)], C.c_int),
    "qsv_jit_compile": ([C.c_char_p, C.POINTER(C.c_int64)], C.c_int),
    "qsv_plan_segments": ([_P, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_int, _P, _P, C.POINTER(C.c_int64)],
                          C.c_int),
    "qsv_ipc_mem_handle": ([_P, _P, C.POINTER(C.c_uint64)], C.c_int),
    "qsv_ipc_mem_open": ([_P, C.c_uint64, C.c_int, C.POINTER(_P)], C.c_int),
    "qsv_ipc_mem_close": ([_P], C.c_int),
    "qsv_copy_async": ([_P, _P, C.c_uint64, _P], C.c_int),
    "qsv_exchange_fusable": ([_P, _P, C.c_int64, C.POINTER(qsv_options), C.c_uint64, C.POINTER(C.c_int)], C.c_int),
    "qsv_run_exchange": ([_P, _P, C.c_int64, C.POINTER(qsv_options), _P, C.POINTER(qsv_run_stats)], C.c_int),
    "qsv_plan_execute_paulis": ([_P, _P, _P, C.c_int64, C.POINTER(qsv_options), C.POINTER(qsv_run_stats)], C.c_int),
    "qsv_plan_execute_probe": ([_P, _P, _P, C.c_int64, _P, C.c_int, _P, C.POINTER(qsv_options),
                                C.POINTER(qsv_run_stats)], C.c_int),
    "qsv_plan_pauli_stream": ([_P, _P, C.c_int64, _P, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64)],
                              C.c_int),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def lib():
    """The loaded library (raises NativeLibraryMissing when it is not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run `python -m paper_2008_07140_b200.build_native` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def check(rc: int, handle=None) -> None:
    """Raise the errors.py class of a failed status; the message comes from the
    handle the call acted on when given (qsv_state_last_error), else from the
    calling thread's last failure."""
    if rc != 0:
        L = lib()
        msg = L.qsv_state_last_error(handle) if handle is not None else L.qsv_last_error()
        raise_for_status(rc, (msg or b"").decode(errors="replace"))


def last_launches(handle):
    """(ms, algorithmic bytes) per launch of the last profiled call on `handle`."""
    L = lib()
    n = C.c_int64()
    check(L.qsv_last_launches(handle, None, None, 0, C.byref(n)), handle)
    ms = np.zeros(n.value)
    by = np.zeros(n.value)
    check(L.qsv_last_launches(handle, ms.ctypes.data, by.ctypes.data, n.value, C.byref(n)), handle)
    return ms, by


def options(fuse=True, tile_qubits=0, reg_qubits=0, low_qubits=0, profile=False, n_global=0,
            jit=0, super_qubits=0, product_start=0, plan_objective=0) -> qsv_options:
    """jit: 0 auto (specialised kernels for n >= 16), 1 always, -1 never;
    super_qubits: L2 super-tile size s (0 = default 21; s <= tile_qubits disables);
    product_start: 1 plan with a product-state start (runs only from set_basis), -1 never,
    0 auto (qsv_run: on for basis starts with specialised kernels);
    plan_objective: what the scheduler's look-ahead minimises - 0/2 modeled time (default),
    1 the number of passes."""
    o = qsv_options()
    o.fuse, o.tile_qubits, o.reg_qubits = int(bool(fuse)), int(tile_qubits), int(reg_qubits)
    o.low_qubits, o.profile, o.n_global = int(low_qubits), int(bool(profile)), int(n_global)
    o.jit = int(jit)
    o.super_qubits = int(super_qubits)
    o.product_start = int(product_start)
    o.plan_objective = int(plan_objective)
    return o


def gate_records(items) -> np.ndarray:
    """Pack (base matrix, targets, controls) triples into a qsv_gate array."""
    items = list(items)
    rec = np.zeros(len(items), dtype=GATE_DTYPE)
    for i, (u, targets, controls) in enumerate(items):
        u = np.asarray(u, dtype=np.complex128)
        nt = len(targets)
        rec["n_targets"][i] = nt
        rec["targets"][i, :nt] = targets
        mask = 0
        for c in controls:
            mask |= 1 << int(c)
        rec["control_mask"][i] = mask
        flat = u.reshape(-1)
        rec["u"][i, : 2 * flat.size] = flat.view(np.float64)
    return rec
