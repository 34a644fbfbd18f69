"""Test helper: execute an exported libqsv plan on the CPU with numpy.

The scheduler (csrc/qsv_plan.cpp) is pure host code, so its output can be
validated without a GPU: read every pass/op through the C ABI
(qsv_plan_pass / qsv_plan_op), re-apply the ops in plan order as plain
global-qubit gates, and compare with the oracle.  This checks the fusion,
reordering, peephole merging and local/external control bookkeeping; the
GPU tests then check the CUDA kernel that executes the same plan.

It also checks the residency invariants the kernel relies on: every
non-diagonal op acts on qubits that are register-resident in its stage, and
the stage registers are tile qubits.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from paper_2008_07140_b200 import _native as N


def _apply(psi, n, u, qubits, cmask):
    """Dense apply of u (first qubit = MSB) on `qubits` where all cmask bits are 1."""
    k = len(qubits)
    t = psi.reshape((2,) * n)  # axis j <-> qubit n-1-j
    axes = [n - 1 - q for q in qubits]
    moved = np.moveaxis(t, axes, list(range(k)))
    shp = moved.shape
    flat = moved.reshape(1 << k, -1).copy()
    # column index of the remaining axes -> global index bits for controls
    rest = [q for q in range(n - 1, -1, -1) if q not in qubits]
    if cmask:
        cols = np.arange(flat.shape[1])
        ok = np.ones(flat.shape[1], dtype=bool)
        for pos, q in enumerate(rest):
            if (cmask >> q) & 1:
                bit = (cols >> (len(rest) - 1 - pos)) & 1
                ok &= bit == 1
        flat[:, ok] = u @ flat[:, ok]
    else:
        flat = u @ flat
    out = np.moveaxis(flat.reshape(shp), list(range(k)), axes)
    psi[:] = out.reshape(-1)


def plan_ops(plan_handle):
    L = N.lib()
    info = N.qsv_plan_info()
    N.check(L.qsv_plan_summary(plan_handle, C.byref(info)))
    passes = []
    for p in range(info.passes):
        pi = N.qsv_pass_info()
        N.check(L.qsv_plan_pass(plan_handle, p, C.byref(pi)))
        ops = []
        for o in range(pi.n_ops):
            oi = N.qsv_op_info()
            N.check(L.qsv_plan_op(plan_handle, p, o, C.byref(oi)))
            m = np.frombuffer(bytes(oi.m), dtype=np.complex128).copy()
            ops.append(dict(stage=oi.stage, kind=oi.kind, qa=oi.qa, qb=oi.qb,
                            cmask=oi.control_mask, regs=oi.stage_regs, m=m))
        passes.append(dict(tile_mask=pi.tile_mask, m=pi.m, n_stages=pi.n_stages, ops=ops))
    return info, passes


def build_plan(records: np.ndarray, n: int, **opts):
    L = N.lib()
    h = C.c_void_p()
    o = N.options(**opts)
    N.check(L.qsv_plan_create(records.ctypes.data, len(records), n, C.byref(o), C.byref(h)))
    try:
        return plan_ops(h)
    finally:
        L.qsv_plan_destroy(h)


def execute(passes, n, psi):
    """Apply the exported plan to host amplitudes `psi` (in place) and check invariants."""
    for p in passes:
        tile = p["tile_mask"]
        assert bin(tile).count("1") == p["m"]
        for op in p["ops"]:
            regs = op["regs"]
            assert regs & ~tile == 0, "stage registers must be tile qubits"
            kind, qa, qb, m, cm = op["kind"], op["qa"], op["qb"], op["m"], op["cmask"]
            if kind == N.QSV_OP_MAT1:
                assert (regs >> qa) & 1, "non-diagonal target must be register-resident"
                _apply(psi, n, m[:4].reshape(2, 2), (qa,), cm)
            elif kind == N.QSV_OP_MAT2:
                assert (regs >> qa) & 1 and (regs >> qb) & 1
                _apply(psi, n, m[:16].reshape(4, 4), (qa, qb), cm)
            elif kind == N.QSV_OP_DIAG1:
                _apply(psi, n, np.diag(m[:2]), (qa,), cm)
            elif kind == N.QSV_OP_DIAG2:
                _apply(psi, n, np.diag(m[:4]), (qa, qb), cm)
            else:
                raise AssertionError(f"unknown op kind {kind}")
    return psi
