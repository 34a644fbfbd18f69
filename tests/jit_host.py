"""Test helper: run the specialised pass kernels' HOST rendering on the CPU.

libqsv generates one CUDA kernel per fused pass (csrc/qsv_jit.cpp) and can
render the very same op emission as plain C++ (`qsv_plan_kernel_source(...,
host=1, ...)`).  Compiling that with gcc and running it against the oracle
checks the generator (register classes, smem swizzle offsets, pending-phase
merging, scalar/thread/external conditions) without a GPU.  Test
infrastructure only.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import subprocess
import tempfile
from pathlib import Path

import numpy as np

from paper_2008_07140_b200 import _native as N

_CACHE = Path(tempfile.gettempdir()) / "qsv_jit_host"


def plan_handle(records: np.ndarray, n: int, **opts):
    h = C.c_void_p()
    o = N.options(**opts)
    N.check(N.lib().qsv_plan_create(records.ctypes.data, len(records), n, C.byref(o), C.byref(h)))
    return h


def kernel_source(h, p: int, host: bool) -> str:
    L = N.lib()
    need = C.c_int64()
    N.check(L.qsv_plan_kernel_source(h, p, int(host), None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    N.check(L.qsv_plan_kernel_source(h, p, int(host), buf, need.value, C.byref(need)))
    return buf.value.decode()


def _compile(src: str):
    _CACHE.mkdir(exist_ok=True)
    key = hashlib.sha1(src.encode()).hexdigest()[:20]
    so = _CACHE / f"p_{key}.so"
    if not so.exists():
        cpp = _CACHE / f"p_{key}.cpp"
        cpp.write_text(src)
        subprocess.run(["/usr/bin/g++", "-O1", "-shared", "-fPIC", "-o", str(so), str(cpp)], check=True)
    lib = C.CDLL(str(so))
    lib.qsv_pass_host.argtypes = [C.c_void_p, C.c_ulonglong]
    lib.qsv_pass_host.restype = None
    return lib


def run_plan_host(records: np.ndarray, n: int, psi: np.ndarray, **opts) -> np.ndarray:
    """Apply every pass of the plan through its generated host rendering."""
    h = plan_handle(records, n, **opts)
    try:
        info = N.qsv_plan_info()
        N.check(N.lib().qsv_plan_summary(h, C.byref(info)))
        out = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        for p in range(info.passes):
            pi = N.qsv_pass_info()
            N.check(N.lib().qsv_plan_pass(h, p, C.byref(pi)))
            lib = _compile(kernel_source(h, p, True))
            lib.qsv_pass_host(out.ctypes.data, 1 << (n - pi.m))
        return out
    finally:
        N.lib().qsv_plan_destroy(h)


def product_tables(h, basis: int) -> np.ndarray:
    L = N.lib()
    cnt = C.c_int64()
    N.check(L.qsv_plan_product_tables(h, basis, None, 0, C.byref(cnt)))
    tab = np.zeros(cnt.value, dtype=np.complex128)
    N.check(L.qsv_plan_product_tables(h, basis, tab.ctypes.data, cnt.value, C.byref(cnt)))
    return tab


def run_product_plan_host(records: np.ndarray, n: int, basis: int, **opts):
    """A product-start plan (qsv_options.product_start = 1) through the host rendering:
    pass 0 synthesises the product state from the plan's factor tables for `basis`
    (the state buffer is not read), the other passes run as usual.  Returns
    (amplitudes, plan passes) or None when the stream has nothing to absorb."""
    h = plan_handle(records, n, product_start=1, **opts)
    try:
        info = N.qsv_plan_info()
        N.check(N.lib().qsv_plan_summary(h, C.byref(info)))
        if not info.product_start:
            return None
        out = np.full(1 << n, np.nan + 0j)  # never read by the synthesising pass
        tab = product_tables(h, basis)
        for p in range(info.passes):
            pi = N.qsv_pass_info()
            N.check(N.lib().qsv_plan_pass(h, p, C.byref(pi)))
            lib = _compile(kernel_source(h, p, True))
            if p == 0:
                lib.qsv_pass_host.argtypes = [C.c_void_p, C.c_ulonglong, C.c_void_p]
                lib.qsv_pass_host(out.ctypes.data, 1 << (n - pi.m), tab.ctypes.data)
            else:
                lib.qsv_pass_host(out.ctypes.data, 1 << (n - pi.m))
        return out, info.passes
    finally:
        N.lib().qsv_plan_destroy(h)


def super_source(h, si: int, host: bool) -> str:
    L = N.lib()
    need = C.c_int64()
    N.check(L.qsv_plan_super_source(h, si, int(host), None, 0, C.byref(need)))
    buf = C.create_string_buffer(need.value)
    N.check(L.qsv_plan_super_source(h, si, int(host), buf, need.value, C.byref(need)))
    return buf.value.decode()


def super_batch_log2(n: int, s: int, budget: int = 64 << 20) -> int:
    b = 0
    while b < n - s and (16 << (s + b + 1)) <= budget:
        b += 1
    return b


def run_plan_host_super(records: np.ndarray, n: int, psi: np.ndarray, budget: int = 64 << 20,
                        **opts) -> np.ndarray:
    """Execute the plan super-pass by super-pass through the generated
    persistent super kernels (host rendering), like the GPU executor does."""
    import os

    os.environ["QSV_L2_BYTES"] = str(budget)
    h = plan_handle(records, n, **opts)
    try:
        info = N.qsv_plan_info()
        N.check(N.lib().qsv_plan_summary(h, C.byref(info)))
        out = np.ascontiguousarray(psi, dtype=np.complex128).copy()
        passes = []
        for p in range(info.passes):
            pi = N.qsv_pass_info()
            N.check(N.lib().qsv_plan_pass(h, p, C.byref(pi)))
            passes.append((pi.super_index, pi.m, bin(pi.super_mask).count("1")))
        for si in range(info.super_passes):
            mine = [p for p, (s_i, _, _) in enumerate(passes) if s_i == si]
            s = passes[mine[0]][2]
            if len(mine) > 1 and info.super_qubits > info.tile_qubits:
                src = super_source(h, si, True)
                lib = _compile(src.replace("qsv_super_host", "qsv_pass_host"))
                lb = super_batch_log2(n, info.super_qubits, budget)
                lib.qsv_pass_host.argtypes = [C.c_void_p, C.c_ulonglong, C.c_void_p]
                lib.qsv_pass_host(out.ctypes.data, 1 << (n - s - lb), None)
            else:
                for p in mine:
                    lib = _compile(kernel_source(h, p, True))
                    lib.qsv_pass_host(out.ctypes.data, 1 << (n - passes[p][1]))
        return out
    finally:
        N.lib().qsv_plan_destroy(h)
