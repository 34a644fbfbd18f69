"""Test helper: a numpy stand-in for the few libqsv entry points the batched
noisy-trajectory host logic calls (noisy_batch.py), so the CPU suite can check
that logic — draw order, branch choice, renormalisation, MEASURE/PMEASURE
bookkeeping, grouping — against the oracle without a GPU.  Each fake computes
what include/qsv.h specifies, densely on host arrays.  Test infrastructure only:
the product path always binds the real library (and fails loudly without it).
"""

from __future__ import annotations

import ctypes as C
import itertools

import numpy as np

from paper_2008_07140_b200 import _native as N
from plan_emulator import _apply


def _arr(ptr, dtype, count):
    dtype = np.dtype(dtype)
    return np.frombuffer((C.c_char * (dtype.itemsize * count)).from_address(ptr), dtype=dtype)


class FakeLib:
    def __init__(self):
        self.states = {}
        self._ids = itertools.count(1)
        self.staged = {}
        self.run_calls = 0

    def qsv_create(self, n, device, stream, out):
        h = next(self._ids)
        self.states[h] = np.zeros(1 << n, dtype=np.complex128)
        out._obj.value = h
        return 0

    def _psi(self, h):
        return self.states[h.value if hasattr(h, "value") else h]

    def qsv_destroy(self, h):
        self.states.pop(h.value if hasattr(h, "value") else h, None)
        return 0

    def qsv_set_basis(self, h, index):
        psi = self._psi(h)
        psi[:] = 0
        psi[index] = 1
        return 0

    def qsv_upload_strided(self, h, host, offset, count, stride):
        self._psi(h)[offset:offset + count * stride:stride] = _arr(host, np.complex128, count)
        return 0

    def qsv_upload(self, h, host, offset, count):
        self._psi(h)[offset:offset + count] = _arr(host, np.complex128, count)
        return 0

    def qsv_gather_rows(self, h, offs_ptr, n_rows, row_len, host_out):
        psi = self._psi(h)
        offs = _arr(offs_ptr, np.uint64, n_rows)
        out = _arr(host_out, np.complex128, n_rows * row_len).reshape(n_rows, row_len)
        for r, o in enumerate(offs):
            out[r] = psi[int(o):int(o) + row_len]
        return 0

    def qsv_download(self, h, host, offset, count):
        _arr(host, np.complex128, count)[:] = self._psi(h)[offset:offset + count]
        return 0

    def qsv_synchronize(self, h):
        return 0

    def qsv_run(self, h, rec_ptr, n_rec, opts, stats):
        self.run_calls += 1
        psi = self._psi(h)
        n = psi.size.bit_length() - 1
        for r in _arr(rec_ptr, N.GATE_DTYPE, n_rec):
            k = int(r["n_targets"])
            u = r["u"][: 2 * 4 ** k].view(np.complex128).reshape(1 << k, 1 << k)
            _apply(psi, n, u, tuple(int(t) for t in r["targets"][:k]), int(r["control_mask"]))
        return 0

    def qsv_pmeasure(self, h, qubits, m, table_ptr):
        psi = self._psi(h)
        if isinstance(qubits, int):  # a raw pointer (statevector.pmeasure) or a ctypes array
            qubits = _arr(qubits, np.int32, m)
        idx = np.arange(psi.size)
        key = np.zeros(psi.size, dtype=np.int64)
        for pos in range(m):
            key |= ((idx >> qubits[pos]) & 1) << (m - 1 - pos)
        _arr(table_ptr, np.float64, 1 << m)[:] = np.bincount(key, weights=np.abs(psi) ** 2, minlength=1 << m)
        return 0

    def qsv_noisy_batch_step_async(self, h, bl, gk, gq, mats_ptr, nk, nq):
        psi = self._psi(h)
        n = psi.size.bit_length() - 1
        nsub, B = n - bl, 1 << bl
        blocks = psi.reshape(B, 1 << nsub)
        if gk:
            mats = _arr(mats_ptr, np.complex128, 16 * B).reshape(B, 16)
            for t in range(B):
                D = 1 << gk
                _apply(blocks[t], nsub, mats[t, : D * D].reshape(D, D), tuple(gq[i] for i in range(gk)), 0)
        out = np.zeros((B, 4, 4), dtype=np.complex128)
        if nk:
            qs = [nq[i] for i in range(nk)]
            for t in range(B):
                tens = np.moveaxis(blocks[t].reshape((2,) * nsub), [nsub - 1 - q for q in qs], list(range(nk)))
                v = tens.reshape(1 << nk, -1)
                rho = v @ v.conj().T
                out[t, : 1 << nk, : 1 << nk] = np.triu(rho)  # the kernel returns the upper triangle
        self.staged[h.value if hasattr(h, "value") else h] = out.reshape(B, 16)
        return 0

    def qsv_noisy_batch_wait(self, h, bl, rdm_ptr):
        out = self.staged.get(h.value if hasattr(h, "value") else h)
        if rdm_ptr and out is not None:
            _arr(rdm_ptr, np.complex128, out.size)[:] = out.reshape(-1)
        return 0

    def qsv_prob_bit0(self, h, k, out):
        psi = self._psi(h)
        idx = np.arange(psi.size)
        out._obj.value = float(np.sum(np.abs(psi[((idx >> k) & 1) == 0]) ** 2))
        return 0

    def qsv_norm_sq(self, h, out):
        out._obj.value = float(np.sum(np.abs(self._psi(h)) ** 2))
        return 0

    def qsv_collapse(self, h, k, outcome, scale):
        psi = self._psi(h)
        idx = np.arange(psi.size)
        psi[((idx >> k) & 1) != outcome] = 0
        psi *= scale
        return 0

    def qsv_plan_create(self, rec_ptr, n_rec, n, opts, out):
        out._obj.value = next(self._ids)
        return 0

    def qsv_plan_destroy(self, plan):
        return 0

    def qsv_plan_execute_paulis(self, h, plan, paulis, n_paulis, opts, stats):
        return N.QSV_E_UNSUPPORTED  # the host then inserts the Paulis as explicit gates

    def qsv_plan_execute_probe(self, h, plan, paulis, n_paulis, probe, m, table, opts, stats):
        return N.QSV_E_UNSUPPORTED

    def qsv_last_error(self):
        return b""

    def qsv_state_last_error(self, h):
        return b""
