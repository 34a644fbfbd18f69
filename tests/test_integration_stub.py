"""the ctypes stub a qcsim maintainer would add - executed on
the CPU.  The stub's text is taken from INTEGRATION.md itself and run with the
REFERENCE's `gates` module (qcsim.gates, imported from /root/reference in this
container) packing the records; the five libqsv entry points it binds are served
by the real planner (`qsv_plan_create`, host code in libqsv.so) and the host
rendering of the generated pass kernels (tests/jit_host.py), so the record layout
(`struct qsv_gate`), the controlled-form packing and the fused schedule are all
checked against the reference's own `run_full` (statevector.py:397-430)."""

import ctypes as C
import re
import sys
from pathlib import Path

import numpy as np
import pytest

from jit_host import run_plan_host
from paper_2008_07140_b200 import _native as N

ROOT = Path(__file__).resolve().parent.parent
REF_SRC = Path("/root/reference/pkg/src")


def _stub_source() -> str:
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index("## 3."):text.index("## 4.")]
    return re.search(r"```python\n(.*?)```", sec, re.S).group(1)


class _HostLib:
    """qsv_create / qsv_run / qsv_download / qsv_destroy / qsv_last_error on the CPU."""

    def __init__(self):
        self.states = {}
        self.next = 1
        for name in ("qsv_create", "qsv_run", "qsv_download", "qsv_destroy", "qsv_last_error",
                     "qsv_state_last_error"):
            # plain functions (the stub sets .argtypes / .restype on them, as on ctypes symbols)
            bound = getattr(self, "_" + name)
            setattr(self, name, (lambda f: lambda *a: f(*a))(bound))

    def _qsv_create(self, n, device, stream, out):
        psi = np.zeros(1 << n, np.complex128)
        psi[0] = 1
        self.states[self.next] = psi
        out._obj.value = self.next
        self.next += 1
        return 0

    def _qsv_run(self, h, rec_ptr, n_rec, opts, stats):
        psi = self.states[h.value]
        n = psi.size.bit_length() - 1
        rec = np.frombuffer((C.c_char * (N.GATE_DTYPE.itemsize * n_rec)).from_address(rec_ptr),
                            dtype=N.GATE_DTYPE).copy()
        psi[:] = run_plan_host(rec, n, psi)
        return 0

    def _qsv_download(self, h, out_ptr, offset, count):
        psi = self.states[h.value]
        np.frombuffer((C.c_char * (16 * count)).from_address(out_ptr), np.complex128)[:] = psi[offset:offset + count]
        return 0

    def _qsv_destroy(self, h):
        self.states.pop(h.value, None)
        return 0

    def _qsv_last_error(self):
        return b""

    def _qsv_state_last_error(self, h):
        return b""


@pytest.mark.skipif(not REF_SRC.exists(), reason="the reference package is only in the build container")
def test_integration_stub_runs_golden_programs(golden):
    sys.path.insert(0, str(REF_SRC))
    try:
        from qcsim import gates as ref_gates
        from qcsim.program import parse_program as ref_parse
        from qcsim.statevector import run_full as ref_run_full
    finally:
        sys.path.remove(str(REF_SRC))
    src = _stub_source().replace("from . import gates\n", "").replace('C.CDLL("libqsv.so")', "_HOSTLIB")
    ns = {"_HOSTLIB": _HostLib(), "gates": ref_gates}
    exec(compile(src, "INTEGRATION.md#3", "exec"), ns)
    # the stub's record dtype is the C struct the library reads
    assert ns["GATE"].itemsize == N.GATE_DTYPE.itemsize
    assert ns["GATE"].fields["u"][1] == N.GATE_DTYPE.fields["u"][1]
    done = 0
    for name, rec in golden["programs"].items():
        prog = ref_parse(rec["text"])
        if any(i.name in ("MEASURE", "PMEASURE") for i in prog.instructions) or prog.qubit_count > 12:
            continue
        got = ns["run_full_gpu"](prog)
        want = ref_run_full(prog).state.amplitudes
        assert np.abs(got - want).max() <= 1e-12, name
        done += 1
    assert done >= 5
