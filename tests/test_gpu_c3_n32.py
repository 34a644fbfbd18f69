"""BASELINE config 3 correctness at its single-GPU size (n = 32, 64 GiB state):
the mirror circuit C followed by `DAGGER C ENDDAGGER` (program.py:328-333) must
return |0..0> - amplitude 1 at index 0 and <= 1e-10 everywhere else (SURVEY
8(c)(iii)).  The CPU oracle cannot hold 2^32 amplitudes in this container,
so this is the size-independent known answer at the C3 size.

The residual is measured without cancellation: amplitude 0 is read back, set
to zero on the device, and the norm of what is left is sum_{i>0} |a_i|^2, so
max_{i>0} |a_i| <= sqrt(that)."""

import math

import numpy as np
import pytest

from bigsize import need_device_gib
from paper_2008_07140_b200 import _native as N
from paper_2008_07140_b200 import statevector as SV
from paper_2008_07140_b200 import workloads
from paper_2008_07140_b200.program import parse_program

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("n", [32])
def test_c3_mirror_returns_basis_state(n):
    need_device_gib(66)
    prog = parse_program(workloads.mirror_text(workloads.rqc_for_qubits(n, 24, 0)))
    res = SV.run_full(prog, max_qubits=n, jit=1)  # specialised kernels (product start)
    st = res.state
    try:
        a0 = np.empty(1, np.complex128)
        st.download(a0, 0)
        assert abs(a0[0] - 1.0) <= 1e-10, a0[0]
        zero = np.zeros(1, np.complex128)
        N.check(N.lib().qsv_upload(st.handle, zero.ctypes.data, 0, 1))
        rest = st.norm_sq()
        assert math.sqrt(rest) <= 1e-10, rest
    finally:
        st.close()
