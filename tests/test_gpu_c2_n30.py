"""BASELINE config 2 at its full size: the 30-qubit 5x6, 24-cycle RQC (603 gates,
16 GiB complex128 state) on the GPU vs the oracle port of the reference
`run_full` (qcsim/statevector.py:397-430) at the reference's own ceiling
(DEFAULT_MAX_QUBITS = 30, statevector.py:27).

The oracle runs once per module (all host threads, ~2 min); its end state is
uploaded to the device and every GPU configuration is compared there:
the default fused plan, `fuse=False` (one kernel per gate, the reference's
sweep per gate), and the fused plan with k = 2, 3, 4, 5 register qubits per
stage (BASELINE C2 "with and without host gate fusion, k = 2..5"), plus the
interpreted pass kernel (no NVRTC)."""

import numpy as np
import pytest

from bigsize import assert_device_parity, need_device_gib, need_host_gib, threads
from paper_2008_07140_b200 import statevector as SV
from paper_2008_07140_b200 import workloads
from paper_2008_07140_b200.program import parse_program

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N = 30


@pytest.fixture(scope="module")
def c2():
    from oracle import oracle as O

    need_host_gib(20)
    need_device_gib(34)
    prog = parse_program(workloads.rqc_text(*workloads.C2_SHAPE, seed=0))
    assert prog.qubit_count == N and len(prog.gate_instructions()) == 603
    ref = O.run_full(prog, workers=threads())
    dev_ref = SV.StateVector(N, ref.state.amplitudes)
    del ref
    yield prog, dev_ref
    dev_ref.close()


# jit=1: the specialised kernels, compiled before the run (jit=0, the default, would run a
# circuit's first call on the interpreted kernel while they compile in the background -
# covered by "cold-mixed"); product_start follows run_full's default (on for |0..0>)
# (cold-mixed first: no C2 kernel is compiled yet, so most of its passes run interpreted)
@pytest.mark.parametrize("cfg", [dict(), dict(jit=1), dict(fuse=False), dict(reg_qubits=2, jit=1),
                                 dict(reg_qubits=3, jit=1), dict(reg_qubits=4, jit=1), dict(reg_qubits=5, jit=1),
                                 dict(jit=-1)],
                         ids=["cold-mixed", "fused-default", "unfused", "k2", "k3", "k4", "k5", "interpreted"])
def test_c2_n30_vs_oracle(c2, cfg):
    prog, ref = c2
    res = SV.run_full(prog, **cfg)
    try:
        assert_device_parity(res.state, ref, f"C2 n=30 {cfg} (compiled passes {res.stats.get('compiled_passes')}"
                                             f" of {res.stats.get('passes')})")
        # the reference's readout on the same state (statevector.py:311-328)
        assert abs(res.state.norm_sq() - 1.0) <= 1e-12
    finally:
        res.state.close()


def test_c2_n30_pmeasure_vs_oracle_state(c2):
    """PMEASURE over four qubits of the GPU end state equals the table of the
    uploaded oracle state (both tabulated by the device reduction)."""
    prog, ref = c2
    res = SV.run_full(prog, jit=1)
    try:
        qs = (0, 11, 22, 29)
        assert np.abs(SV.pmeasure(res.state, qs) - SV.pmeasure(ref, qs)).max() <= 1e-12
    finally:
        res.state.close()
