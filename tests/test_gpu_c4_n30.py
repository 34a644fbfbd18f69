"""BASELINE config 4 at its full size: the 30-qubit QFT (480 gates) on an i.i.d.
complex Gaussian state, and the DAGGER round trip (program.py:328-333).

* forward QFT(psi0) on the GPU vs the oracle port of the reference driving
  `apply_instruction` from the same psi0 (`run_full` cannot start
  from an arbitrary state, so the oracle is seeded with psi0);
* QFT then DAGGER-QFT on the GPU must return psi0.
Both compared on the device (tests/bigsize.py)."""

import pytest

from bigsize import assert_device_parity, need_device_gib, need_host_gib, threads
from paper_2008_07140_b200 import statevector as SV
from paper_2008_07140_b200 import workloads
from paper_2008_07140_b200.program import parse_program

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N = 30


def test_c4_n30_forward_and_round_trip():
    from oracle import oracle as O

    need_host_gib(36)
    need_device_gib(50)
    psi0 = workloads.gaussian_state(N, 0)
    fwd_prog = parse_program(workloads.qft_text(N))
    rt_prog = parse_program(workloads.qft_text(N, round_trip=True))
    assert len(fwd_prog.gate_instructions()) == 480 and len(rt_prog.gate_instructions()) == 960
    fwd = SV.run_full(fwd_prog, initial_state=psi0, jit=1).state
    rt = SV.run_full(rt_prog, initial_state=psi0, jit=1).state
    check = SV.StateVector(N, psi0)
    try:
        assert_device_parity(rt, check, "C4 n=30 QFT + DAGGER-QFT round trip vs psi0")
        rt.close()
        ref = O.run_full(fwd_prog, initial=psi0, workers=threads())
        del psi0
        check.amplitudes = ref.state.amplitudes
        del ref
        assert_device_parity(fwd, check, "C4 n=30 forward QFT vs oracle")
    finally:
        for s in (fwd, rt, check):
            s.close()
