"""Pin the oracle (oracle/) to the REAL reference: golden vectors produced by
tests/golden/make_golden.py from qcsim itself.  CPU only."""

import math

import numpy as np
import pytest

from conftest import program_text
from oracle import oracle as O
from paper_2008_07140_b200.program import parse_program


def test_run_full_bit_exact_all_programs(golden, golden_arrays):
    """statevector.run_full end states, PMEASURE tables and cregs, bit-exact."""
    for name, rec in golden["runs"].items():
        prog = parse_program(program_text(golden, name))
        for workers in (1, 4):
            res = O.run_full(prog, np.random.default_rng(rec["seed"]), workers=workers)
            assert np.array_equal(res.state.amplitudes, golden_arrays[f"run/{name}"]), (name, workers)
            assert res.cregs == rec["cregs"], name
            for t_i, qubits in enumerate(rec["tables"]):
                assert tuple(res.tables[t_i][0]) == tuple(qubits)
                assert np.array_equal(res.tables[t_i][1], golden_arrays[f"run/{name}/table{t_i}"]), name


def test_kernel_streams_bit_exact(golden, golden_arrays):
    """apply_single_qubit / apply_controlled / apply_two_qubit / apply_projector
    streams on random states and random chunk sizes (test_statevector.py:218-250)."""
    for s_idx, rec in enumerate(golden["kernel_streams"]):
        psi = golden_arrays[f"stream{s_idx}/psi0"].copy()
        st = O.OracleState(rec["n"], psi, rec["chunk_log2"])
        for o_idx, op in enumerate(rec["ops"]):
            u = golden_arrays[f"stream{s_idx}/u{o_idx}"]
            O.apply_gate(st, u, op["targets"], op["controls"])
        assert np.array_equal(st.amplitudes, golden_arrays[f"stream{s_idx}/final"]), s_idx


@pytest.mark.parametrize("n", [3, 6, 9])
def test_qft_on_random_state(golden, golden_arrays, n):
    psi0 = golden_arrays[f"qft{n}/psi0"]
    for tag in ("forward", "round_trip"):
        prog = parse_program(golden["qft"][str(n)][tag])
        res = O.run_full(prog, initial=psi0)
        assert np.array_equal(res.state.amplitudes, golden_arrays[f"qft{n}/{tag}"]), (n, tag)
    # independent KAT: forward QFT = sqrt(N) * ifft
    fwd = golden_arrays[f"qft{n}/forward"]
    assert np.abs(fwd - math.sqrt(1 << n) * np.fft.ifft(psi0)).max() < 1e-12


def test_noisy_trajectories_match_reference(golden, golden_arrays):
    """Depolarising run_full(prog, default_rng(s), make_noise_model(...)) (noise.py:188-222)."""
    for rec in golden["noise"]:
        prog = parse_program(rec["text"])
        res = O.run_full(prog, np.random.default_rng(rec["traj_seed"]), noise=("depolarizing", rec["p"]))
        assert np.abs(res.state.amplitudes - golden_arrays[rec["key"]]).max() <= 1e-15, rec["key"]


def test_c1_sampled_amplitudes(golden, golden_arrays):
    """20-qubit BASELINE config 1 circuit: oracle vs reference at 2k sampled indices."""
    prog = parse_program(golden["c1"]["text"])
    res = O.run_full(prog, workers=O.cpu_threads())
    idx = golden_arrays["c1/idx"]
    assert np.array_equal(res.state.amplitudes[idx], golden_arrays["c1/amps"])
    assert np.array_equal(O.pmeasure(res.state, (0, 7, 13, 19)), golden_arrays["c1/pm_0_7_13_19"])
    assert res.state.norm_sq() == pytest.approx(golden["c1"]["norm_sq"], abs=0)


def test_measure_statistics():
    rng = np.random.default_rng(42)
    ones = 0
    for _ in range(20000):
        st = O.OracleState(1, np.array([1, 1], dtype=complex) / math.sqrt(2), 0)
        ones += O.measure(st, 0, rng)
    assert abs(ones - 10000) < 3 * math.sqrt(20000 * 0.25)


def test_default_chunk_log2_matches_reference_rule():
    for n in range(1, 12):
        for w in (1, 2, 3, 4, 8, 16):
            want = max(0, n - (max(1, max(4, 4 * w) - 1).bit_length()))
            assert O.default_chunk_log2(n, w) == want
