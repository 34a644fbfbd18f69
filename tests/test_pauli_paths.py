"""Noisy trajectories on a compiled plan (qsv_plan_execute_paulis): every
Pauli error is moved to a pass boundary, the gates on its qubit it crosses are
replaced by their Pauli conjugates.  CPU check of the host logic: the gate
stream the execution applies (qsv_plan_pauli_stream), run through the oracle,
must equal the oracle's run of the program with the Paulis inserted."""

import ctypes as C

import numpy as np
import pytest

from oracle import oracle as O
from paper_2008_07140_b200 import _native as N
from paper_2008_07140_b200 import workloads
from paper_2008_07140_b200.program import Instruction, Program, parse_program
from paper_2008_07140_b200.statevector import compile_gates


def _plan(rec, n, **opts):
    h = C.c_void_p()
    o = N.options(**opts)
    N.check(N.lib().qsv_plan_create(rec.ctypes.data, len(rec), n, C.byref(o), C.byref(h)))
    return h


def _stream(h, paulis, cap=20000):
    pa = np.zeros(len(paulis), dtype=N.PAULI_DTYPE)
    for i, (g, q, k) in enumerate(paulis):
        pa[i] = (g, q, k)
    out = np.zeros(cap, dtype=N.GATE_DTYPE)
    n_out, n_mod = C.c_int64(), C.c_int64()
    N.check(N.lib().qsv_plan_pauli_stream(h, pa.ctypes.data, len(pa), out.ctypes.data, cap, C.byref(n_out),
                                          C.byref(n_mod)))
    return out[:n_out.value], n_mod.value


def _run_records(recs, n):
    st = O.OracleState(n, np.zeros(1 << n, complex), 0)
    st.amplitudes[0] = 1
    for r in recs:
        nt = int(r["n_targets"])
        d = 1 << nt
        u = r["u"][: 2 * d * d].view(np.complex128).reshape(d, d)
        t = tuple(int(x) for x in r["targets"][:nt])
        c = tuple(q for q in range(n) if (int(r["control_mask"]) >> q) & 1)
        O.apply_gate(st, u, t, c)
    return st.amplitudes


def _inserted(prog, paulis):
    """Program with Pauli gates inserted before gate-instruction indices."""
    gates = [i for i in prog.instructions if i.is_gate]
    by = {}
    for g, q, k in paulis:
        by.setdefault(g, []).append(Instruction("_XYZ"[k], (q,)))
    insts = []
    for i, inst in enumerate(gates):
        insts += by.get(i, [])
        insts.append(inst)
    insts += by.get(len(gates), [])
    return Program(prog.qubit_count, prog.creg_count, tuple(insts))


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("opts", [dict(tile_qubits=6, reg_qubits=3, low_qubits=2), dict(tile_qubits=8, reg_qubits=4)])
def test_random_paulis_match_inserted_program(seed, opts):
    n = 11
    prog = parse_program(workloads.rqc_for_qubits(n, 14, seed) if seed % 2 == 0 else workloads.qft_text(n))
    gates = [i for i in prog.instructions if i.is_gate]
    rec = compile_gates(gates)
    h = _plan(rec, n, **opts)
    try:
        rng = np.random.default_rng(seed)
        for trial in range(4):
            k = int(rng.integers(1, 6))
            paulis = [(int(rng.integers(0, len(gates) + 1)), int(rng.integers(0, n)), int(rng.integers(1, 4)))
                      for _ in range(k)]
            if trial == 0:  # same qubit, anticommuting, both orders
                g0 = int(rng.integers(0, len(gates)))
                paulis = [(g0, 3, 1), (g0, 3, 3), (len(gates) // 2, 3, 2)]
            try:
                stream, n_mod = _stream(h, paulis)
            except Exception as e:  # crossing a gate controlled by the qubit (QFT CR): not movable
                assert "cannot be moved" in str(e) or "controlled" in str(e)
                continue
            got = _run_records(stream, n)
            ref = O.run_full(_inserted(prog, paulis)).state.amplitudes
            assert np.abs(got - ref).max() <= 1e-12, (seed, trial, paulis)
    finally:
        N.lib().qsv_plan_destroy(h)


def test_c5_trajectories_move_to_boundaries():
    """C5 shape (4x6, 20 cycles): sampled depolarising errors, few interpreted passes."""
    prog = parse_program(workloads.rqc_text(4, 6, 20, seed=0))
    gates = [i for i in prog.instructions if i.is_gate]
    gidx = {i: k for k, i in enumerate(j for j, inst in enumerate(prog.instructions) if inst.is_gate)}
    rec = compile_gates(gates)
    h = _plan(rec, 24)
    try:
        mods = []
        checked = 0
        for t in range(200):
            ins = workloads.sample_pauli_insertions(prog, 1e-3, workloads.trajectory_seed(0, t))
            if not ins:
                continue
            paulis = [(gidx[i], q, "IXYZ".index(p)) for i, lst in ins.items() for q, p in lst]
            stream, n_mod = _stream(h, paulis)
            mods.append(n_mod)
            if checked < 2:  # full 24-qubit check on two trajectories
                got = _run_records(stream, 24)
                ref = O.run_full(workloads.noisy_trajectory_program(prog, 1e-3, workloads.trajectory_seed(0, t)),
                                 workers=O.cpu_threads()).state.amplitudes
                assert np.abs(got - ref).max() <= 1e-12
                checked += 1
        assert np.mean(mods) <= 1.5, mods
    finally:
        N.lib().qsv_plan_destroy(h)
