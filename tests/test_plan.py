"""Scheduler/fuser (pure host code in libqsv.so) validated on CPU: the exported
plan, re-executed as plain gates, must reproduce the oracle; residency
invariants must hold.  Also checks the C ABI exports every declared symbol."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, program_text
from oracle import oracle as O
from paper_2008_07140_b200 import _native as N
from paper_2008_07140_b200 import errors, workloads
from paper_2008_07140_b200.program import parse_program
from paper_2008_07140_b200.statevector import compile_gates
from plan_emulator import build_plan, execute


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "qsv.h").read_text()
    declared = set(re.findall(r"^\s*(?:const\s+char\s*\*\s*|int\s+)(qsv_\w+)\s*\(", header, re.M))
    L = N.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(N.EXPORTED)
    assert N.GATE_DTYPE.itemsize == 280  # sizeof(qsv_gate)
    assert C.sizeof(N.qsv_op_info) == 288
    assert L.qsv_version().decode().startswith("qsv")


CONFIGS = [dict(), dict(tile_qubits=3, reg_qubits=2, low_qubits=1), dict(tile_qubits=4, reg_qubits=2),
           dict(tile_qubits=2, reg_qubits=2), dict(tile_qubits=5, reg_qubits=3, low_qubits=2),
           dict(tile_qubits=6, reg_qubits=4, low_qubits=3)]


@pytest.mark.parametrize("cfg", CONFIGS)
def test_plan_reproduces_reference_runs(golden, golden_arrays, cfg):
    for name, rec in golden["runs"].items():
        prog = parse_program(program_text(golden, name))
        if any(not i.is_gate for i in prog.instructions):
            continue
        n = prog.qubit_count
        _, passes = build_plan(compile_gates(prog.gate_instructions()), n, **cfg)
        psi = np.zeros(1 << n, complex)
        psi[0] = 1
        execute(passes, n, psi)
        assert np.abs(psi - golden_arrays[f"run/{name}"]).max() <= 1e-12, (name, cfg)


@pytest.mark.parametrize("seed", range(6))
def test_plan_random_dense_streams(seed):
    """Random 1q/2q/controlled/diagonal streams incl. repeated targets (peephole paths)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 9))
    items = []
    for _ in range(120):
        kind = rng.integers(0, 5)
        qs = [int(q) for q in rng.permutation(n)]
        z = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
        q4, _ = np.linalg.qr(z)
        if kind == 0:
            items.append((q4[:2, :2] / np.linalg.norm(q4[:2, :2], 2), (qs[0],), ()))
        elif kind == 1:
            items.append((np.diag(np.exp(1j * rng.uniform(0, 6, 2))), (qs[0],), tuple(qs[1:1 + int(rng.integers(0, 3))])))
        elif kind == 2:
            items.append((q4, (qs[0], qs[1]), tuple(qs[2:2 + int(rng.integers(0, 2))])))
        elif kind == 3:
            items.append((np.diag(np.exp(1j * rng.uniform(0, 6, 4))), (qs[0], qs[1]), tuple(qs[2:3])))
        else:
            u = q4[:2, :2]
            items.append((u, (qs[0],), tuple(qs[1:1 + int(rng.integers(1, 3))])))
    recs = N.gate_records(items)
    psi0 = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    ref = O.OracleState(n, psi0.copy(), 0)
    for u, t, c in items:
        O.apply_gate(ref, u, t, c)
    for cfg in CONFIGS:
        _, passes = build_plan(recs, n, **cfg)
        psi = psi0.copy()
        execute(passes, n, psi)
        assert np.abs(psi - ref.amplitudes).max() <= 1e-12, cfg


def test_plan_qft_and_rqc_pass_counts():
    prog = parse_program(workloads.qft_text(12, round_trip=True))
    recs = compile_gates(prog.gate_instructions())
    info, passes = build_plan(recs, 12, tile_qubits=8, reg_qubits=4, low_qubits=3)
    g = np.random.default_rng(1)
    psi0 = workloads.gaussian_state(12, 3)
    psi = psi0.copy()
    execute(passes, 12, psi)
    assert np.abs(psi - psi0).max() < 1e-12  # QFT followed by DAGGER QFT = identity
    assert info.passes < len(recs)
    c2 = parse_program(workloads.rqc_text(5, 6, 24, 0))
    info, _ = build_plan(compile_gates(c2.gate_instructions()), 30)
    assert info.passes <= 16  # fused: a handful of HBM passes instead of 603


def test_plan_rejects_bad_gates():
    L = N.lib()
    h = C.c_void_p()
    bad = N.gate_records([(np.eye(2), (5,), ())])
    with pytest.raises(errors.ParseError):
        N.check(L.qsv_plan_create(bad.ctypes.data, 1, 3, None, C.byref(h)))
    bad = N.gate_records([(np.eye(2), (0,), (0,))])
    with pytest.raises(errors.ParseError):
        N.check(L.qsv_plan_create(bad.ctypes.data, 1, 3, None, C.byref(h)))
    bad = N.gate_records([(np.eye(2), (0,), ())])
    bad["n_targets"][0] = 3
    with pytest.raises(errors.UnsupportedGate):
        N.check(L.qsv_plan_create(bad.ctypes.data, 1, 3, None, C.byref(h)))


def test_state_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2008_07140_b200.statevector import init_state

    with pytest.raises(errors.DeviceError):
        init_state(3)


@pytest.mark.parametrize("work", [6.0, 20.0])
def test_plan_balanced_passes_keep_the_result(monkeypatch, work):
    """Opt-in pass balancing (QSV_BALANCE_WORK) moves gates between passes; the
    emulated plan must equal the unbalanced one (checked against the oracle
    elsewhere), and gates must really have moved."""
    n = 12
    prog = parse_program(workloads.rqc_for_qubits(n, 10, 3))
    recs = compile_gates(prog.gate_instructions())
    psi0 = workloads.gaussian_state(n, 5)
    cfg = dict(tile_qubits=7, reg_qubits=3, low_qubits=2)
    monkeypatch.setenv("QSV_PLAN_ROLLOUT", "0")  # greedy tiles (front-loaded work to balance)
    monkeypatch.setenv("QSV_BALANCE_WORK", "0")
    _, flat = build_plan(recs, n, **cfg)
    monkeypatch.setenv("QSV_BALANCE_WORK", str(work))
    _, bal = build_plan(recs, n, **cfg)
    outs = []
    for passes in (flat, bal):
        psi = psi0.copy()
        execute(passes, n, psi)
        outs.append(psi)
    assert np.abs(outs[0] - outs[1]).max() <= 1e-12
    assert [len(p["ops"]) for p in flat] != [len(p["ops"]) for p in bal]


@pytest.mark.parametrize("seed", range(3))
def test_plan_swaps_relabel_qubits(seed):
    """Uncontrolled SWAPs become a qubit relabelling (no data movement) with
    restoring SWAPs at the end; controlled SWAPs stay gates."""
    rng = np.random.default_rng(seed)
    n = 9
    swap = np.eye(4)[[0, 2, 1, 3]]
    items = []
    for _ in range(80):
        qs = [int(q) for q in rng.permutation(n)]
        k = rng.integers(0, 4)
        if k == 0:
            items.append((swap, (qs[0], qs[1]), ()))
        elif k == 1:
            items.append((swap, (qs[0], qs[1]), (qs[2],)))
        elif k == 2:
            z = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
            q2, _ = np.linalg.qr(z)
            items.append((q2, (qs[0],), tuple(qs[1:1 + int(rng.integers(0, 2))])))
        else:
            items.append((np.diag(np.exp(1j * rng.uniform(0, 6, 4))), (qs[0], qs[1]), ()))
    recs = N.gate_records(items)
    psi0 = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
    ref = O.OracleState(n, psi0.copy(), 0)
    for u, t, c in items:
        O.apply_gate(ref, u, t, c)
    for cfg in CONFIGS:
        info, passes = build_plan(recs, n, **cfg)
        psi = psi0.copy()
        execute(passes, n, psi)
        assert np.abs(psi - ref.amplitudes).max() <= 1e-12, cfg
    # QFT round trip: the forward and inverse SWAP layers cancel, no SWAP op remains
    prog = parse_program(workloads.qft_text(12, round_trip=True))
    _, passes = build_plan(compile_gates(prog.gate_instructions()), 12, tile_qubits=8, reg_qubits=4, low_qubits=3)
    assert not any(o["kind"] == 2 and np.allclose(o["m"][:16].reshape(4, 4), swap) for p in passes for o in p["ops"])


def test_plan_objective_option():
    """qsv_options.plan_objective: the look-ahead minimises the modeled pass time (default) or
    the number of passes (1).  Both schedules reproduce the oracle; on the C2 circuit the time
    objective needs no more passes and spreads the non-diagonal gates more evenly."""
    prog = parse_program(workloads.rqc_for_qubits(14, 10, 3))
    recs = compile_gates(prog.gate_instructions())
    ref = O.run_full(prog).state.amplitudes
    for objective in (0, 1, 2):
        _, passes = build_plan(recs, 14, tile_qubits=6, reg_qubits=3, low_qubits=2, plan_objective=objective)
        psi = np.zeros(1 << 14, complex)
        psi[0] = 1
        execute(passes, 14, psi)
        assert np.abs(psi - ref).max() <= 1e-12, objective
    c2 = compile_gates(parse_program(workloads.rqc_text(5, 6, 24, 0)).gate_instructions())

    def mixing_per_pass(objective):
        info, passes = build_plan(c2, 30, plan_objective=objective)
        return info.passes, [sum(1 for o in p["ops"] if o["kind"] in (N.QSV_OP_MAT1, N.QSV_OP_MAT2)) for p in passes]

    n_time, w_time = mixing_per_pass(0)
    n_pass, w_pass = mixing_per_pass(1)
    assert n_time <= n_pass + 1
    assert max(w_time) <= max(w_pass) and min(w_time) >= min(w_pass)
