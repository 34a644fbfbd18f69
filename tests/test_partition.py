"""Partial-amplitude mode (reference pkg/tests/test_partition.py, partition.py:1-192).

CPU tests: plan / decomposition structure and errors (as the reference's
tests), and the batched branch streams executed through the specialised
pass kernels' HOST rendering (tests/jit_host.py) against amplitudes of the
real reference `run_partial` (tests/golden/partial.json, made by
tests/golden/make_golden_partial.py).  GPU tests: `run_partial` on the B200
against the same golden amplitudes and against full-state runs.
"""

import json
import math
from pathlib import Path

import numpy as np
import pytest

from paper_2008_07140_b200 import gates
from paper_2008_07140_b200.errors import BranchExplosion, MalformedTarget, UncuttableGate, UnsupportedGate
from paper_2008_07140_b200.partition import (
    batch_bits, branch_streams, decompose_crossing, parse_target, plan_partition, run_partial)
from paper_2008_07140_b200.program import parse_program
from paper_2008_07140_b200 import _native as N

GOLD = json.loads((Path(__file__).parent / "golden" / "partial.json").read_text())
INV_SQRT2 = 1 / math.sqrt(2)


def fig1_like_program():
    return parse_program(GOLD["fig1_8"]["text"])


def test_decomposition_identities():
    cz = np.kron(gates.P0, gates.I2) + np.kron(gates.P1, gates.Z)
    assert np.abs(cz - np.diag([1, 1, 1, -1])).max() == 0
    cnot = np.kron(gates.P0, gates.I2) + np.kron(gates.P1, gates.X)
    assert np.abs(cnot - np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]])).max() == 0


def test_plan_structure_and_errors():
    plan = plan_partition(fig1_like_program(), 4)
    assert (plan.c, plan.branch_count, plan.subcircuit_count) == (2, 4, 8)
    with pytest.raises(UncuttableGate):
        plan_partition(parse_program("QINIT 4\nH 0\nSWAP 1,2\n"), 2)
    with pytest.raises(UncuttableGate):
        plan_partition(parse_program("QINIT 4\nTOFFOLI 0,1,3\n"), 2)
    with pytest.raises(UncuttableGate):
        plan_partition(parse_program("QINIT 4\nH 0\n"), 0)
    with pytest.raises(UnsupportedGate):
        plan_partition(parse_program("QINIT 2\nCREG 1\nH 0\nMEASURE 0,$0\n"), 1)
    with pytest.raises(BranchExplosion):
        plan_partition(parse_program("QINIT 4\n" + "CZ 1,2\n" * 5), 2, branch_budget=16)
    plan = plan_partition(parse_program("QINIT 4\nH 0\nCNOT 0,1\nCNOT 2,3\n"), 2)
    assert (plan.c, plan.branch_count, plan.subcircuit_count) == (0, 1, 2)


def test_decompose_matches_reference_shape():
    plan = plan_partition(fig1_like_program(), 4)
    branches = decompose_crossing(plan)
    assert [b.branch_id for b in branches] == [0, 1, 2, 3]
    for b in branches:
        assert b.upper_program.qubit_count == 4 and b.lower_program.qubit_count == 4
        for inst in b.upper_program.instructions + b.lower_program.instructions:
            assert all(0 <= q < 4 for q in inst.all_qubits())
    b0, b1 = decompose_crossing(plan_partition(parse_program("QINIT 2\nH 0\nCNOT 0,1\n"), 1))
    assert [i.name for i in b0.lower_program.instructions] == ["H", "P0"]
    assert [i.name for i in b0.upper_program.instructions] == []
    assert [i.name for i in b1.lower_program.instructions] == ["H", "P1"]
    assert [i.name for i in b1.upper_program.instructions] == ["U4"]
    assert np.array_equal(np.array(b1.upper_program.instructions[0].matrix).reshape(2, 2), gates.X)


def test_parse_target():
    assert parse_target("101", 3) == 5
    with pytest.raises(MalformedTarget):
        parse_target("0", 2)
    with pytest.raises(MalformedTarget):
        parse_target("02", 2)


def test_batch_bits_split():
    plan = plan_partition(parse_program(GOLD["rqc_2x7_s2"]["text"]), 7)
    assert plan.c == 14
    assert batch_bits(plan, 28) == 14
    assert batch_bits(plan, 12) == 5
    assert batch_bits(plan, 3) == 0


def _dense_run(triplets, m, cb):
    """Numpy dense application of the batched stream (independent of libqsv)."""
    from plan_emulator import _apply

    psi = np.zeros(1 << m, dtype=np.complex128)
    psi[: 1 << cb] = 1.0
    for u, targets, controls in triplets:
        cm = 0
        for c in controls:
            cm |= 1 << c
        _apply(psi, m, np.asarray(u), tuple(targets), cm)
    return psi


def _host_kernels_run(triplets, m, cb):
    """The same stream through libqsv's planner + the specialised kernels' host rendering."""
    from jit_host import run_plan_host

    psi = np.zeros(1 << m, dtype=np.complex128)
    psi[: 1 << cb] = 1.0
    if not triplets:
        return psi
    return run_plan_host(N.gate_records(triplets), m, psi)


def _recombine(name, batch_qubits, runner):
    g = GOLD[name]
    prog = parse_program(g["text"])
    n, cut = prog.qubit_count, g["cut"]
    plan = plan_partition(prog, cut)
    cb = batch_bits(plan, max(batch_qubits, max(cut, n - cut)))
    idx = [parse_target(t, n) for t in g["targets"]]
    got = np.zeros(len(idx), dtype=np.complex128)
    for fixed in range(1 << (plan.c - cb)):
        (tl, ml), (tu, mu) = branch_streams(plan, cb, fixed)
        lo = runner(tl, ml, cb).reshape(-1, 1 << cb)
        up = runner(tu, mu, cb).reshape(-1, 1 << cb)
        for k, i in enumerate(idx):
            got[k] += np.dot(up[i >> cut], lo[i & ((1 << cut) - 1)])
    want = np.array(g["re"]) + 1j * np.array(g["im"])
    return np.abs(got - want).max()


@pytest.mark.parametrize("name", sorted(GOLD))
@pytest.mark.parametrize("batch_qubits", [0, 9, 64])
def test_branch_streams_dense(name, batch_qubits):
    """Batched selector streams reproduce the reference's partial amplitudes,
    with all, some and none of the selector bits as branch qubits."""
    assert _recombine(name, batch_qubits, _dense_run) <= 1e-12


@pytest.mark.parametrize("name", ["fig1_8", "rqc_1x8_s5", "rqc_1x16_s4", "rqc_2x7_s2"])
def test_branch_streams_through_host_kernels(name):
    """Projector diagonals and branch-controlled actions through the real
    planner and generated kernel code (host rendering)."""
    assert _recombine(name, 18, _host_kernels_run) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD))
@pytest.mark.parametrize("batch_qubits", [0, 64])
def test_run_partial_gpu_golden(name, batch_qubits):
    g = GOLD[name]
    amps = run_partial(parse_program(g["text"]), g["cut"], g["targets"], batch_qubits=batch_qubits)
    want = np.array(g["re"]) + 1j * np.array(g["im"])
    got = np.array([amps[t] for t in g["targets"]])
    assert np.abs(got - want).max() <= 1e-10


@pytest.mark.gpu
def test_run_partial_gpu_matches_full_state():
    """A 24-qubit RQC cut in the middle (c = 12 branch qubits per 12-qubit half
    -> two 24-qubit batched states) against the full-state engine."""
    from paper_2008_07140_b200.rqc import RqcConfig, generate_rqc
    from paper_2008_07140_b200.statevector import run_full

    prog = parse_program(generate_rqc(RqcConfig(4, 6, depth=8, seed=11)))
    n = prog.qubit_count
    cut = 12
    plan = plan_partition(prog, cut)
    assert plan.c == 12
    rng = np.random.default_rng(3)
    idx = sorted({int(i) for i in rng.integers(0, 1 << n, 200)})
    targets = [format(i, f"0{n}b") for i in idx]
    amps = run_partial(prog, cut, targets)
    full = run_full(prog).state.amplitudes
    assert max(abs(amps[t] - full[i]) for t, i in zip(targets, idx)) <= 1e-10
    # the norm over all targets of a small program (reference test_norm_consistency)
    small = parse_program(GOLD["rqc_1x8_s0"]["text"])
    all_t = [format(i, "08b") for i in range(256)]
    tot = sum(abs(a) ** 2 for a in run_partial(small, 4, all_t).values())
    assert tot == pytest.approx(1.0, abs=1e-9)


@pytest.mark.gpu
def test_run_partial_gpu_edge_cases():
    """No targets, duplicate targets, no crossing gates (c = 0), PMEASURE ignored."""
    prog = parse_program("QINIT 4\nH 0\nCNOT 0,1\nH 2\nCNOT 2,3\nPMEASURE 0,1\n")
    assert run_partial(prog, 2, []) == {}
    amps = run_partial(prog, 2, ["0000", "0000", "1111"])
    assert list(amps) == ["0000", "1111"]
    assert abs(amps["0000"] - 0.5) < 1e-12 and abs(amps["1111"] - 0.5) < 1e-12


def _sharded_partial_worker(rank, world, port, name, batch_qubits, out):
    import os
    import sys

    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(__file__))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from fake_qsv import FakeLib

        fake = FakeLib()
        N.lib = lambda: fake  # numpy stand-in for the native steps (this process only)
        g = GOLD[name]
        amps = run_partial(parse_program(g["text"]), g["cut"], g["targets"], batch_qubits=batch_qubits,
                           rank=rank, world=world)
        if rank == 0:
            np.save(out, np.array([amps[t] for t in g["targets"]]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,batch_qubits", [("rqc_1x8_s0", 64), ("rqc_1x16_s4", 0), ("rqc_2x7_s2", 12)])
def test_sharded_partial_over_gloo(name, batch_qubits, tmp_path):
    """Selector runs dealt over 2 ranks + one all-reduce of the per-target sums
    reproduce the reference's partial amplitudes (host logic over gloo)."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "amps.npy")
    mp.spawn(_sharded_partial_worker, args=(2, port, name, batch_qubits, out), nprocs=2, join=True)
    g = GOLD[name]
    want = np.array(g["re"]) + 1j * np.array(g["im"])
    assert np.abs(np.load(out) - want).max() <= 1e-12
