"""Host-side mirror of the reference front end vs reference outputs (CPU)."""

import math

import numpy as np
import pytest

from paper_2008_07140_b200 import errors, gates, noise, rqc, workloads
from paper_2008_07140_b200.program import (
    Instruction,
    eval_angle,
    expand_control,
    expand_dagger,
    parse_complex_literal,
    parse_program,
    to_script,
)


def _inst_matches(inst, rec):
    assert inst.name == rec["name"]
    assert list(inst.qubits) == rec["qubits"]
    assert list(inst.controls) == rec["controls"]
    assert inst.creg == rec["creg"]
    assert inst.line == rec["line"]
    assert list(inst.params) == rec["params"]
    if rec["matrix"] is None:
        assert inst.matrix is None
    else:
        got = np.array(inst.matrix, dtype=complex)
        want = np.array([complex(*z) for z in rec["matrix"]])
        assert np.array_equal(got, want), (inst, rec)
    if "base" in rec:
        base, targets, controls = gates.controlled_form(inst)
        assert list(targets) == rec["targets"] and list(controls) == rec["all_controls"]
        want = np.array([complex(*z) for z in rec["base"]])
        assert np.array_equal(np.asarray(base).reshape(-1), want), inst
    if "base_error" in rec:
        with pytest.raises(getattr(errors, rec["base_error"])):
            gates.controlled_form(inst)


@pytest.mark.parametrize("bucket", ["programs", "random_programs"])
def test_parse_matches_reference(golden, bucket):
    for name, rec in golden[bucket].items():
        prog = parse_program(rec["text"])
        assert prog.qubit_count == rec["qubit_count"] and prog.creg_count == rec["creg_count"]
        assert len(prog.instructions) == len(rec["instructions"]), name
        for inst, irec in zip(prog.instructions, rec["instructions"]):
            _inst_matches(inst, irec)
        assert to_script(prog) == rec["to_script"], name
        assert parse_program(to_script(prog)) == prog


def test_error_corpus(golden):
    from paper_2008_07140_b200.statevector import DEFAULT_MAX_QUBITS

    for name, rec in golden["errors"].items():
        if rec["stage"] == "parse":
            with pytest.raises(getattr(errors, rec["error"])) as exc:
                parse_program(rec["text"])
            assert exc.value.line == rec["line"], name
            assert exc.value.render() == rec["render"], name
            assert exc.value.exit_code == rec["exit_code"]
        else:
            prog = parse_program(rec["text"])
            if rec["stage"] == "run" and rec["error"] == "TooManyQubits":
                assert prog.qubit_count > DEFAULT_MAX_QUBITS
            elif rec["stage"] == "run":
                with pytest.raises(getattr(errors, rec["error"])) as exc:
                    for inst in prog.gate_instructions():
                        gates.controlled_form(inst)
                assert exc.value.line == rec["line"]


def test_angles_and_literals(golden):
    for expr, want in golden["angles"].items():
        if want == "MalformedAngle":
            with pytest.raises(errors.MalformedAngle):
                eval_angle(expr)
        else:
            assert eval_angle(expr) == want, expr
    for lit, (re_, im_) in golden["complex"].items():
        assert parse_complex_literal(lit) == complex(re_, im_), lit


def test_golden_pmeasure_format_helper(golden):
    assert golden["format_pmeasure"]["golden"].splitlines()[0] == "000: 0.820083"


def test_dagger_and_control_algebra():
    inv = expand_dagger([Instruction("H", (0,)), Instruction("S", (0,))])
    assert [i.name for i in inv] == ["U4", "H"]
    assert np.allclose(np.array(inv[0].matrix).reshape(2, 2), gates.S.conj().T)
    assert expand_dagger([Instruction("RY", (3,), params=(0.5,))])[0].params == (-0.5,)
    ctl = expand_control([Instruction("CNOT", (1, 0))], 2)
    assert ctl[0].controls == (2,)
    with pytest.raises(errors.ControlQubitCollision):
        expand_control([Instruction("H", (0,))], 0)


def test_reference_rqc_generator_byte_identical(golden):
    for rec in golden["rqc"]:
        cfg = rqc.RqcConfig(rec["rows"], rec["cols"], rec["depth"], rec["seed"],
                            pmeasure=tuple(rec.get("pmeasure", ())))
        assert rqc.generate_rqc(cfg) == rec["text"]


@pytest.mark.parametrize("rows,cols", [(4, 5), (5, 6), (4, 8), (3, 11), (2, 17), (5, 7), (4, 6)])
def test_eight_pattern_rqc_properties(rows, cols):
    cfg = rqc.RqcConfig(rows, cols, 16, seed=3, patterns=8, no_repeat=True)
    edges = set()
    for layer in range(8):
        seen = set()
        for a, b in rqc.layer_pairs(cfg, layer):
            assert a not in seen and b not in seen
            seen.update((a, b))
            dr, dc = b // cols - a // cols, b % cols - a % cols
            assert (dr, dc) in ((0, 1), (1, 0))
            assert (a, b) not in edges
            edges.add((a, b))
    all_edges = {(r * cols + c, r * cols + c + 1) for r in range(rows) for c in range(cols - 1)}
    all_edges |= {(r * cols + c, (r + 1) * cols + c) for r in range(rows - 1) for c in range(cols)}
    assert edges == all_edges  # every grid edge exactly once per 8 cycles
    prog = parse_program(rqc.generate_rqc(cfg))
    last = {}
    for inst in prog.instructions[rows * cols:]:
        if inst.name in ("RX", "RY", "T"):
            q = inst.qubits[0]
            assert last.get(q) != inst.name  # never the same pool gate twice in a row
            last[q] = inst.name


def test_workload_grid_shapes():
    assert [workloads.grid_shape(n) for n in (20, 24, 30, 31, 32, 33, 34, 35)] == [
        (4, 5), (4, 6), (5, 6), (6, 6), (4, 8), (6, 6), (6, 6), (5, 7)]


def test_partial_row_grid_edges():
    """31 qubits on 6 columns: the last row holds one qubit; every CZ is a grid edge
    between existing qubits, no qubit is touched twice per cycle, and over 8 cycles
    every existing edge appears exactly once (the 8-pattern property)."""
    cfg = rqc.RqcConfig(6, 6, 8, 0, patterns=8, no_repeat=True, qubits=31)
    seen = []
    for layer in range(8):
        pairs = rqc.layer_pairs(cfg, layer)
        flat = [q for pr in pairs for q in pr]
        assert len(flat) == len(set(flat)) and max(flat) < 31
        for a, b in pairs:
            assert b - a in (1, 6) and (b - a != 1 or a // 6 == b // 6)
        seen += pairs
    edges = {(a, a + 1) for a in range(31) if a % 6 != 5 and a + 1 < 31} | {(a, a + 6) for a in range(31) if a + 6 < 31}
    assert sorted(seen) == sorted(edges)
    assert parse_program(workloads.rqc_for_qubits(31, 4, 0)).qubit_count == 31


def test_pauli_insertion_replays_reference_draws(golden):
    """Host pre-sampling reproduces the reference's branch choices exactly."""
    for rec in golden["noise"]:
        prog = parse_program(rec["text"])
        ins = workloads.sample_pauli_insertions(prog, rec["p"], rec["traj_seed"])
        nonzero = [i for i, c in enumerate(rec["choices"]) if c]
        gate_idx = [i for i, inst in enumerate(prog.instructions) if inst.is_gate]
        assert sorted(ins) == [gate_idx[i] for i in nonzero]
        for k, c in enumerate(rec["choices"]):
            idx = gate_idx[k]
            if not c:
                continue
            inst = prog.instructions[idx]
            _, t, ctl = gates.controlled_form(inst)
            qs = tuple(ctl) + tuple(t)
            want = [(qs[0], "IXYZ"[c])] if len(qs) == 1 else [(qs[0], "IXYZ"[c // 4]), (qs[1], "IXYZ"[c % 4])]
            assert ins[idx] == [(q, g) for q, g in want if g != "I"]


def test_noise_models():
    for kind in noise.KINDS:
        for p in (0.0, 0.3, 1.0):
            ops = noise.kraus_ops(kind, p)
            assert np.abs(sum(k.conj().T @ k for k in ops) - np.eye(2)).max() <= 1e-12
    assert len(noise.two_qubit_kraus(noise.NoiseChannel("depolarizing", 0.1),
                                     noise.NoiseChannel("bitflip", 0.2))) == 8
    with pytest.raises(errors.InvalidProbability):
        noise.parse_noise_spec("bitflip:2.0")
    assert noise.parse_noise_spec("depolarizing:0.1:CNOT,CZ").rules[0].mnemonics == frozenset({"CNOT", "CZ"})


def test_gaussian_state_recipe():
    g = np.random.default_rng(7)
    v = g.standard_normal(1 << 9) + 1j * g.standard_normal(1 << 9)
    v /= np.linalg.norm(v)
    assert np.abs(workloads.gaussian_state(9, 7, chunk=100) - v).max() < 1e-15


def test_qft_text_shape():
    prog = parse_program(workloads.qft_text(30))
    names = [i.name for i in prog.instructions]
    assert names.count("H") == 30 and names.count("CR") == 435 and names.count("SWAP") == 15
    rt = parse_program(workloads.qft_text(5, round_trip=True))
    assert len(rt.instructions) == 2 * len(parse_program(workloads.qft_text(5)).instructions)
    crs = [i for i in prog.instructions if i.name == "CR"]
    assert crs[0].qubits == (28, 29) and crs[0].params[0] == math.pi / 2
    assert max(crs, key=lambda i: i.qubits[1] - i.qubits[0]).params[0] == math.pi / 536870912
