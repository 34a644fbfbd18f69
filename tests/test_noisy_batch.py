"""Batched noisy trajectories for every Kraus channel (noisy_batch.py) against
the oracle's restatement of the reference trajectory semantics
(oracle.sample_noisy_gate / measure, restating noise.py:188-222 and
statevector.py:298-308), trajectory by trajectory with the same seeds."""

import numpy as np
import pytest

from paper_2008_07140_b200 import _native as N
from paper_2008_07140_b200.noise import make_noise_model
from paper_2008_07140_b200.program import parse_program
from paper_2008_07140_b200.rqc import RqcConfig, generate_rqc


def test_step_symbol_declared_and_exported():
    from conftest import ROOT

    assert "qsv_noisy_batch_step" in (ROOT / "include" / "qsv.h").read_text()
    assert hasattr(N.lib(), "qsv_noisy_batch_step")


def _program(extra=""):
    return parse_program(generate_rqc(RqcConfig(2, 4, depth=6, seed=7)) + extra)


@pytest.mark.gpu
@pytest.mark.parametrize("kind,p", [("ampdamp", 0.15), ("depolarizing", 0.08), ("phasedamp", 0.2),
                                    ("bitflip", 0.9), ("bitphaseflip", 0.95)])
def test_batched_trajectories_match_oracle(kind, p):
    from oracle import oracle as O
    from paper_2008_07140_b200.noisy_batch import run_noisy_batch

    prog = _program("PMEASURE 0,3,5\n")
    B = 16
    seeds = [1000 + t for t in range(B)]
    res = run_noisy_batch(prog, make_noise_model(kind, p), [np.random.default_rng(s) for s in seeds])
    try:
        for t, s in enumerate(seeds):
            ref = O.run_full(prog, np.random.default_rng(s), (kind, p))
            got = res.amplitudes(t)
            assert np.abs(got - ref.state.amplitudes).max() <= 1e-10, (kind, t)
            (q, table), = res.tables[t]
            (rq, rtable), = ref.tables
            assert tuple(q) == tuple(rq)
            assert np.abs(table - rtable).max() <= 1e-12
    finally:
        res.close()


@pytest.mark.gpu
def test_batched_measure_and_noise_free_gates():
    """MEASURE per trajectory (own draw, own collapse) between noiseless and
    noisy gates (noise only on CNOT)."""
    from oracle import oracle as O
    from paper_2008_07140_b200.noisy_batch import run_noisy_batch

    text = "QINIT 6\nCREG 2\n" + "".join(f"H {q}\n" for q in range(6)) + \
        "CNOT 0,1\nT 1\nMEASURE 1,$0\nCNOT 1,2\nRY 3,\"0.4\"\nCNOT 3,4\nMEASURE 4,$1\nCNOT 4,5\nPMEASURE 5,2\n"
    prog = parse_program(text)
    B = 32
    seeds = list(range(B))
    model = make_noise_model("ampdamp", 0.3, ["CNOT"])
    res = run_noisy_batch(prog, model, [np.random.default_rng(s) for s in seeds])
    try:
        outcomes = set()
        for t, s in enumerate(seeds):
            rng = np.random.default_rng(s)
            st = O.init_state(6)
            st.amplitudes[:] = 0
            st.amplitudes[0] = 1
            cregs = [0, 0]
            tables = []
            for inst in prog.instructions:
                if inst.name == "CNOT":
                    base, targets, controls = O.controlled_form(inst)
                    k1 = O.kraus_ops("ampdamp", 0.3)
                    O.sample_noisy_gate(st, O.embed_controls(base, 1), controls + targets,
                                        [np.kron(a, b) for a in k1 for b in k1], rng)
                else:
                    r = O.OracleResult(cregs=cregs)
                    O.apply_instruction(st, inst, rng, None, r)
                    tables += r.tables
            assert res.cregs[t] == cregs
            outcomes.add(tuple(cregs))
            assert np.abs(res.amplitudes(t) - st.amplitudes).max() <= 1e-10
            assert np.abs(res.tables[t][0][1] - tables[0][1]).max() <= 1e-12
        assert len(outcomes) > 1  # the trajectories really diverge
    finally:
        res.close()


@pytest.mark.gpu
def test_batched_matches_sequential_run_full():
    """The batched engine and the sequential reference-shaped path (run_full with a
    noise model) draw identically: same branch choices, same amplitudes."""
    from paper_2008_07140_b200.noisy_batch import run_noisy_batch
    from paper_2008_07140_b200.statevector import run_full

    prog = parse_program(generate_rqc(RqcConfig(3, 4, depth=8, seed=3)))
    model = make_noise_model("depolarizing", 0.02)
    B = 8
    res = run_noisy_batch(prog, model, [np.random.default_rng(50 + t) for t in range(B)])
    try:
        for t in range(B):
            ref = run_full(prog, np.random.default_rng(50 + t), model,
                           noise_engine="sequential").state.amplitudes
            assert np.abs(res.amplitudes(t) - ref).max() <= 1e-10
    finally:
        res.close()


@pytest.mark.gpu
def test_batched_without_noise_and_single_trajectory():
    """noise=None: only MEASURE draws; B = 1 is the reference's single run_full."""
    from oracle import oracle as O
    from paper_2008_07140_b200.noisy_batch import run_noisy_batch

    prog = parse_program("QINIT 3\nCREG 1\nH 0\nCNOT 0,1\nMEASURE 1,$0\nH 2\n")
    res = run_noisy_batch(prog, None, [np.random.default_rng(9)])
    try:
        ref = O.run_full(prog, np.random.default_rng(9))
        assert res.cregs[0] == ref.cregs
        assert np.abs(res.amplitudes(0) - ref.state.amplitudes).max() <= 1e-12
    finally:
        res.close()
    with pytest.raises(ValueError):
        run_noisy_batch(prog, None, [np.random.default_rng(0)] * 3)


@pytest.mark.gpu
def test_one_and_two_groups_agree():
    """Splitting the batch over two asynchronous states changes nothing per trajectory."""
    from paper_2008_07140_b200.noisy_batch import run_noisy_batch

    prog = _program("PMEASURE 1,2\n")
    model = make_noise_model("depolarizing", 0.05)
    a = run_noisy_batch(prog, model, [np.random.default_rng(70 + t) for t in range(8)], groups=1)
    b = run_noisy_batch(prog, model, [np.random.default_rng(70 + t) for t in range(8)], groups=2)
    try:
        assert a.choices == b.choices
        for t in range(8):
            assert np.abs(a.amplitudes(t) - b.amplitudes(t)).max() <= 1e-13
            assert np.abs(a.tables[t][0][1] - b.tables[t][0][1]).max() <= 1e-14
    finally:
        a.close()
        b.close()


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["fused", "sequential"])
def test_noisy_projectors_renormalise_like_reference(engine):
    """A noisy P0/P1 is renormalised by its post-apply norm (noise.py:219-221)."""
    from oracle import oracle as O
    from paper_2008_07140_b200.statevector import run_full

    from paper_2008_07140_b200.program import Instruction, Program

    # projectors are not user mnemonics (program.py:407); partial mode builds them as Instructions
    base = parse_program('QINIT 3\nH 0\nRY 1,"0.7"\nCNOT 0,2\nH 1\nRX 2,"0.3"\n').instructions
    prog = Program(3, 0, base[:3] + (Instruction("P1", (0,)),) + base[3:4] + (Instruction("P0", (1,)),) + base[4:])
    for s in range(6):
        res = run_full(prog, np.random.default_rng(s), make_noise_model("bitflip", 0.8), noise_engine=engine)
        ref = O.run_full(prog, np.random.default_rng(s), ("bitflip", 0.8))
        assert np.abs(res.state.amplitudes - ref.state.amplitudes).max() <= 1e-12
        res.state.close()


@pytest.fixture
def fake_native(monkeypatch):
    from fake_qsv import FakeLib

    from paper_2008_07140_b200 import statevector as SV

    fake = FakeLib()
    monkeypatch.setattr(N, "lib", lambda: fake)
    monkeypatch.setattr(SV, "_PLAN_CACHE", {})  # fake plan handles never reach the real library
    return fake


@pytest.mark.parametrize("groups", [1, 2])
@pytest.mark.parametrize("kind,p", [("ampdamp", 0.2), ("depolarizing", 0.1), ("phasedamp", 0.3)])
def test_host_logic_against_oracle_on_cpu(fake_native, groups, kind, p):
    """The batched host logic (draw order, weights from the upper-triangle reduced
    densities, branch choice, renormalisation, MEASURE/PMEASURE bookkeeping,
    grouping) over a numpy stand-in of the native steps, against the oracle's
    restatement of the reference sampling, trajectory by trajectory."""
    from oracle import oracle as O
    from paper_2008_07140_b200.noisy_batch import run_noisy_batch

    prog = parse_program(generate_rqc(RqcConfig(2, 3, depth=5, seed=4)) + "PMEASURE 0,4\n")
    B = 8
    res = run_noisy_batch(prog, make_noise_model(kind, p), [np.random.default_rng(300 + t) for t in range(B)],
                          groups=groups)
    for t in range(B):
        ref = O.run_full(prog, np.random.default_rng(300 + t), (kind, p))
        assert np.abs(res.amplitudes(t) - ref.state.amplitudes).max() <= 1e-12
        assert np.abs(res.tables[t][0][1] - ref.tables[0][1]).max() <= 1e-12
    assert len({tuple(c) for c in res.choices}) > 1  # trajectories took different branches


def test_host_measure_logic_on_cpu(fake_native):
    from oracle import oracle as O
    from paper_2008_07140_b200.noisy_batch import run_noisy_batch

    prog = parse_program("QINIT 4\nCREG 2\nH 0\nH 1\nCNOT 1,2\nMEASURE 2,$1\nRY 3,\"1.1\"\nMEASURE 3,$0\n")
    res = run_noisy_batch(prog, None, [np.random.default_rng(t) for t in range(16)])
    seen = set()
    for t in range(16):
        ref = O.run_full(prog, np.random.default_rng(t))
        assert res.cregs[t] == ref.cregs
        assert np.abs(res.amplitudes(t) - ref.state.amplitudes).max() <= 1e-12
        seen.add(tuple(ref.cregs))
    assert len(seen) > 2


@pytest.mark.parametrize("kind,p", [("depolarizing", 0.2), ("bitflip", 0.7), ("phaseflip", 0.6),
                                    ("bitphaseflip", 0.9)])
def test_presampled_mixed_unitary_run_full_on_cpu(fake_native, kind, p):
    """run_full under a mixed-unitary channel draws its branches up front and stays
    fused: same draws (MEASURE interleaved) and amplitudes as the oracle's reference
    sampling; one qsv_run per MEASURE-separated segment."""
    from oracle import oracle as O
    from paper_2008_07140_b200.statevector import run_full

    text = generate_rqc(RqcConfig(2, 3, depth=5, seed=8)).replace("QINIT 6", "QINIT 6\nCREG 2")
    prog = parse_program(text + "MEASURE 2,$0\nCNOT 2,3\nH 4\nMEASURE 4,$1\nCZ 0,5\nPMEASURE 1,3\n")
    for s in range(6):
        fake_native.run_calls = 0
        res = run_full(prog, np.random.default_rng(s), make_noise_model(kind, p))
        assert res.stats.get("noise_engine") == "presampled"
        assert fake_native.run_calls == 3  # the segments between MEASURE, MEASURE and PMEASURE
        ref = O.run_full(prog, np.random.default_rng(s), (kind, p))
        assert res.cregs == ref.cregs
        assert np.abs(res.state.amplitudes - ref.state.amplitudes).max() <= 1e-12
        assert np.abs(res.tables[0][1] - ref.tables[0][1]).max() <= 1e-12


def test_state_dependent_channels_are_not_presampled(fake_native):
    from paper_2008_07140_b200.statevector import _mixed_unitary

    prog = parse_program("QINIT 2\nH 0\nCNOT 0,1\n")
    assert _mixed_unitary(prog, make_noise_model("depolarizing", 0.1))
    assert not _mixed_unitary(prog, make_noise_model("ampdamp", 0.1))
    assert not _mixed_unitary(prog, make_noise_model("phasedamp", 0.1))


def test_chunked_batches_match_one_batch_on_cpu(fake_native):
    """Batches above max_batch_bytes run in power-of-two chunks with identical
    per-trajectory draws, outcomes and tables."""
    from paper_2008_07140_b200.noisy_batch import run_noisy_batch

    prog = parse_program(generate_rqc(RqcConfig(2, 3, depth=4, seed=6)).replace("QINIT 6", "QINIT 6\nCREG 1")
                         + "MEASURE 3,$0\nPMEASURE 0,2\n")
    model = make_noise_model("ampdamp", 0.25)
    whole = run_noisy_batch(prog, model, [np.random.default_rng(900 + t) for t in range(8)])
    parts = run_noisy_batch(prog, model, [np.random.default_rng(900 + t) for t in range(8)],
                            max_batch_bytes=2 * (16 << 6))
    assert parts.stats["chunks"] == 4
    assert parts.cregs == whole.cregs and parts.choices == whole.choices
    for a, b in zip(parts.tables, whole.tables):
        assert np.abs(a[0][1] - b[0][1]).max() <= 1e-14
    with pytest.raises(ValueError):
        parts.amplitudes(0)
