"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Test infrastructure only.  Run in the build container, where the reference
package is importable read-only:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

It imports `qcsim` (reference `pkg/src/qcsim`) and records, for a fixed set
of seeded inputs, what the reference itself computes:

* programs.json  - script text -> expanded instruction stream
                   (reference `program.parse_program`, program.py:369-476),
                   `gates.controlled_form` per instruction (gates.py:150-159),
                   error-corpus outcomes (errors.py classes + line numbers),
                   RQC texts (rqc.py:64-85), format_pmeasure text (cli.py:23-34)
* states.npz     - final amplitudes / PMEASURE tables / cregs of
                   `statevector.run_full` (statevector.py:397-430), kernel-API
                   random-gate streams (statevector.py:255-289, mirrors
                   tests/test_statevector.py:218-250), QFT on a random state
                   via `apply_instruction` (statevector.py:360-394), noisy
                   depolarising trajectories (noise.py:188-222), a QSVDUMP
                   byte image (cli.py:37-42) and sampled amplitudes of the
                   20-qubit C1 circuit.

/root/reference does not exist on the GPU box; only the committed outputs
travel.  Nothing in the product imports this file.
"""

from __future__ import annotations

import io
import json
import math
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import qcsim  # noqa: E402
from qcsim import errors as qerr  # noqa: E402
from qcsim import gates as qgates  # noqa: E402
from qcsim import noise as qnoise  # noqa: E402
from qcsim import program as qprog  # noqa: E402
from qcsim import rqc as qrqc  # noqa: E402
from qcsim import statevector as qsv  # noqa: E402
from qcsim.cli import format_pmeasure, save_state  # noqa: E402
from qcsim.parallel import WorkerPool  # noqa: E402

HERE = Path(__file__).parent
REPO = HERE.parent.parent
sys.path.insert(0, str(REPO))


def cplx(z):
    return [float(np.real(z)), float(np.imag(z))]


def inst_record(inst):
    rec = {
        "name": inst.name,
        "qubits": list(inst.qubits),
        "params": [float(p) for p in inst.params],
        "matrix": None if inst.matrix is None else [cplx(z) for z in inst.matrix],
        "controls": list(inst.controls),
        "creg": inst.creg,
        "line": inst.line,
    }
    if inst.is_gate:
        try:
            base, targets, controls = qgates.controlled_form(inst)
            rec["base"] = [cplx(z) for z in np.asarray(base).reshape(-1)]
            rec["targets"] = list(targets)
            rec["all_controls"] = list(controls)
        except qerr.SimulatorError as exc:
            rec["base_error"] = type(exc).__name__
    return rec


def program_record(text):
    prog = qprog.parse_program(text)
    return {
        "text": text,
        "qubit_count": prog.qubit_count,
        "creg_count": prog.creg_count,
        "instructions": [inst_record(i) for i in prog.instructions],
        "to_script": qprog.to_script(prog),
    }


# --------------------------------------------------------------------------
# inputs
# --------------------------------------------------------------------------

GOLDEN_TEXT = (REF / "tests/data/golden.qprog").read_text()

SMALL_PROGRAMS = {
    "golden": GOLDEN_TEXT,
    "minimal": "QINIT 2\nCREG 1\nH 0\nPMEASURE 0\n",
    "ghz": "QINIT 3\nH 0\nCNOT 0,1\nCNOT 1,2\nPMEASURE 2,1,0\n",
    "comments": "% hello\nQINIT 1\n\n% more\nX 0\n",
    "spaces": "QINIT 3\nCNOT 0 , 2\n",
    "dagger_mix": 'QINIT 4\nDAGGER\nS 0\nT 1\niSWAP 1,2\nENDDAGGER\nU4 3,"0.1,0.2,0.3,0.4"\n',
    "control_nest": "QINIT 3\nCONTROL 2\nCONTROL 1\nX 0\nENDCONTROL 1\nENDCONTROL 2\n",
    "control_dagger": "QINIT 3\nCONTROL 2\nDAGGER\nS 0\nCNOT 0,1\nENDDAGGER\nENDCONTROL 2\n",
    "rx_cnot_measure": 'QINIT 3\nCREG 2\nRX 1,"pi/2"\nCNOT 0,2\nMEASURE 2,$1\n',
    "u4_element": 'QINIT 1\nU4 0,"0,1+0i,1+0i,0"\n',
    "u4_complex": 'QINIT 2\nU4 1,"0.6+0i,0.8i,0.8i,0.6"\nH 0\n',
    "angles": 'QINIT 2\nRX 0,"2*pi/3"\nRY 1,"-3.5*2"\nRZ 0,"1e-3"\nCR 0,1,"-pi/8"\n',
    "iswap_dagger": "QINIT 2\nH 0\nDAGGER\niSWAP 0,1\nENDDAGGER\n",
    "measure_seq": "QINIT 3\nCREG 3\nH 0\nH 1\nH 2\nMEASURE 0,$0\nMEASURE 1,$1\nMEASURE 2,$2\nPMEASURE 2,1,0\n",
    "measure_x": "QINIT 2\nCREG 2\nX 0\nMEASURE 0,$1\nMEASURE 1,$0\n",
    "bell_measure": "QINIT 2\nCREG 1\nH 0\nCNOT 0,1\nMEASURE 0,$0\nPMEASURE 1,0\n",
    "invariance": "QINIT 6\nH 0\nCNOT 0,5\nRY 2,\"0.37\"\nCZ 1,4\nCR 0,3,\"pi/4\"\nSWAP 1,2\nT 3\nTOFFOLI 0,1,5\n",
    "controlled_swap": "QINIT 4\nH 1\nH 3\nCONTROL 3\nSWAP 1,0\nENDCONTROL 3\nCONTROL 2\nCONTROL 0\niSWAP 1,3\nENDCONTROL 0\nENDCONTROL 2\n",
}

ERROR_CORPUS = sorted((REF / "tests/data/errors").glob("*.qprog"))

EXTRA_ERRORS = {
    "unbalanced_enddagger": "QINIT 1\nENDDAGGER\n",
    "mismatch_control": "QINIT 3\nCONTROL 1\nH 0\nENDCONTROL 2\n",
    "control_enddagger": "QINIT 2\nCONTROL 1\nH 0\nENDDAGGER\n",
    "duplicate_toffoli": "QINIT 3\nTOFFOLI 0,2,2\n",
    "p0_mnemonic": "QINIT 1\nP0 0\n",
    "measure_in_dagger_p": "QINIT 1\nDAGGER\nPMEASURE 0\nENDDAGGER\n",
    "dup_qinit": "QINIT 1\nQINIT 2\n",
    "bad_qinit": "QINIT x\n",
    "zero_qinit": "QINIT 0\n",
    "creg_negative": "QINIT 1\nCREG -1\n",
    "measure_noreg": "QINIT 1\nCREG 1\nMEASURE 0,0\n",
    "unterminated": 'QINIT 1\nRX 0,"pi\n',
    "u4_count": 'QINIT 1\nU4 0,"1,0,0"\n',
    "arity": "QINIT 2\nCNOT 0\n",
    "bad_qubit": "QINIT 2\nH a\n",
    "pmeasure_dup": "QINIT 2\nPMEASURE 0,0\n",
    "pmeasure_empty": "QINIT 2\nPMEASURE\n",
    "angle_plus": 'QINIT 1\nRZ 0,"pi+1"\n',
    "only_comments": "% only comments\n",
}

ANGLE_EXPRS = ["pi/2", "-pi/4", "-pi/8", "0", "2*pi/3", "0.25", "1e-3", "-3.5*2",
               "--pi", "pi*pi/4", ".5", "3.", "pi/536870912", "-0.0"]
BAD_ANGLES = ["", "pi+1", "pie", "(pi)", "1//2", "2*", "x"]
COMPLEX_LITS = ["1", "-0.5", "2i", "-i", "1-2i", "1e-3+2.5i", "i", "+i", "0.6+0.8i", "1e-3-1e-2i"]

RQC_CONFIGS = [(1, 2, 1, 7), (2, 3, 8, 42), (2, 3, 8, 1), (3, 3, 10, 0), (3, 4, 12, 9),
               (4, 5, 20, 0), (2, 13, 10, 26), (4, 6, 20, 3)]


def random_program_text(rng, n, n_gates):
    """Seeded program over the whole mnemonic set incl. CONTROL/DAGGER blocks."""
    lines = [f"QINIT {n}"]
    one = ["H", "X", "Y", "Z", "S", "T"]
    rot = ["RX", "RY", "RZ"]

    def gate_line(avoid=()):
        qs = [q for q in range(n) if q not in avoid]
        kind = int(rng.integers(0, 8))
        if kind == 0 or len(qs) < 2:
            return f"{one[int(rng.integers(0, 6))]} {int(rng.choice(qs))}"
        if kind == 1:
            return f'{rot[int(rng.integers(0, 3))]} {int(rng.choice(qs))},"{rng.uniform(-4, 4):.6f}"'
        if kind == 2:
            a = rng.uniform(-3, 3, size=4)
            return f'U4 {int(rng.choice(qs))},"{a[0]:.5f},{a[1]:.5f},{a[2]:.5f},{a[3]:.5f}"'
        pair = [int(x) for x in rng.choice(qs, size=2, replace=False)]
        if kind == 3:
            return f"CNOT {pair[0]},{pair[1]}"
        if kind == 4:
            return f"CZ {pair[0]},{pair[1]}"
        if kind == 5:
            return f'CR {pair[0]},{pair[1]},"pi/{int(rng.integers(1, 9))}"'
        if kind == 6:
            return f"{'SWAP' if rng.random() < 0.5 else 'iSWAP'} {pair[0]},{pair[1]}"
        if len(qs) >= 3:
            t = [int(x) for x in rng.choice(qs, size=3, replace=False)]
            return f"TOFFOLI {t[0]},{t[1]},{t[2]}"
        return f"CNOT {pair[0]},{pair[1]}"

    i = 0
    while i < n_gates:
        r = rng.random()
        if r < 0.08 and n >= 3:
            c = int(rng.integers(0, n))
            lines.append(f"CONTROL {c}")
            for _ in range(int(rng.integers(1, 4))):
                lines.append(gate_line(avoid=(c,)))
                i += 1
            lines.append(f"ENDCONTROL {c}")
        elif r < 0.14:
            lines.append("DAGGER")
            for _ in range(int(rng.integers(1, 5))):
                lines.append(gate_line())
                i += 1
            lines.append("ENDDAGGER")
        else:
            lines.append(gate_line())
            i += 1
    return "\n".join(lines) + "\n"


def qft_text(n):
    """Little-endian QFT: H j, CR i,j for i<j, then swaps."""
    lines = [f"QINIT {n}"]
    body = []
    for j in range(n - 1, -1, -1):
        body.append(f"H {j}")
        for i in range(j - 1, -1, -1):
            body.append(f'CR {i},{j},"pi/{2 ** (j - i)}"')
    for q in range(n // 2):
        body.append(f"SWAP {q},{n - 1 - q}")
    return lines + body


def main():
    out = {"programs": {}, "errors": {}, "angles": {}, "complex": {}, "rqc": [],
           "random_programs": {}, "format_pmeasure": {}, "qft": {}, "noise": [],
           "kernel_streams": [], "c1": {}}
    arrays = {}

    # ---------------- parser -----------------
    for name, text in SMALL_PROGRAMS.items():
        out["programs"][name] = program_record(text)

    def outcome(text):
        try:
            prog = qprog.parse_program(text)
        except qerr.SimulatorError as exc:
            return {"stage": "parse", "error": type(exc).__name__, "line": exc.line,
                    "render": exc.render(), "exit_code": exc.exit_code}
        try:
            qsv.run_full(prog, np.random.default_rng(0))
        except qerr.SimulatorError as exc:
            return {"stage": "run", "error": type(exc).__name__, "line": exc.line,
                    "render": exc.render(), "exit_code": exc.exit_code}
        return {"stage": "ok"}

    for path in ERROR_CORPUS:
        text = path.read_text()
        out["errors"][path.stem] = {"text": text, **outcome(text)}
    for name, text in EXTRA_ERRORS.items():
        out["errors"][name] = {"text": text, **outcome(text)}

    for e in ANGLE_EXPRS:
        out["angles"][e] = qprog.eval_angle(e)
    for e in BAD_ANGLES:
        try:
            qprog.eval_angle(e)
            out["angles"][e] = "ok?"
        except qerr.MalformedAngle:
            out["angles"][e] = "MalformedAngle"
    for lit in COMPLEX_LITS:
        out["complex"][lit] = cplx(qprog.parse_complex_literal(lit))

    # ---------------- rqc generator (reference 4-pattern) -----------------
    for rows, cols, depth, seed in RQC_CONFIGS:
        text = qrqc.generate_rqc(qrqc.RqcConfig(rows, cols, depth, seed))
        out["rqc"].append({"rows": rows, "cols": cols, "depth": depth, "seed": seed,
                           "text": text})
    text = qrqc.generate_rqc(qrqc.RqcConfig(3, 3, 10, 2, pmeasure=(0, 1)))
    out["rqc"].append({"rows": 3, "cols": 3, "depth": 10, "seed": 2, "pmeasure": [0, 1],
                       "text": text})

    # ---------------- run_full end states -----------------
    run_inputs = dict(SMALL_PROGRAMS)
    rng = np.random.default_rng(20261020)
    for idx in range(12):
        n = int(rng.integers(3, 11))
        text = random_program_text(rng, n, int(rng.integers(20, 70)))
        run_inputs[f"random{idx}"] = text
        out["random_programs"][f"random{idx}"] = program_record(text)
    for rows, cols, depth, seed in [(2, 3, 8, 42), (3, 4, 12, 9), (3, 3, 10, 0), (2, 5, 16, 5)]:
        run_inputs[f"rqc_{rows}x{cols}_{depth}_{seed}"] = qrqc.generate_rqc(
            qrqc.RqcConfig(rows, cols, depth, seed))

    out["runs"] = {}
    for name, text in run_inputs.items():
        prog = qprog.parse_program(text)
        seed = 123
        res = qsv.run_full(prog, np.random.default_rng(seed))
        key = f"run/{name}"
        arrays[key] = res.state.amplitudes.copy()
        rec = {"seed": seed, "cregs": list(res.cregs), "tables": []}
        for t_i, (qubits, table) in enumerate(res.tables):
            arrays[f"{key}/table{t_i}"] = table.copy()
            rec["tables"].append(list(qubits))
        out["runs"][name] = rec
        # worker / chunk invariance of the reference itself
        with WorkerPool(4) as pool:
            res4 = qsv.run_full(prog, np.random.default_rng(seed), pool=pool, chunk_log2=0)
        assert np.array_equal(res4.state.amplitudes, res.state.amplitudes), name

    # golden table text (cli.format_pmeasure)
    res = qsv.run_full(qprog.parse_program(GOLDEN_TEXT))
    out["format_pmeasure"]["golden"] = format_pmeasure(res.tables[0][1])
    for name in ("ghz", "measure_seq", "bell_measure"):
        r = qsv.run_full(qprog.parse_program(SMALL_PROGRAMS[name]), np.random.default_rng(123))
        out["format_pmeasure"][name] = format_pmeasure(r.tables[0][1])

    # ---------------- kernel-API random streams (test_statevector.py:218-250 shape) ------
    rng = np.random.default_rng(2024)

    def random_state(n):
        v = rng.standard_normal(1 << n) + 1j * rng.standard_normal(1 << n)
        return v / np.linalg.norm(v)

    def random_unitary(dim):
        z = rng.standard_normal((dim, dim)) + 1j * rng.standard_normal((dim, dim))
        q, r = np.linalg.qr(z)
        return q * (np.diag(r) / np.abs(np.diag(r)))

    for s_idx in range(40):
        n = int(rng.integers(2, 11))
        psi = random_state(n)
        cl = int(rng.integers(0, n + 1))
        st = qsv.StateVector(n, psi.copy(), cl)
        ops = []
        for g in range(int(rng.integers(5, 25))):
            kind = int(rng.integers(0, 5))
            if kind == 0:
                u = random_unitary(2)
                k = int(rng.integers(0, n))
                qsv.apply_single_qubit(st, u, k)
                ops.append({"kind": "single", "targets": [k], "controls": []})
            elif kind == 1 and n >= 2:
                u = random_unitary(2)
                qs = rng.permutation(n)
                n_ctrl = int(rng.integers(1, min(3, n)))
                controls = [int(q) for q in qs[:n_ctrl]]
                k = int(qs[n_ctrl])
                qsv.apply_controlled(st, u, controls, k)
                ops.append({"kind": "controlled", "targets": [k], "controls": controls})
            elif kind == 2 and n >= 2:
                u = random_unitary(4)
                qs = rng.permutation(n)
                hi, lo = int(qs[0]), int(qs[1])
                ctrl = [int(q) for q in qs[2:2 + int(rng.integers(0, min(2, n - 2) + 1))]]
                qsv.apply_two_qubit(st, u, hi, lo, controls=tuple(ctrl))
                ops.append({"kind": "two", "targets": [hi, lo], "controls": ctrl})
            elif kind == 3:
                ph = np.exp(1j * rng.uniform(-math.pi, math.pi, size=2))
                u = np.diag(ph)
                k = int(rng.integers(0, n))
                qs = [q for q in range(n) if q != k]
                ctrl = [int(q) for q in rng.choice(qs, size=int(rng.integers(0, min(2, len(qs)) + 1)), replace=False)] if qs else []
                qsv.apply_controlled(st, u, ctrl, k)
                ops.append({"kind": "controlled" if ctrl else "single", "targets": [k], "controls": ctrl})
            else:
                u = np.diag([1.0, 0.0]).astype(complex) if rng.random() < 0.5 else np.diag([0.0, 1.0]).astype(complex)
                k = int(rng.integers(0, n))
                if rng.random() < 0.7:
                    # skip projectors most of the time so the state keeps norm
                    u = random_unitary(2)
                    qsv.apply_single_qubit(st, u, k)
                    ops.append({"kind": "single", "targets": [k], "controls": []})
                else:
                    qsv.apply_projector(st, u, k)
                    ops.append({"kind": "projector", "targets": [k], "controls": []})
            arrays[f"stream{s_idx}/u{len(ops) - 1}"] = np.asarray(u, dtype=np.complex128)
        arrays[f"stream{s_idx}/psi0"] = psi
        arrays[f"stream{s_idx}/final"] = st.amplitudes.copy()
        out["kernel_streams"].append({"n": n, "chunk_log2": cl, "ops": ops})

    # ---------------- QFT on a random state (apply_instruction loop) ---------------
    for n in (3, 6, 9):
        lines = qft_text(n)
        fwd = "\n".join(lines) + "\n"
        rt = "\n".join(lines + ["DAGGER"] + lines[1:] + ["ENDDAGGER"]) + "\n"
        g = np.random.default_rng(n)
        psi = g.standard_normal(1 << n) + 1j * g.standard_normal(1 << n)
        psi /= np.linalg.norm(psi)
        out["qft"][str(n)] = {"forward": fwd, "round_trip": rt}
        for tag, text in (("forward", fwd), ("round_trip", rt)):
            prog = qprog.parse_program(text)
            st = qsv.StateVector(n, psi.copy(), qsv.default_chunk_log2(n))
            for inst in prog.instructions:
                qsv.apply_instruction(st, inst)
            arrays[f"qft{n}/{tag}"] = st.amplitudes.copy()
        arrays[f"qft{n}/psi0"] = psi

    # ---------------- noisy trajectories (reference semantics) ----------------------
    for rows, cols, depth, seed, p, traj_seed in [(2, 3, 8, 42, 0.3, 5), (2, 3, 8, 42, 0.1, 11),
                                                  (2, 3, 8, 42, 1e-3, 7), (3, 3, 6, 1, 0.05, 3),
                                                  (2, 4, 6, 9, 0.2, 17)]:
        text = qrqc.generate_rqc(qrqc.RqcConfig(rows, cols, depth, seed))
        prog = qprog.parse_program(text)
        model = qnoise.make_noise_model("depolarizing", p)
        choices = []
        orig = qnoise.sample_noisy_gate

        def spy(*a, **k):
            c = orig(*a, **k)
            choices.append(int(c))
            return c

        qnoise.sample_noisy_gate = spy
        try:
            res = qsv.run_full(prog, np.random.default_rng(traj_seed), model)
        finally:
            qnoise.sample_noisy_gate = orig
        key = f"noise/{rows}x{cols}_{depth}_{seed}_{p}_{traj_seed}"
        arrays[key] = res.state.amplitudes.copy()
        out["noise"].append({"rows": rows, "cols": cols, "depth": depth, "seed": seed,
                             "p": p, "traj_seed": traj_seed, "text": text,
                             "choices": choices, "key": key})

    # ---------------- QSVDUMP image ------------------
    st = qsv.StateVector(3, arrays["run/ghz"].copy(), 1)
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "s.qsv"
        save_state(st, path)
        arrays["qsvdump/ghz_bytes"] = np.frombuffer(path.read_bytes(), dtype=np.uint8).copy()

    # ---------------- C1 (20 qubits, BASELINE 8-pattern generator) ---------------
    from paper_2008_07140_b200 import workloads

    c1_text = workloads.rqc_text(4, 5, 20, seed=0)
    prog = qprog.parse_program(c1_text)
    with WorkerPool(8) as pool:
        res = qsv.run_full(prog, pool=pool)
    amps = res.state.amplitudes
    idx = np.unique(np.concatenate([
        np.arange(64), np.arange(amps.size - 64, amps.size),
        np.random.default_rng(1).integers(0, amps.size, size=2048)]))
    arrays["c1/idx"] = idx.astype(np.int64)
    arrays["c1/amps"] = amps[idx].copy()
    arrays["c1/pm_0_7_13_19"] = qsv.pmeasure(res.state, (0, 7, 13, 19))
    arrays["c1/probs_sum_by_q0"] = np.array([qsv.probability_bit0(res.state, q) for q in range(20)])
    out["c1"] = {"text": c1_text, "norm_sq": res.state.norm_sq(),
                 "gate_count": len(prog.gate_instructions())}

    (HERE / "programs.json").write_text(json.dumps(out, indent=1, sort_keys=True))
    buf = io.BytesIO()
    np.savez_compressed(buf, **arrays)
    (HERE / "states.npz").write_bytes(buf.getvalue())
    print("wrote", len(arrays), "arrays;", (HERE / "states.npz").stat().st_size, "bytes")


if __name__ == "__main__":
    main()
