"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is involved; every input is generated
here from a recorded seed and emitted as .qprog text in the reference
grammar, so the oracle and the GPU engine consume the identical gate stream.

* C1/C2/C3 - eight-pattern no-repeat grid RQC (`rqc.py`, patterns=8)
* C4       - little-endian QFT (H + CR "pi/2^k" + reversal SWAPs) on an
             i.i.d. complex Gaussian state, inverse via DAGGER
* C5       - depolarising trajectories: Pauli errors pre-sampled on the host
             with the reference's exact draw rule (`noise.py:188-222`) and
             inserted as explicit X/Y/Z gates BEFORE the noisy gate (the
             reference applies U.K_i, `noise.py:214`).
"""

from __future__ import annotations

import math

import numpy as np

from .rqc import RqcConfig, generate_rqc

C2_SHAPE = (5, 6, 24)   # n=30, 24 cycles
C1_SHAPE = (4, 5, 20)   # n=20, 20 cycles
C5_SHAPE = (4, 6, 20)   # n=24, 20 cycles


def grid_shape(n: int) -> tuple[int, int]:
    """Grid of an n-qubit RQC: the most square full rectangle rows x cols = n
    (rows <= cols) when its aspect ratio is at most 2 (30 -> 5x6, 32 -> 4x8,
    35 -> 5x7), else ceil(sqrt(n)) columns with a partial last row
    (31 -> 6x6 holding 31, 33 -> 6x6 holding 33, 34 -> 6x6 holding 34;
    SURVEY.md Appendix C.4)."""
    best = (1, n)
    for r in range(1, int(math.isqrt(n)) + 1):
        if n % r == 0:
            best = (r, n // r)
    if best[1] <= 2 * best[0] or n < 4:
        return best
    c = math.isqrt(n - 1) + 1
    return (-(-n // c), c)


def rqc_text(rows: int, cols: int, depth: int, seed: int = 0, pmeasure=(), qubits: int = 0) -> str:
    """BASELINE RQC: 8 cycled CZ patterns, no repeated pool gate per qubit."""
    return generate_rqc(RqcConfig(rows, cols, depth, seed, pmeasure=tuple(pmeasure),
                                  patterns=8, no_repeat=True, qubits=qubits))


def rqc_for_qubits(n: int, depth: int = 24, seed: int = 0) -> str:
    r, c = grid_shape(n)
    return rqc_text(r, c, depth, seed, qubits=n if r * c != n else 0)


def qft_lines(n: int) -> list[str]:
    """QFT body: for j = n-1..0: H j; CR i,j,"pi/2^(j-i)" for i = j-1..0; swaps."""
    body = []
    for j in range(n - 1, -1, -1):
        body.append(f"H {j}")
        for i in range(j - 1, -1, -1):
            body.append(f'CR {i},{j},"pi/{2 ** (j - i)}"')
    body += [f"SWAP {q},{n - 1 - q}" for q in range(n // 2)]
    return body


def qft_text(n: int, round_trip: bool = False) -> str:
    body = qft_lines(n)
    lines = [f"QINIT {n}"] + body
    if round_trip:
        lines += ["DAGGER"] + body + ["ENDDAGGER"]
    return "\n".join(lines) + "\n"


def gaussian_state(n: int, seed: int = 0, chunk: int = 1 << 24) -> np.ndarray:
    """i.i.d. complex Gaussian amplitudes, unit norm (tests/helpers.py:50-52 recipe:
    all real parts are drawn first, then all imaginary parts)."""
    size = 1 << n
    rng = np.random.default_rng(seed)
    out = np.empty(size, dtype=np.complex128)
    view = out.view(np.float64).reshape(size, 2)
    for part in (0, 1):
        for s in range(0, size, chunk):
            e = min(size, s + chunk)
            view[s:e, part] = rng.standard_normal(e - s)
    # pairwise (numpy) sum of squares per chunk, chunks added exactly (fsum): no
    # state-sized temporary at n = 30 (a single chunk below 2^24 amplitudes)
    big = 1 << 26
    norm = math.sqrt(math.fsum(float(np.sum(view[s:s + big] * view[s:s + big], dtype=np.float64))
                               for s in range(0, size, big)))
    for s in range(0, size, big):
        out[s:s + big] /= norm
    return out


def mirror_text(text: str) -> str:
    """C followed by DAGGER C ENDDAGGER (program.py:328-333): the identity circuit
    used as a size-independent known answer (|0..0> -> |0..0>)."""
    lines = [ln for ln in text.splitlines() if ln.strip() and not ln.lstrip().startswith("%")]
    head, body = lines[0], lines[1:]
    if not head.startswith("QINIT"):
        raise ValueError("mirror_text: program must start with QINIT")
    return "\n".join([head] + body + ["DAGGER"] + body + ["ENDDAGGER"]) + "\n"


# --------------------------------------------------------------------------
# C5: depolarising trajectories as explicit Pauli insertions
# --------------------------------------------------------------------------

_PAULI = ("I", "X", "Y", "Z")


def _depolarizing_weights(p: float) -> list[float]:
    """||K_i psi||^2 / ||psi||^2 for the depolarising Kraus set (noise.py:56-63)."""
    c = [math.sqrt(1.0 - 0.75 * p)] + [0.5 * math.sqrt(p)] * 3
    return [x * x for x in c]


_DRAW_PLANS: dict = {}


def _draw_plan(program):
    """Per program (cached): for every random draw of a trajectory, the
    instruction index and its qubits (controls + targets), None for MEASURE."""
    key = id(program)
    hit = _DRAW_PLANS.get(key)
    if hit is not None and hit[0] is program:
        return hit[1]
    from . import gates

    plan = []
    for idx, inst in enumerate(program.instructions):
        if inst.name == "MEASURE":
            plan.append((idx, None))
            continue
        if not inst.is_gate:
            continue
        _, targets, controls = gates.controlled_form(inst)
        qubits = tuple(controls) + tuple(targets)
        if len(qubits) <= 2:
            plan.append((idx, qubits))
    if len(_DRAW_PLANS) > 64:
        _DRAW_PLANS.clear()
    _DRAW_PLANS[key] = (program, plan)
    return plan


def sample_pauli_insertions(program, p: float, seed: int):
    """Replay the reference trajectory draw rule on the host.

    For each <=2-qubit gate in program order the reference draws one
    `rng.random() * sum(probs)` and picks the first branch whose cumulative
    weight exceeds it (`noise.py:202-213`); 2-qubit gates use the Kronecker
    set K_a (x) M_b with index a*4+b, K_a acting on the first qubit of
    controls+targets (`noise.py:77-79`, `statevector.py:347-356`).  MEASURE
    consumes one draw too (`statevector.py:304`).  Returns {instruction index:
    [(qubit, pauli), ...]} for non-identity branches.  All draws of a
    trajectory come from one `rng.random(k)` call (the same stream as k
    scalar calls); the cumulative weights are summed left to right as the
    reference loop does.
    """
    w1 = _depolarizing_weights(p)
    w2 = [a * b for a in w1 for b in w1]
    plan = _draw_plan(program)
    draws = np.random.default_rng(seed).random(len(plan))
    out = {}
    for w, nq in ((w1, 1), (w2, 2)):
        acc, run = [], 0.0
        for wi in w:
            run += wi
            acc.append(run)
        sel = [k for k, (_, qs) in enumerate(plan) if qs is not None and len(qs) == nq]
        if not sel:
            continue
        r = draws[sel] * sum(w)
        # first branch with r < acc[i] (the last one if none)
        choice = np.minimum(np.searchsorted(np.asarray(acc), r, side="right"), len(w) - 1)
        for k in np.nonzero(choice)[0]:
            idx, qs = plan[sel[k]]
            c = int(choice[k])
            picks = [(qs[0], _PAULI[c])] if nq == 1 else [(qs[0], _PAULI[c // 4]), (qs[1], _PAULI[c % 4])]
            picks = [(q, g) for q, g in picks if g != "I"]
            if picks:
                out[idx] = picks
    return dict(sorted(out.items()))


def noisy_trajectory_program(program, p: float, seed: int):
    """The program with the sampled Paulis inserted before their gates."""
    from .program import Instruction, Program

    ins = sample_pauli_insertions(program, p, seed)
    insts = []
    for idx, inst in enumerate(program.instructions):
        insts += [Instruction(g, (q,), line=inst.line) for q, g in ins.get(idx, ())]
        insts.append(inst)
    return Program(program.qubit_count, program.creg_count, tuple(insts))


def noisy_trajectory_text(program, p: float, seed: int) -> str:
    from .program import to_script

    return to_script(noisy_trajectory_program(program, p, seed))


def trajectory_seed(base_seed: int, t: int) -> int:
    return base_seed * 1_000_003 + t
