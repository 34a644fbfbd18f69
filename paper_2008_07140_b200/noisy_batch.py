"""Batched noisy trajectories for any Kraus channel.

Per trajectory the semantics are exactly the reference's
`run_full(program, rng_t, noise_model)` (statevector.py:343-430,
noise.py:188-222): before each noisy gate the branch weights ||K_i psi||^2
come from the current state, ONE `rng_t.random()` draw picks the branch, the
gate U.K_c is applied and the state renormalised when its norm left 1;
MEASURE draws against p0 and collapses; PMEASURE records a table.  State-
dependent channels (ampdamp, phasedamp) are therefore supported, not only the
pre-sampled Pauli case of `trajectories.py`.

B200 layout: the B = 2^b trajectories are consecutive 2^n-amplitude blocks of
batched device states (two groups of B/2, each an (n + b - 1)-qubit state on
its own stream).  Gates without noise are identical for every trajectory and
run through the fused scheduler over a whole group (`qsv_run`, trajectories
as extra top qubits).  A noisy gate or MEASURE is one
`qsv_noisy_batch_step` launch: every trajectory's own matrix
U.K_c(t)/sqrt(p) is applied and, in the same pass, every trajectory's
reduced density of the NEXT noisy gate's qubits is reduced — the weights that
gate needs — so a run of noisy gates costs one HBM pass + one small D2H each
(the reference: #Kraus + 2 passes per noisy gate per trajectory).  Steps are
enqueued asynchronously (`qsv_noisy_batch_step_async` / `_wait`), so one
group's host sampling overlaps the other group's pass.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from . import gates
from .errors import DegenerateBranch, DegenerateState, UnsupportedGate
from .program import Program

_SLOTS = 16  # complex128 slots per trajectory (row-major 4x4) in the step's matrix / rdm buffers


@dataclass
class NoisyBatchResult:
    """Per-trajectory `RunResult` analogue: cregs[t], tables[t] (list of
    (qubits, table)) and the batched device `states` (trajectory t's amplitudes
    are `amplitudes(t)`)."""

    cregs: list
    tables: list
    choices: list  # per trajectory: Kraus branch index per noisy gate (diagnostic)
    state: object = None
    qubit_count: int = 0
    stats: dict = field(default_factory=dict)

    states: list = field(default_factory=list)  # one batched state per group
    group_log2: int = 0  # trajectories per group = 2^group_log2

    def amplitudes(self, t: int) -> np.ndarray:
        if not self.states:
            raise ValueError("no device states kept (chunked or closed batch)")
        out = np.empty(1 << self.qubit_count, dtype=np.complex128)
        g, k = divmod(t, 1 << self.group_log2)
        return self.states[g].download(out, k << self.qubit_count)

    def close(self) -> None:
        for st in self.states:
            st.close()
        self.states = []
        self.state = None


def _step_info(inst, noise):
    """('noisy', dense base with controls embedded, qubits MSB-first, (K, K^dag K)) for a noisy
    gate; ('measure', None, (q,), None); None for everything else."""
    if inst.name == "MEASURE":
        return "measure", None, (inst.qubits[0],), None
    if not inst.is_gate:
        return None
    base, targets, controls = gates.controlled_form(inst)
    qubits = tuple(controls) + tuple(targets)
    if len(qubits) > 2:
        return None
    kraus = noise.kraus_for(inst, len(qubits))
    if kraus is None:
        return None
    K = np.asarray(kraus)
    unitary = inst.name not in ("P0", "P1")
    return "noisy", gates.embed_controls(base, len(controls)), qubits, (K, np.einsum("kji,kjl->kil", K.conj(), K),
                                                                         unitary)


class _Group:
    """Trajectories [lo, lo + 2^bg) in one batched device state on its own stream."""

    def __init__(self, state, lo: int, bg: int):
        self.state, self.lo, self.bg = state, lo, bg
        self.B = 1 << bg
        self.mats = np.zeros((self.B, _SLOTS), dtype=np.complex128)
        self.rdm = np.zeros((self.B, _SLOTS), dtype=np.complex128)
        self.pending: tuple | None = None  # qubits whose rdm the in-flight / last step reduces
        self.inflight = False

    def launch(self, gate_qubits, next_qubits) -> None:
        gq = (C.c_int32 * 2)(*(list(gate_qubits) + [0, 0])[:2])
        nq = (C.c_int32 * 2)(*(list(next_qubits) + [0, 0])[:2])
        N.check(N.lib().qsv_noisy_batch_step_async(self.state.handle, self.bg, len(gate_qubits), gq,
                                                   self.mats.ctypes.data, len(next_qubits), nq))
        self.inflight = True
        self.pending = tuple(next_qubits) if next_qubits else None

    def wait(self) -> None:
        if self.inflight:
            N.check(N.lib().qsv_noisy_batch_wait(self.state.handle, self.bg, self.rdm.ctypes.data))
            self.inflight = False


DEFAULT_MAX_BATCH_BYTES = 96 << 30  # device memory one batch of trajectory states may take


def run_noisy_batch(program: Program, noise, rngs, *, device: int = 0, max_qubits: int = 30,
                    fuse: bool = True, groups: int = 2,
                    max_batch_bytes: int = DEFAULT_MAX_BATCH_BYTES) -> NoisyBatchResult:
    """Run len(rngs) = 2^b trajectories of `program` under `noise`.

    When 2^b trajectory states exceed `max_batch_bytes` they run in consecutive
    power-of-two chunks; the result then carries cregs, tables and choices for
    every trajectory but no device states (each chunk's states are freed once its
    tables are read), so `amplitudes(t)` is unavailable.

    rngs[t] plays the role of the `rng` argument of the reference `run_full` for
    trajectory t (e.g. `np.random.default_rng(seed_t)`); draws happen in program
    order, one per noisy gate and per MEASURE, as in the reference.  The batch is
    split into `groups` (1 or 2) batched states on their own streams: while one
    group's pass runs, the host samples the other group's branches."""
    B = len(rngs)
    if B < 1 or B & (B - 1):
        raise ValueError("the batch holds a power-of-two number of trajectories")
    per = 16 << program.qubit_count
    if B > 1 and B * per > max_batch_bytes:
        chunk = 1 << max(0, (max(1, max_batch_bytes // per)).bit_length() - 1)
        out = NoisyBatchResult(cregs=[], tables=[], choices=[], qubit_count=program.qubit_count)
        out.stats = {"noisy_steps": 0, "trajectories": B, "chunks": B // chunk}
        for c0 in range(0, B, chunk):
            part = _run_noisy_batch(program, noise, rngs[c0:c0 + chunk], device=device, max_qubits=max_qubits,
                                    fuse=fuse, groups=groups)
            part.close()
            out.cregs += part.cregs
            out.tables += part.tables
            out.choices += part.choices
            out.stats["noisy_steps"] += part.stats["noisy_steps"]
        return out
    return _run_noisy_batch(program, noise, rngs, device=device, max_qubits=max_qubits, fuse=fuse, groups=groups)


def _run_noisy_batch(program: Program, noise, rngs, *, device: int, max_qubits: int, fuse: bool,
                     groups: int) -> NoisyBatchResult:
    from .statevector import init_state

    B = len(rngs)
    b = B.bit_length() - 1
    n = program.qubit_count
    if n > max_qubits:
        from .errors import TooManyQubits

        raise TooManyQubits(f"{n} qubits exceed the limit of {max_qubits}")
    G = 2 if (groups >= 2 and B >= 2) else 1
    bg = b - (G - 1)
    L = N.lib()
    grps = []
    try:
        for g in range(G):
            st = init_state(n + bg, max_qubits=n + bg, device=device)
            grps.append(_Group(st, g << bg, bg))
            st.set_basis(0)
            # every trajectory block starts at |0..0>: amplitude 1 at t << n (one strided copy)
            starts = np.ones(1 << bg, dtype=np.complex128)
            N.check(L.qsv_upload_strided(st.handle, starts.ctypes.data, 0, 1 << bg, 1 << n))
    except Exception:
        for gr in grps:
            gr.state.close()
        raise
    res = NoisyBatchResult(cregs=[[0] * program.creg_count for _ in range(B)], tables=[[] for _ in range(B)],
                           choices=[[] for _ in range(B)], state=grps[0].state, qubit_count=n)
    res.states = [gr.state for gr in grps]
    res.group_log2 = bg
    opts = N.options(fuse=fuse)
    insts = list(program.instructions)
    if noise is not None:
        info = [_step_info(i, noise) for i in insts]
    else:
        info = [("measure", None, (i.qubits[0],), None) if i.name == "MEASURE" else None for i in insts]
    # each trajectory draws exactly once per noisy gate / MEASURE, in program order, so its
    # whole stream is drawn up front: rng.random(k) yields the same doubles as k scalar calls
    n_draws = sum(1 for x in info if x is not None)
    uniforms = np.stack([g.random(n_draws) for g in rngs]) if n_draws else None
    draw = 0
    choices: list = []  # per noisy gate: the B branch indices
    batch: list = []
    steps = 0

    def flush():
        if batch:
            from .statevector import compile_gates

            rec = compile_gates(batch)
            for gr in grps:
                stt = N.qsv_run_stats()
                N.check(L.qsv_run(gr.state.handle, rec.ctypes.data, len(rec), C.byref(opts), C.byref(stt)))
                gr.pending = None
            batch.clear()

    def next_need(pos):
        """Qubits whose rdm the instruction after `pos` needs, if it is noisy / MEASURE."""
        if pos + 1 < len(insts) and info[pos + 1] is not None:
            return info[pos + 1][2]
        return ()

    for pos, inst in enumerate(insts):
        kind = info[pos]
        if kind is None:
            if inst.name == "PMEASURE":
                flush()
                for gr in grps:
                    qs = [n + j for j in range(bg - 1, -1, -1)] + list(inst.qubits)
                    if len(qs) > 30:
                        raise UnsupportedGate("PMEASURE table too large for the batch", inst.line)
                    arr = (C.c_int32 * len(qs))(*qs)
                    table = np.zeros(1 << len(qs), dtype=np.float64)
                    N.check(L.qsv_pmeasure(gr.state.handle, arr, len(qs), table.ctypes.data))
                    per = table.reshape(gr.B, -1)
                    for t in range(gr.B):
                        res.tables[gr.lo + t].append((tuple(inst.qubits), per[t].copy()))
            else:
                batch.append(inst)
            continue
        flush()
        what, u, qubits, kraus = kind
        D = 1 << len(qubits)
        nxt = next_need(pos)
        step_choice = []
        for gr in grps:
            if gr.pending != tuple(qubits):
                gr.launch((), qubits)  # weights of this step's qubits
                steps += 1
            gr.wait()
            Bg, U = gr.B, uniforms[gr.lo:gr.lo + gr.B, draw]
            up = gr.rdm.reshape(Bg, 4, 4)[:, :D, :D]  # the kernel returns the upper triangle
            rhos = np.triu(up) + np.conj(np.swapaxes(np.triu(up, 1), 1, 2))  # (rho is Hermitian)
            gr.mats[:] = 0
            if what == "measure":
                for t in range(Bg):
                    p0 = float(rhos[t, 0, 0].real)
                    p1 = float(rhos[t, 1, 1].real)
                    if p0 < 1e-12 and p1 < 1e-12:
                        raise DegenerateState("measurement of a (numerically) zero state")
                    outcome = 0 if U[t] < p0 else 1
                    res.cregs[gr.lo + t][inst.creg] = outcome
                    gr.mats[t, 3 * outcome] = 1.0 / math.sqrt(p0 if outcome == 0 else p1)
            else:
                K, KdK, unitary = kraus
                # ||K_i psi_t||^2 = tr(K_i^dag K_i rho_t) for all trajectories and branches at once
                probs = np.einsum("klj,bjl->bk", KdK, rhos).real
                total = probs.sum(axis=1)
                if (total < 1e-12).any():
                    raise DegenerateBranch("all Kraus branches have ~zero probability")
                r = U * total
                cum = np.cumsum(probs, axis=1)  # the reference's running `acc += p` (noise.py:206-212)
                hit = r[:, None] < cum
                choice = np.where(hit.any(axis=1), hit.argmax(axis=1), len(K) - 1)
                pc = probs[np.arange(Bg), choice]
                m = np.einsum("ij,bjk->bik", u, K[choice])
                # the reference renormalises by the post-apply norm when it left 1
                # (noise.py:219-221); for a normalised state and a unitary gate that norm is
                # probs[choice]; for a noisy projector it is tr(M^dag M rho)
                if not unitary:
                    pc = np.einsum("bji,bjk,bki->b", m.conj(), m, rhos).real
                renorm = np.abs(pc - 1.0) > 1e-12
                m[renorm] /= np.sqrt(pc[renorm])[:, None, None]
                gr.mats[:, : D * D] = m.reshape(Bg, -1)
                step_choice.append(choice)
            gr.launch(qubits, nxt)
            steps += 1
        if step_choice:
            choices.append(np.concatenate(step_choice))
        draw += 1
    flush()
    for gr in grps:
        gr.wait()
        gr.state.synchronize()
    if choices:
        res.choices = np.stack(choices, axis=1).tolist()
    res.stats = {"noisy_steps": steps, "trajectories": B, "groups": G}
    return res
