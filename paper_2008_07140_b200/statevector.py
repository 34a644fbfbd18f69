"""Full-amplitude engine: the reference API, executed by libqsv on a B200.

Drop-in mirror of `qcsim/statevector.py` (statevector.py:27-430): the same
names, arguments and error classes, with the amplitudes resident in HBM.

* `StateVector` owns a device buffer of 2^n complex128 amplitudes.
  `.amplitudes` downloads a host copy (numpy) and assigning to it uploads;
  `chunk_log2` is kept for signature compatibility (the GPU layout does not
  use chunks).
* `apply_single_qubit / apply_controlled / apply_two_qubit / apply_projector`
  launch one unfused gate kernel each (the reference kernel API,
  statevector.py:255-289).
* `run_full` hands maximal runs of gates to the native scheduler, which fuses
  them into a few HBM passes (`qsv_run`); MEASURE, PMEASURE and noisy gates
  are executed between runs with the reference's RNG semantics.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from . import gates
from .errors import DegenerateBranch, DegenerateState, TooManyQubits, UnsupportedGate
from .program import Instruction, Program

DEFAULT_MAX_QUBITS = 30


def default_chunk_log2(n: int, workers: int = 1) -> int:
    """Reference chunk sizing (statevector.py:46-49); informational on the GPU."""
    want = max(4, 4 * max(1, workers))
    return max(0, n - (max(1, want - 1).bit_length()))


class StateVector:
    """2^n complex128 amplitudes in device memory (reference statevector.py:32-43)."""

    def __init__(self, qubit_count: int, amplitudes=None, chunk_log2: int | None = None, *,
                 device: int = 0, stream=None, _handle=None):
        self.qubit_count = int(qubit_count)
        self.chunk_log2 = default_chunk_log2(self.qubit_count) if chunk_log2 is None else chunk_log2
        self.device = device
        L = N.lib()
        if _handle is None:
            h = C.c_void_p()
            N.check(L.qsv_create(self.qubit_count, device,
                                 C.c_void_p(-1 if stream is None else stream), C.byref(h)))
            _handle = h
        self._h = _handle
        if amplitudes is not None:
            self.amplitudes = amplitudes

    # -- lifetime ---------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            N.lib().qsv_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def device_ptr(self) -> int:
        p = C.c_void_p()
        N.check(N.lib().qsv_device_ptr(self._h, C.byref(p)), self._h)
        return p.value

    @property
    def chunk_count(self) -> int:
        return 1 << (self.qubit_count - self.chunk_log2)

    # -- data movement ----------------------------------------------------
    @property
    def amplitudes(self) -> np.ndarray:
        out = np.empty(1 << self.qubit_count, dtype=np.complex128)
        self.download(out)
        return out

    @amplitudes.setter
    def amplitudes(self, values) -> None:
        values = np.ascontiguousarray(values, dtype=np.complex128)
        if values.size != 1 << self.qubit_count:
            raise ValueError(f"expected {1 << self.qubit_count} amplitudes, got {values.size}")
        N.check(N.lib().qsv_upload(self._h, values.ctypes.data, 0, values.size), self._h)

    def download(self, out: np.ndarray, offset: int = 0) -> np.ndarray:
        assert out.dtype == np.complex128 and out.flags.c_contiguous
        N.check(N.lib().qsv_download(self._h, out.ctypes.data, offset, out.size), self._h)
        return out

    def set_basis(self, index: int) -> None:
        N.check(N.lib().qsv_set_basis(self._h, int(index)), self._h)

    def synchronize(self) -> None:
        N.check(N.lib().qsv_synchronize(self._h), self._h)

    # -- readout ------------------------------------------------------------
    def norm_sq(self) -> float:
        out = C.c_double()
        N.check(N.lib().qsv_norm_sq(self._h, C.byref(out)), self._h)
        return out.value

    def inner(self, other: "StateVector") -> complex:
        """<self|other> computed on the device."""
        re, im = C.c_double(), C.c_double()
        N.check(N.lib().qsv_inner(self._h, C.c_void_p(other.device_ptr), C.byref(re), C.byref(im)), self._h)
        return complex(re.value, im.value)

    def max_abs_diff(self, other: "StateVector") -> float:
        out = C.c_double()
        N.check(N.lib().qsv_max_abs_diff(self._h, C.c_void_p(other.device_ptr), C.byref(out)), self._h)
        return out.value

    def reduced_density(self, qubits) -> np.ndarray:
        qubits = tuple(int(q) for q in qubits)
        d = 1 << len(qubits)
        out = np.empty((d, d), dtype=np.complex128)
        q = np.asarray(qubits, dtype=np.int32)
        N.check(N.lib().qsv_reduced_density(self._h, len(qubits), q.ctypes.data, out.ctypes.data), self._h)
        return out


def init_state(n: int, *, chunk_log2: int | None = None, max_qubits: int = DEFAULT_MAX_QUBITS,
               device: int = 0, stream=None) -> StateVector:
    """|0...0> on n qubits (statevector.py:52-65); TooManyQubits above the ceiling."""
    if n < 1:
        raise TooManyQubits(f"need at least 1 qubit, got {n}")
    if n > max_qubits:
        raise TooManyQubits(f"{n} qubits exceed the {max_qubits}-qubit memory ceiling")
    if chunk_log2 is None:
        chunk_log2 = default_chunk_log2(n)
    return StateVector(n, None, min(max(chunk_log2, 0), n), device=device, stream=stream)


# --------------------------------------------------------------------------
# kernel API (one gate, one launch)
# --------------------------------------------------------------------------


def _apply_gate(state: StateVector, u, targets, controls=()) -> None:
    rec = N.gate_records([(np.asarray(u, dtype=np.complex128), tuple(targets), tuple(controls))])
    N.check(N.lib().qsv_apply_gate(state.handle, rec.ctypes.data), state.handle)


def apply_single_qubit(state, u, k, pool=None) -> None:
    """(a_i, a_{i+2^k}) <- U (a_i, a_{i+2^k}) for every index with bit k = 0."""
    _apply_gate(state, u, (k,))


def apply_controlled(state, u, controls, k, pool=None) -> None:
    """Pair update on indices whose control bits are all 1; others untouched."""
    _apply_gate(state, u, (k,), tuple(controls))


def apply_two_qubit(state, u, q_hi, q_lo, pool=None, controls=()) -> None:
    """4x4 update; q_hi indexes the high matrix bit, q_lo the low one."""
    _apply_gate(state, u, (q_hi, q_lo), tuple(controls))


def apply_projector(state, p, k, pool=None) -> None:
    """Non-unitary diagonal update (no renormalisation)."""
    _apply_gate(state, p, (k,))


# --------------------------------------------------------------------------
# readout (statevector.py:292-328)
# --------------------------------------------------------------------------


def probability_bit0(state: StateVector, k: int) -> float:
    out = C.c_double()
    N.check(N.lib().qsv_prob_bit0(state.handle, int(k), C.byref(out)), state.handle)
    return out.value


def measure(state: StateVector, k: int, rng: np.random.Generator) -> int:
    """Projective measurement: collapse and renormalise (statevector.py:298-308)."""
    p0 = probability_bit0(state, k)
    p1 = state.norm_sq() - p0
    if p0 < 1e-12 and p1 < 1e-12:
        raise DegenerateState(f"both outcomes of qubit {k} have ~zero probability")
    outcome = 0 if rng.random() < p0 else 1
    N.check(N.lib().qsv_collapse(state.handle, int(k), outcome,
                                 1.0 / math.sqrt(p0 if outcome == 0 else p1)))
    return outcome


def pmeasure(state: StateVector, qubits) -> np.ndarray:
    """Probability table over the listed qubits, first listed = MSB; state untouched."""
    q = np.asarray(tuple(qubits), dtype=np.int32)
    table = np.empty(1 << q.size, dtype=np.float64)
    N.check(N.lib().qsv_pmeasure(state.handle, q.ctypes.data, int(q.size), table.ctypes.data), state.handle)
    return table


# --------------------------------------------------------------------------
# program execution
# --------------------------------------------------------------------------


@dataclass
class RunResult:
    cregs: list[int]
    tables: list[tuple[tuple[int, ...], np.ndarray]] = field(default_factory=list)
    state: StateVector | None = None
    stats: dict = field(default_factory=dict)
    amplitudes: np.ndarray | None = None  # host copy (run_batch)


def _gate_triplet(inst):
    base, targets, controls = gates.controlled_form(inst)
    if len(targets) > 2:
        raise UnsupportedGate(f"{inst.name} targets {targets}", inst.line)
    return base, targets, controls


def compile_gates(instructions) -> np.ndarray:
    """Gate instructions -> packed qsv_gate records (controlled form)."""
    return N.gate_records(_gate_triplet(i) for i in instructions)


def _noisy(state, inst, noise, rng) -> bool:
    """Reference trajectory step (statevector.py:343-357, noise.py:188-222).

    Branch weights ||K_i psi||^2 = tr(K_i rho K_i^dag) come from ONE on-device
    reduced-density pass over the gate's qubits; U.K_i / sqrt(p_i) is then
    applied as a single dense gate (renormalisation folded in when the
    reference would renormalise, i.e. |p_i - 1| > 1e-12)."""
    if noise is None:
        return False
    base, targets, controls = gates.controlled_form(inst)
    qubits = tuple(controls) + tuple(targets)
    if len(qubits) > 2:
        return False
    kraus = noise.kraus_for(inst, len(qubits))
    if kraus is None:
        return False
    rho = state.reduced_density(qubits)
    probs = [float(np.real(np.trace(k @ rho @ k.conj().T))) for k in kraus]
    total = sum(probs)
    if total < 1e-12:
        raise DegenerateBranch("all Kraus branches have ~zero probability")
    r = rng.random() * total
    acc, choice = 0.0, len(probs) - 1
    for i, p in enumerate(probs):
        acc += p
        if r < acc:
            choice = i
            break
    noisy = gates.embed_controls(base, len(controls)) @ kraus[choice]
    # post-apply norm (noise.py:219-221): probs[choice] for a unitary gate, tr(M^dag M rho)
    # for a noisy projector
    nsq = probs[choice] if inst.name not in ("P0", "P1") else float(np.real(np.trace(noisy.conj().T @ noisy @ rho)))
    if abs(nsq - 1.0) > 1e-12:
        noisy = noisy / math.sqrt(nsq)
    _apply_gate(state, noisy, qubits)
    return True


def _flush(state, batch, options, stats) -> None:
    if not batch:
        return
    rec = compile_gates(batch)
    st = N.qsv_run_stats()
    N.check(N.lib().qsv_run(state.handle, rec.ctypes.data, len(rec), C.byref(options), C.byref(st)), state.handle)
    for k, v in st.as_dict().items():
        stats[k] = stats.get(k, 0) + v
    batch.clear()


def apply_instruction(state: StateVector, inst: Instruction, pool=None, rng=None, noise=None,
                      result: RunResult | None = None) -> None:
    """Execute one expanded instruction (statevector.py:360-394)."""
    if inst.name == "MEASURE":
        if rng is None:
            raise UnsupportedGate("MEASURE needs a random stream", inst.line)
        bit = measure(state, inst.qubits[0], rng)
        if result is not None:
            result.cregs[inst.creg] = bit
        return
    if inst.name == "PMEASURE":
        table = pmeasure(state, inst.qubits)
        if result is not None:
            result.tables.append((inst.qubits, table))
        return
    if _noisy(state, inst, noise, rng):
        return
    base, targets, controls = _gate_triplet(inst)
    _apply_gate(state, base, targets, controls)


def run_full(program: Program, rng: np.random.Generator | None = None, noise=None, *,
             workers: int = 1, pool=None, chunk_log2: int | None = None,
             max_qubits: int = DEFAULT_MAX_QUBITS, initial_index: int = 0,
             initial_state=None, fuse: bool = True, tile_qubits: int = 0, reg_qubits: int = 0,
             low_qubits: int = 0, jit: int = 0, device: int = 0, stream=None,
             state: StateVector | None = None, profile: bool = False,
             noise_engine: str = "fused") -> RunResult:
    """Run a program on the B200 full-amplitude backend (statevector.py:397-430).

    Extra keywords over the reference: `initial_state` (host amplitudes to
    start from), `fuse`/`tile_qubits`/`reg_qubits`/`low_qubits` (scheduler
    knobs), `device`/`stream`, `state` (reuse an existing device state) and
    `profile` (per-launch CUDA-event timing into `RunResult.stats`), `jit`
    (0: specialised per-pass kernels from n >= 16, 1: always, -1: never) and
    `noise_engine` ("fused": mixed-unitary channels (flips, depolarising) draw their
    branches up front and the run stays fused; other channels run as a batch of one in
    `noisy_batch`, one pass per noisy gate; "sequential": branch weights via
    `qsv_reduced_density`, then the gate, per noisy gate).
    `workers`, `pool` and `chunk_log2` are accepted and ignored.
    """
    n = program.qubit_count
    if noise is not None and noise_engine == "fused" and rng is not None and _mixed_unitary(program, noise):
        # every matching channel is a mixture of scaled unitaries: its branch weights do not
        # depend on the state, so the branches are drawn up front and the run stays fused
        return _run_presampled(program, rng, noise, state=state, device=device, stream=stream,
                               max_qubits=max_qubits, chunk_log2=chunk_log2, initial_index=initial_index,
                               initial_state=initial_state,
                               opts=N.options(fuse=fuse, tile_qubits=tile_qubits, reg_qubits=reg_qubits,
                                              low_qubits=low_qubits, profile=profile, jit=jit,
                                              plan_objective=1))
    if (noise is not None and noise_engine == "fused" and rng is not None and state is None
            and initial_state is None and initial_index == 0 and stream is None):
        # one trajectory = a batch of one: each noisy gate is ONE pass that applies U.K_c and
        # reduces the next noisy gate's branch weights (noisy_batch.py), instead of a weight
        # pass + an apply pass per noisy gate; the same draws from `rng`
        from .noisy_batch import run_noisy_batch

        nb = run_noisy_batch(program, noise, [rng], device=device, max_qubits=max_qubits, fuse=fuse, groups=1)
        return RunResult(cregs=nb.cregs[0], tables=nb.tables[0], state=nb.states[0], stats=nb.stats)
    if state is None:
        state = init_state(n, chunk_log2=chunk_log2, max_qubits=max_qubits, device=device, stream=stream)
    elif state.qubit_count != n:
        raise ValueError("state has a different qubit count")
    if initial_state is not None:
        state.amplitudes = initial_state
    else:
        state.set_basis(initial_index)
    result = RunResult(cregs=[0] * program.creg_count, state=state)
    opts = N.options(fuse=fuse, tile_qubits=tile_qubits, reg_qubits=reg_qubits,
                     low_qubits=low_qubits, profile=profile, jit=jit)
    batch: list = []
    for inst in program.instructions:
        if inst.is_gate and noise is None:
            batch.append(inst)
            continue
        _flush(state, batch, opts, result.stats)
        apply_instruction(state, inst, None, rng, noise, result)
    _flush(state, batch, opts, result.stats)
    return result


def _noisy_kraus(inst, noise):
    """(dense base with controls embedded, qubits, kraus) of a noisy gate, else None
    (the reference's _noisy_dispatch conditions, statevector.py:343-357)."""
    if not inst.is_gate:
        return None
    base, targets, controls = gates.controlled_form(inst)
    qubits = tuple(controls) + tuple(targets)
    if len(qubits) > 2:
        return None
    kraus = noise.kraus_for(inst, len(qubits))
    if kraus is None:
        return None
    return gates.embed_controls(base, len(controls)), qubits, kraus


def _mixed_unitary(program, noise) -> bool:
    """True when every noisy gate's Kraus operators are scaled unitaries
    (K^dag K = w I: bit/phase/bit-phase flips, depolarising) on a unitary gate, so
    ||K_i psi||^2 = w_i for every normalised state."""
    for inst in program.instructions:
        if inst.is_gate and inst.name in ("P0", "P1") and noise.kraus_for(inst, 1) is not None:
            return False
        nk = _noisy_kraus(inst, noise)
        if nk is None:
            continue
        for k in nk[2]:
            kk = k.conj().T @ k
            if np.abs(kk - kk[0, 0] * np.eye(k.shape[0])).max() > 1e-14:
                return False
    return True


class _Replay:
    """Hands out pre-drawn uniforms in order (stands in for `rng.random()`)."""

    def __init__(self, values):
        self.values, self.i = values, 0

    def random(self):
        v = self.values[self.i]
        self.i += 1
        return float(v)


_PAULIS = (gates.I2, gates.X, gates.Y, gates.Z)
_PLAN_CACHE: dict = {}  # (records bytes, n, options) -> qsv_plan handle (clean segments with errors)


def _pauli_kinds(v: np.ndarray):
    """Kinds (0 I, 1 X, 2 Y, 3 Z) per qubit, MSB first, if v is a Pauli string, else None."""
    if v.shape[0] == 2:
        for k, P in enumerate(_PAULIS):
            if np.abs(v - P).max() < 1e-12:
                return (k,)
        return None
    for a, Pa in enumerate(_PAULIS):
        for b, Pb in enumerate(_PAULIS):
            if np.abs(v - np.kron(Pa, Pb)).max() < 1e-12:
                return (a, b)
    return None


def _cached_plan(rec: np.ndarray, n: int, opts):
    key = (rec.tobytes(), n, opts.fuse, opts.tile_qubits, opts.reg_qubits, opts.low_qubits, opts.jit)
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        plan = C.c_void_p()
        N.check(N.lib().qsv_plan_create(rec.ctypes.data, len(rec), n, C.byref(opts), C.byref(plan)))
        if len(_PLAN_CACHE) >= 8:
            old = next(iter(_PLAN_CACHE))
            N.lib().qsv_plan_destroy(_PLAN_CACHE.pop(old))
        _PLAN_CACHE[key] = plan
    return plan


def _run_presampled(program, rng, noise, *, state, device, stream, max_qubits, chunk_log2, initial_index,
                    initial_state, opts) -> RunResult:
    """run_full for mixed-unitary noise (the reference trajectory, noise.py:188-222): one
    uniform per noisy gate and per MEASURE, in program order, drawn up front (the same
    stream); noisy gate j's branch is picked with the reference's cumulative rule.  K_c /
    sqrt(w_c) is a Pauli string for the flip and depolarising channels, so the reference's
    renormalised U.K_c/sqrt(w_c) is "Pauli error(s) before U": each MEASURE-separated
    segment runs the CLEAN gates' fused plan with the errors handed to
    `qsv_plan_execute_paulis` (no new kernels to compile; error-free runs are the
    noiseless run).  A branch that is not a Pauli string falls back to the dense gate."""
    n = program.qubit_count
    infos = [_noisy_kraus(i, noise) for i in program.instructions]
    n_draws = sum(1 for i, x in zip(program.instructions, infos) if x is not None or i.name == "MEASURE")
    replay = _Replay(rng.random(n_draws) if n_draws else [])
    if state is None:
        state = init_state(n, chunk_log2=chunk_log2, max_qubits=max_qubits, device=device, stream=stream)
    elif state.qubit_count != n:
        raise ValueError("state has a different qubit count")
    if initial_state is not None:
        state.amplitudes = initial_state
    else:
        state.set_basis(initial_index)
    result = RunResult(cregs=[0] * program.creg_count, state=state)
    L = N.lib()
    seg: list = []      # clean gate triplets of the current segment
    errs: list = []     # (gate index in seg, qubit, kind)
    dense = [False]     # a non-Pauli branch forces a plain run with explicit gates

    def account(st):
        for k, v in st.as_dict().items():
            result.stats[k] = result.stats.get(k, 0) + v

    def flush():
        if not seg:
            return
        rec = N.gate_records(seg)
        st = N.qsv_run_stats()
        rc = None  # None: no Pauli-plan attempt (a dense branch in the segment)
        if not dense[0]:  # error-free segments use the same cached plan (and its compiled kernels)
            pa = np.zeros(len(errs), dtype=N.PAULI_DTYPE)
            for k, e in enumerate(errs):
                pa[k] = e
            rc = L.qsv_plan_execute_paulis(state.handle, _cached_plan(rec, n, opts), pa.ctypes.data, len(errs),
                                           C.byref(opts), C.byref(st))
            if rc not in (0, N.QSV_E_UNSUPPORTED):
                N.check(rc)
        if rc != 0:
            if errs:  # the plan cannot take Pauli errors (or a dense branch is present): explicit gates
                items = []
                by_gate: dict = {}
                for g, q, kind in errs:
                    by_gate.setdefault(g, []).append((q, kind))
                for g, t in enumerate(seg):
                    for q, kind in by_gate.get(g, ()):
                        items.append((_PAULIS[kind], (q,), ()))
                    items.append(t)
                rec = N.gate_records(items)
            N.check(L.qsv_run(state.handle, rec.ctypes.data, len(rec), C.byref(opts), C.byref(st)))
        account(st)
        seg.clear()
        errs.clear()
        dense[0] = False

    for inst, nk in zip(program.instructions, infos):
        if nk is not None:
            u, qubits, kraus = nk
            w = [float(np.real(np.trace(k.conj().T @ k))) / k.shape[0] for k in kraus]
            r = replay.random() * sum(w)
            acc, choice = 0.0, len(w) - 1
            for i, wi in enumerate(w):
                acc += wi
                if r < acc:
                    choice = i
                    break
            kinds = _pauli_kinds(kraus[choice] / math.sqrt(w[choice]))
            if kinds is None:
                m = u @ kraus[choice]
                if abs(w[choice] - 1.0) > 1e-12:
                    m = m / math.sqrt(w[choice])
                seg.append((m, qubits, ()))
                dense[0] = True
                continue
            for q, kind in zip(qubits, kinds):
                if kind:
                    errs.append((len(seg), q, kind))
            seg.append(_gate_triplet(inst))
        elif inst.is_gate:
            seg.append(_gate_triplet(inst))
        else:
            flush()
            apply_instruction(state, inst, None, replay, None, result)
    flush()
    result.stats["noise_engine"] = "presampled"
    return result


def run_batch(programs, outputs, *, device: int = 0, max_qubits: int = DEFAULT_MAX_QUBITS,
              rng: np.random.Generator | None = None, states=None, **run_kw) -> list[RunResult]:
    """Run several programs and bring every final state to host memory.

    The reference equivalent is a loop of `run_full(program)` followed by
    reading `result.state.amplitudes` (statevector.py:397-430).  Here two
    device states alternate, each on its own stream: program i's device->host
    copy (PCIe, ~5x longer than simulating C2) overlaps program i+1's fused
    passes.  `outputs[i]` must be a pinned, C-contiguous complex128 host array
    of 2^n amplitudes (e.g. ``torch.empty(2**n, dtype=torch.complex128,
    pin_memory=True).numpy()``); it is complete when this function returns.
    Programs may be given as text (parsed in turn).  A buffer may be repeated
    every second program (its earlier result is then overwritten, in order).
    All programs must have the same qubit count.  The returned results carry
    `amplitudes` (= outputs[i]) instead of a device `state`.  Extra keywords
    go to `run_full`; `states` optionally supplies the two device states
    (kept open; otherwise they are created and freed here).
    """
    from .program import parse_program

    programs = list(programs)
    if not programs:
        return []
    if len(outputs) != len(programs):
        raise ValueError("one output buffer per program")
    # program texts are parsed as their turn comes (host work that overlaps the
    # previous download)
    first = programs[0] if not isinstance(programs[0], str) else parse_program(programs[0])
    n = first.qubit_count

    for out in outputs:
        if out.dtype != np.complex128 or not out.flags.c_contiguous or out.size != 1 << n:
            raise ValueError("outputs must be C-contiguous complex128 arrays of 2^n amplitudes")
    own = states is None
    if own:
        states = [init_state(n, max_qubits=max_qubits, device=device) for _ in range(min(2, len(programs)))]
    results = []
    try:
        for i, (prog, out) in enumerate(zip(programs, outputs)):
            if isinstance(prog, str):
                prog = first if i == 0 else parse_program(prog)
            if prog.qubit_count != n:
                raise ValueError("run_batch needs programs of one qubit count")
            st = states[i % len(states)]
            # the state's stream orders this run after its previous download
            res = run_full(prog, rng, state=st, max_qubits=max_qubits, **run_kw)
            N.check(N.lib().qsv_download_async(st.handle, out.ctypes.data, 0, out.size))
            res.state = None
            res.amplitudes = out
            results.append(res)
        for st in states:
            st.synchronize()
    finally:
        if own:
            for st in states:
                st.close()
    return results
