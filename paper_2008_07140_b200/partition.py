"""Partial-amplitude mode on the B200 engine (reference `qcsim/partition.py:1-192`).

Same API as the reference: `plan_partition`, `decompose_crossing`,
`parse_target`, `run_partial`, with the same error classes (`UncuttableGate`,
`BranchExplosion`, `MalformedTarget`, `UnsupportedGate`).

The reference cuts the register at qubit `cut`, turns each of the c crossing
controlled gates into a projector selector (P0 on the control | P1 on the
control + the base action on the target, `partition.py:96-140`) and runs the
2·2^c half-circuits one by one through `run_full`, then sums
up_b[t_upper]·lo_b[t_lower] over the branches (`partition.py:182-191`).

Here the 2^c branches of one half are ONE state: the branch index becomes c
extra low qubits ("branch qubits", bit j = crossing gate j's selector), the
half's own qubits sit above them, and the selector logic becomes ordinary
gates on that (m + c)-qubit register:

* control side of crossing gate j: the projector "control bit == branch bit
  j", a 2-qubit diagonal diag(1, 0, 0, 1) on (branch qubit j, control);
* target side: the base action controlled by branch qubit j;
* start: amplitude 1 on every branch (|0..0> of the half in each branch).

So each half is one fused run of the scheduler + specialised pass kernels
(`qsv_run`) over 2^(m+c) amplitudes instead of 2^c tiny launches, and branch
b's amplitude t sits at index (t << c) | b: the recombination reads two
contiguous 2^c slices per target.  When m + c exceeds `batch_qubits` the top
selector bits are fixed per run (concrete projectors / actions, as in the
reference's branch programs) and the runs are summed.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _native as N
from . import gates
from .errors import BranchExplosion, MalformedTarget, TooManyQubits, UncuttableGate, UnsupportedGate
from .program import Instruction, Program

DEFAULT_BRANCH_BUDGET = 1 << 16
DEFAULT_BATCH_QUBITS = 28  # 4 GiB per batched half-state

_PROJ_EQ = np.diag([1.0, 0.0, 0.0, 1.0]).astype(np.complex128)  # keep bit(control) == bit(branch)


@dataclass(frozen=True)
class CrossingGate:
    position: int  # index into program.instructions
    control: int
    target: int
    base: tuple  # 2x2 target action, row-major


@dataclass(frozen=True)
class PartitionPlan:
    program: Program
    cut: int
    qubit_count: int
    crossing_gates: tuple

    @property
    def c(self) -> int:
        return len(self.crossing_gates)

    @property
    def branch_count(self) -> int:
        return 1 << self.c

    @property
    def subcircuit_count(self) -> int:
        return 2 << self.c


@dataclass(frozen=True)
class BranchCircuit:
    branch_id: int
    upper_program: Program
    lower_program: Program


def plan_partition(program: Program, cut: int, branch_budget: int = DEFAULT_BRANCH_BUDGET) -> PartitionPlan:
    """Find the gates spanning the cut; each must be a 1-control 1-target gate
    (reference `partition.py:55-90`)."""
    n = program.qubit_count
    if not 0 < cut < n:
        raise UncuttableGate(f"cut {cut} outside (0, {n})")
    found = []
    for pos, inst in enumerate(program.instructions):
        if inst.name == "MEASURE":
            raise UnsupportedGate("MEASURE is not supported in partial mode", inst.line)
        if not inst.is_gate:
            continue
        qs = inst.all_qubits()
        below = any(q < cut for q in qs)
        above = any(q >= cut for q in qs)
        if not (below and above):
            continue
        base, targets, controls = gates.controlled_form(inst)
        if len(qs) != 2 or len(controls) != 1 or len(targets) != 1:
            raise UncuttableGate(f"crossing gate {inst.name} is not a controlled two-qubit gate", inst.line)
        found.append(CrossingGate(pos, controls[0], targets[0], tuple(np.asarray(base).reshape(-1).tolist())))
    if (1 << len(found)) > branch_budget:
        raise BranchExplosion(f"2^{len(found)} branches exceed the budget of {branch_budget}")
    return PartitionPlan(program, cut, n, tuple(found))


def _side(q: int, cut: int) -> tuple[str, int]:
    return ("lower", q) if q < cut else ("upper", q - cut)


def _routed(inst: Instruction, cut: int) -> tuple[str, Instruction]:
    if all(q < cut for q in inst.all_qubits()):
        return "lower", inst
    return "upper", replace(inst, qubits=tuple(q - cut for q in inst.qubits),
                            controls=tuple(q - cut for q in inst.controls))


def decompose_crossing(plan: PartitionPlan) -> list[BranchCircuit]:
    """The reference's explicit 2^c branch programs (`partition.py:96-140`):
    selector bit j = 0 puts P0 on crossing gate j's control, bit j = 1 puts P1
    there and the base action (as U4) on its target.  `run_partial` does not
    build these; it runs the batched form described in the module docstring."""
    cut = plan.cut
    where = {cg.position: (j, cg) for j, cg in enumerate(plan.crossing_gates)}
    out = []
    for b in range(plan.branch_count):
        halves: dict[str, list] = {"lower": [], "upper": []}
        for pos, inst in enumerate(plan.program.instructions):
            if not inst.is_gate:
                continue
            if pos not in where:
                side, routed = _routed(inst, cut)
                halves[side].append(routed)
                continue
            j, cg = where[pos]
            bit = (b >> j) & 1
            side, q = _side(cg.control, cut)
            halves[side].append(Instruction("P1" if bit else "P0", (q,), line=inst.line))
            if bit:
                side, q = _side(cg.target, cut)
                halves[side].append(Instruction("U4", (q,), matrix=cg.base, line=inst.line))
        out.append(BranchCircuit(b, Program(plan.qubit_count - cut, 0, tuple(halves["upper"])),
                                 Program(cut, 0, tuple(halves["lower"]))))
    return out


def parse_target(text: str, n: int) -> int:
    """An n-character 0/1 string, qubit n-1 leftmost, to an amplitude index
    (reference `partition.py:143-148`)."""
    s = text.strip()
    if len(s) != n or any(ch not in "01" for ch in s):
        raise MalformedTarget(f"target {text!r} is not an {n}-bit 0/1 string")
    return int(s, 2)


def batch_bits(plan: PartitionPlan, batch_qubits: int = DEFAULT_BATCH_QUBITS) -> int:
    """How many selector bits become branch qubits (the rest are looped over)."""
    m = max(plan.cut, plan.qubit_count - plan.cut)
    return max(0, min(plan.c, batch_qubits - m))


def branch_streams(plan: PartitionPlan, cb: int, fixed: int = 0):
    """Gate triplets (base, targets, controls) of the two batched halves.

    Selector bits j < cb are branch qubits j of both halves (the half's qubit
    q becomes qubit q + cb); bits j >= cb take the value bit (j - cb) of
    `fixed`.  Returns ((lower_triplets, m_lower), (upper_triplets, m_upper))
    with m = half qubits + cb.  Pure host code (checked on the CPU by the
    tests against the reference's branch programs)."""
    cut, n = plan.cut, plan.qubit_count
    where = {cg.position: (j, cg) for j, cg in enumerate(plan.crossing_gates)}
    halves: dict[str, list] = {"lower": [], "upper": []}

    def lift(side, base, targets, controls):
        halves[side].append((np.asarray(base, dtype=np.complex128), tuple(q + cb for q in targets),
                             tuple(q + cb for q in controls)))

    for pos, inst in enumerate(plan.program.instructions):
        if not inst.is_gate:
            continue  # PMEASURE does not enter amplitude recombination
        if pos not in where:
            side, routed = _routed(inst, cut)
            base, targets, controls = gates.controlled_form(routed)
            if len(targets) > 2:
                raise UnsupportedGate(f"{inst.name} targets {targets}", inst.line)
            lift(side, base, targets, controls)
            continue
        j, cg = where[pos]
        cside, cq = _side(cg.control, cut)
        tside, tq = _side(cg.target, cut)
        base = np.array(cg.base, dtype=np.complex128).reshape(2, 2)
        if j < cb:
            # branch qubit j (unshifted index j) selects the projector / action
            halves[cside].append((_PROJ_EQ, (j, cq + cb), ()))
            halves[tside].append((base, (tq + cb,), (j,)))
        else:
            bit = (fixed >> (j - cb)) & 1
            lift(cside, gates.P1 if bit else gates.P0, (cq,), ())
            if bit:
                lift(tside, base, (tq,), ())
    return (halves["lower"], cut + cb), (halves["upper"], n - cut + cb)


# device states kept between run_partial calls (keyed by device and qubit count), so
# repeated calls do not pay cudaMalloc/cudaFree of two multi-GiB buffers each time
_POOL: dict = {}


def release_cached_states() -> None:
    """Free the device states run_partial keeps for reuse."""
    for sts in _POOL.values():
        for st in sts:
            st.close()
    _POOL.clear()


def _take_state(m: int, device: int):
    from .statevector import init_state

    free = _POOL.get((device, m))
    if free:
        return free.pop()
    if _POOL:  # keep only states of the current shape
        release_cached_states()
    return init_state(m, max_qubits=m, device=device)


def _give_state(st, device: int) -> None:
    _POOL.setdefault((device, st.qubit_count), []).append(st)


def _run_half(triplets, m: int, cb: int, device: int, max_qubits: int, options):
    st = _take_state(m, device)
    st.set_basis(0)
    if cb:
        ones = np.ones(1 << cb, dtype=np.complex128)  # every branch starts at |0..0>
        N.check(N.lib().qsv_upload(st.handle, ones.ctypes.data, 0, ones.size))
    if triplets:
        rec = N.gate_records(triplets)
        stats = N.qsv_run_stats()
        N.check(N.lib().qsv_run(st.handle, rec.ctypes.data, len(rec), C.byref(options), C.byref(stats)))
    return st


def _slices(st, m: int, cb: int, rows) -> dict:
    """{row: 2^cb amplitudes of half-index `row` across the branches}: one
    device gather of the requested rows + one D2H (`qsv_gather_rows`)."""
    rows = sorted(set(rows))
    out = {}
    for s0 in range(0, len(rows), 4096):
        part = rows[s0:s0 + 4096]
        offs = np.array([r << cb for r in part], dtype=np.uint64)
        buf = np.empty((len(part), 1 << cb), dtype=np.complex128)
        N.check(N.lib().qsv_gather_rows(st.handle, offs.ctypes.data, len(part), 1 << cb, buf.ctypes.data))
        out.update(zip(part, buf))
    return out


def run_partial(program: Program, cut: int, targets, *, workers: int = 1,
                branch_budget: int = DEFAULT_BRANCH_BUDGET, max_qubits: int = 30,
                batch_qubits: int = DEFAULT_BATCH_QUBITS, device: int = 0,
                fuse: bool = True, rank: int = 0, world: int = 1, group=None,
                options=None) -> dict[str, complex]:
    """Amplitudes of the requested basis strings (reference `partition.py:151-192`).

    `workers` is accepted and ignored (the GPU runs each batched half as one
    fused program).  `max_qubits` bounds each half like the reference's
    per-branch `run_full`; `batch_qubits` bounds a batched half-state
    (half qubits + branch qubits).

    Sharded (world > 1, one process per GPU under torch.distributed): the
    selector runs (values of the selector bits that are not branch qubits) are
    dealt round-robin over the ranks — with at least `world` runs, taking bits
    from the branch qubits if needed — and the per-target sums are added with
    one all-reduce; every rank returns the full dict."""
    plan = plan_partition(program, cut, branch_budget)
    n = program.qubit_count
    wanted = [(t, parse_target(t, n)) for t in targets]
    wanted = list(dict(wanted).items())  # a repeated target string is one output entry (partition.py:184-191)
    m_half = max(cut, n - cut)
    if m_half > max_qubits:
        raise TooManyQubits(f"{m_half} qubits in one half exceed the limit of {max_qubits}")
    cb = batch_bits(plan, max(batch_qubits, m_half))
    if world > 1:
        need = (world - 1).bit_length()  # selector runs >= world where the branch count allows
        cb = max(0, min(cb, plan.c - need))
    low = (1 << cut) - 1
    rows_lo = [i & low for _, i in wanted]
    rows_up = [i >> cut for _, i in wanted]
    opts = options or N.options(fuse=fuse)  # `options`: planner tile/register/low qubits
    acc = {t: 0j for t, _ in wanted}
    for fixed in range(rank, 1 << (plan.c - cb), world):
        (tl, ml), (tu, mu) = branch_streams(plan, cb, fixed)
        lo = _run_half(tl, ml, cb, device, max_qubits, opts)  # each state runs on its own stream:
        up = _run_half(tu, mu, cb, device, max_qubits, opts)  # the two halves overlap
        try:
            lo_rows = _slices(lo, ml, cb, rows_lo)
            up_rows = _slices(up, mu, cb, rows_up)
        finally:
            _give_state(lo, device)
            _give_state(up, device)
        for (t, _), rl, ru in zip(wanted, rows_lo, rows_up):
            acc[t] += complex(np.dot(up_rows[ru], lo_rows[rl]))  # branch order b = 0 .. 2^cb - 1
    if world > 1:
        import torch
        import torch.distributed as dist

        vec = np.array([acc[t] for t, _ in wanted], dtype=np.complex128)
        buf = torch.from_numpy(vec.view(np.float64).copy())
        backend = dist.get_backend(group)
        if backend == "nccl":
            buf = buf.cuda(device)
        dist.all_reduce(buf, group=group)
        vec = buf.cpu().numpy().view(np.complex128)
        acc = {t: complex(v) for (t, _), v in zip(wanted, vec)}
    return acc
