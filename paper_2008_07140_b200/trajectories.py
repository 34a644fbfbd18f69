"""Batched depolarising-noise trajectories (BASELINE config 5).

Every trajectory t replays the reference's trajectory semantics
(`run_full(prog, default_rng(seed_t), make_noise_model("depolarizing", p))`,
statevector.py:343-357 + noise.py:188-222) with the Pauli branch of every
<=2-qubit gate pre-sampled on the host (`workloads.sample_pauli_insertions`)
and inserted as explicit X/Y/Z gates before that gate, so each trajectory is a
noiseless program run by the fused engine.

Execution on one GPU: one device state is reused for all trajectories, and
ALL of them run on the clean circuit's plan, whose specialised kernels are
compiled once: a trajectory's errors go to libqsv as (gate, qubit, Pauli)
triples (`qsv_plan_execute_paulis`), which moves each error to a pass
boundary (conjugating the gates on its qubit that it crosses), applies it
there as a Pauli-string kernel, and runs only the (typically one) pass holding
conjugated gates through the interpreted kernel - no per-trajectory NVRTC
compile, no per-trajectory re-planning.  Plans the Pauli path cannot take
(SWAP relabelling, super-passes, errors that would cross a gate controlled by
their qubit) fall back to running the noisy program itself.  With `dedup=True` the error-free
trajectories are simulated once and the result reused - reported separately
(`TrajectoryReport.unique_runs`).  Across GPUs trajectories are independent
replicas: rank r takes t = r, r+P, ... (no collective while they run); with
`gather=True` (default) and an initialised process group the per-trajectory
tables, error counts, norms and kept amplitudes are gathered on rank 0, which
returns the whole batch in trajectory order (`gather_reports`); the other ranks
return their own slice.
"""

from __future__ import annotations

import ctypes as C
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from . import statevector as SV
from .program import Program
from .workloads import noisy_trajectory_program, sample_pauli_insertions, trajectory_seed


@dataclass
class TrajectoryReport:
    n_qubits: int
    trajectories: list          # trajectory ids handled here
    errors: list                # number of inserted Paulis per trajectory
    probe_qubits: tuple
    tables: np.ndarray          # PMEASURE table over probe qubits per trajectory
    norms: np.ndarray
    kept: dict = field(default_factory=dict)   # trajectory id -> amplitudes
    gate_updates: int = 0       # sum over trajectories of (gates incl. Paulis) * 2^n
    unique_runs: int = 0
    seconds: float = 0.0


_PLANS: dict = {}  # (gate records, n, options, device) -> qsv_plan of the clean circuit
_MAX_PLANS = 8


def gather_reports(rep: TrajectoryReport, dist, group=None) -> TrajectoryReport:
    """All ranks' slices on rank 0, trajectories in id order (one all_gather_object;
    the other ranks get their own report back).  Work counters are summed and the
    time is the max over ranks."""
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, rep, group=group)
    if dist.get_rank(group) != 0:
        return rep
    rows = sorted((t, r, i) for r, pr in enumerate(parts) for i, t in enumerate(pr.trajectories))
    tables = np.stack([parts[r].tables[i] for _, r, i in rows]) if rows else rep.tables[:0]
    norms = np.array([parts[r].norms[i] for _, r, i in rows])
    kept = {}
    for pr in parts:
        kept.update(pr.kept)
    return TrajectoryReport(rep.n_qubits, [t for t, _, _ in rows], [parts[r].errors[i] for _, r, i in rows],
                            rep.probe_qubits, tables, norms, kept, sum(pr.gate_updates for pr in parts),
                            sum(pr.unique_runs for pr in parts), max(pr.seconds for pr in parts))


def _run_clean_batches(slots, clean_gates, n, b, pq, tables, device, opts) -> int:
    """Error-free trajectories, 2^b per (n + b)-qubit state (the last batch is padded
    with extra copies so every batch reuses one plan and its compiled kernels); fills
    tables[slot] from one PMEASURE over (batch qubits, probe qubits) per batch."""
    L = N.lib()
    B = 1 << b
    rec = SV.compile_gates(clean_gates)
    st = SV.init_state(n + b, max_qubits=n + b, device=device)
    ones = np.ones(B, dtype=np.complex128)
    qs = np.array([n + j for j in range(b - 1, -1, -1)] + list(pq), dtype=np.int32)
    table = np.zeros(1 << len(qs), dtype=np.float64)
    runs = 0
    try:
        for s0 in range(0, len(slots), B):
            part = slots[s0:s0 + B]
            st.set_basis(0)
            N.check(L.qsv_upload_strided(st.handle, ones.ctypes.data, 0, B, 1 << n))
            stats = N.qsv_run_stats()
            N.check(L.qsv_run(st.handle, rec.ctypes.data, len(rec), C.byref(opts), C.byref(stats)))
            N.check(L.qsv_pmeasure(st.handle, qs.ctypes.data, len(qs), table.ctypes.data))
            per = table.reshape(B, -1)
            for j, k in enumerate(part):
                tables[k] = per[j]
            runs += len(part)
    finally:
        st.close()
    return runs


def run_trajectories(program: Program, p: float, n_traj: int, base_seed: int = 0, *,
                     probe_qubits=(0, 1, 2), keep=(), dedup: bool = False, device: int = 0,
                     stream=None, rank: int = 0, world: int = 1, state: SV.StateVector | None = None,
                     options=None, streams: int = 2, batch_clean: int = 0, gather: bool = True,
                     group=None) -> TrajectoryReport:
    """`batch_clean` = b > 0: the error-free trajectories (not kept, not deduplicated) run
    2^b at a time as ONE (n + b)-qubit state - trajectory index = top qubits - through
    the clean circuit's fused plan (every trajectory block is simulated; the passes are
    2^b times larger, so they run nearer the HBM roofline than 256 MiB passes), and
    their probe tables come from one PMEASURE over (batch qubits, probe qubits).
    Off by default: on C5 (n = 24, b = 6) it measured slower than the one-by-one runs on
    two streams."""
    n = program.qubit_count
    mine = list(range(rank, n_traj, world))
    if state is None:
        state = SV.init_state(n, max_qubits=max(n, SV.DEFAULT_MAX_QUBITS), device=device, stream=stream)
    # consecutive trajectories alternate between `streams` device states, each
    # with its own stream: one trajectory's pass tails and launch gaps overlap
    # the next one's passes
    # (only while a second state is small: at n > 28 it would cost >= 8 GiB)
    states = [state] + [SV.init_state(n, max_qubits=max(n, SV.DEFAULT_MAX_QUBITS), device=device)
                        for _ in range(max(0, streams - 1) if n <= 28 else 0)]
    L = N.lib()
    # 4 forced low tile qubits for the small (2^24) trajectory states: C5 932-940 ms
    # vs 964-988 ms with the C2 default of 3 (same box, alternating)
    # pass-count look-ahead for the clean plan: plans that carry Pauli errors run faster when
    # front-loaded than time-balanced (C5 0.79 s vs 1.06-1.20 s, same box, alternating)
    opts_clean = options or N.options(low_qubits=4 if n >= 16 else 0, plan_objective=1)
    opts_noisy = N.options(fuse=True, jit=-1, tile_qubits=opts_clean.tile_qubits,
                           reg_qubits=opts_clean.reg_qubits, low_qubits=opts_clean.low_qubits)
    clean_gates = [i for i in program.instructions if i.is_gate]
    gate_index = {}
    for j, inst in enumerate(program.instructions):
        if inst.is_gate:
            gate_index[j] = len(gate_index)
    clean_rec = SV.compile_gates(clean_gates)
    # the clean circuit's plan is built once per (circuit, options) and kept, as
    # qsv_run keeps its plans: repeated batches of one circuit skip the planner
    key = (clean_rec.tobytes(), n, bytes(opts_clean), device)
    clean_plan = _PLANS.get(key)
    if clean_plan is None:
        clean_plan = C.c_void_p()
        N.check(L.qsv_plan_create(clean_rec.ctypes.data, len(clean_rec), n, C.byref(opts_clean),
                                  C.byref(clean_plan)))
        while len(_PLANS) >= _MAX_PLANS:
            L.qsv_plan_destroy(_PLANS.pop(next(iter(_PLANS))))
        _PLANS[key] = clean_plan
    pq = np.asarray(probe_qubits, dtype=np.int32)
    tables = np.zeros((len(mine), 1 << len(pq)))
    norms = np.zeros(len(mine))
    errors, kept = [], {}
    clean_cache = None  # (slot of the first simulated clean trajectory)
    dedup_from = {}     # slot -> slot whose table it reuses
    # probe tables land in device memory, one row per trajectory, read once at
    # the end: the host runs ahead of the GPU (no per-trajectory synchronisation)
    import torch

    async_tables = len(pq) <= 4 and torch.cuda.is_available()
    if async_tables:
        # no fill kernel: the libqsv streams are not ordered after torch's; every
        # simulated row is written by its pmeasure, deduplicated rows are copied below
        dev_tables = torch.empty((max(1, len(mine)), 1 << len(pq)), dtype=torch.float64, device=f"cuda:{device}")
    updates = 0
    unique = 0
    t0 = time.perf_counter()
    # QSV_TRAJ_TRACE=<file>: per-trajectory host launch times (diagnostic)
    trace = [] if os.environ.get("QSV_TRAJ_TRACE") else None
    # errors are sampled inside the launch loop, so the host sampling of one
    # trajectory overlaps the GPU passes of the earlier ones (sampling all 1024
    # C5 trajectories up front left the GPU idle for ~78 ms); only the batched
    # clean mode needs them all first, to know which trajectories are error-free
    sampled = {}

    def draws(k, t):
        if k not in sampled:
            ins = sample_pauli_insertions(program, p, trajectory_seed(base_seed, t))
            sampled[k] = (ins, sum(len(v) for v in ins.values()))
        return sampled[k]

    batched = set()
    if batch_clean > 0 and not dedup and n + batch_clean <= 34:
        batched = {k for k, t in enumerate(mine) if draws(k, t)[1] == 0 and t not in keep}
    try:
        if batched:
            unique += _run_clean_batches(sorted(batched), clean_gates, n, batch_clean, pq, tables, device, opts_clean)
        for k, t in enumerate(mine):
            ins, n_err = draws(k, t)
            sampled.pop(k, None)
            errors.append(n_err)
            updates += (len(clean_gates) + n_err) << n
            if k in batched:
                continue
            if n_err == 0 and dedup and clean_cache is not None and t not in keep:
                dedup_from[k] = clean_cache
                continue
            state = states[unique % len(states)]
            state.set_basis(0)
            stats = N.qsv_run_stats()
            pa = np.zeros(n_err, dtype=N.PAULI_DTYPE)
            k2 = 0
            for idx, picks in ins.items():
                for q, g in picks:
                    pa[k2] = (gate_index[idx], q, "IXYZ".index(g))
                    k2 += 1
            if async_tables:
                # the plan's last pass accumulates the probe table while it
                # stores (no extra read of the state)
                rc = L.qsv_plan_execute_probe(state.handle, clean_plan, pa.ctypes.data, n_err, pq.ctypes.data,
                                              len(pq), C.c_void_p(dev_tables[k].data_ptr()), C.byref(opts_clean),
                                              C.byref(stats))
            else:
                rc = L.qsv_plan_execute_paulis(state.handle, clean_plan, pa.ctypes.data, n_err, C.byref(opts_clean),
                                               C.byref(stats))
            if rc == N.QSV_E_UNSUPPORTED:
                noisy = noisy_trajectory_program(program, p, trajectory_seed(base_seed, t))
                rec = SV.compile_gates([i for i in noisy.instructions if i.is_gate])
                rc = L.qsv_run(state.handle, rec.ctypes.data, len(rec), C.byref(opts_noisy), C.byref(stats))
                if rc == 0 and async_tables:
                    rc = L.qsv_pmeasure_async(state.handle, pq.ctypes.data, len(pq),
                                              C.c_void_p(dev_tables[k].data_ptr()))
            N.check(rc)
            if trace is not None:
                trace.append((k, n_err, time.perf_counter() - t0))
            unique += 1
            if not async_tables:
                tables[k] = SV.pmeasure(state, pq)
            if t in keep:
                kept[t] = state.amplitudes
            if n_err == 0 and clean_cache is None:
                clean_cache = k
        if async_tables and mine:
            for st_ in states:
                N.check(L.qsv_synchronize(st_.handle))
            rows = dev_tables.cpu().numpy()[: len(mine)]
            for k in range(len(mine)):
                if k not in batched:
                    tables[k] = rows[k]
        if trace is not None:
            trace.append((-1, 0, time.perf_counter() - t0))
            with open(os.environ["QSV_TRAJ_TRACE"], "a") as fh:
                fh.write(" ".join(f"{a}:{b}:{c:.5f}" for a, b, c in trace) + "\n")
        for k, src in dedup_from.items():
            tables[k] = tables[src]
        norms[:] = tables.sum(axis=1)  # the probe table sums to ||psi||^2
    finally:
        # every state's stream (states[0] included) is idle before dev_tables, which its
        # kernels write, can go back to torch's allocator
        for st_ in states:
            L.qsv_synchronize(st_.handle)
        for st_ in states[1:]:
            st_.close()
    rep = TrajectoryReport(n, mine, errors, tuple(int(q) for q in pq), tables, norms, kept, updates, unique,
                           time.perf_counter() - t0)
    if gather and world > 1:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            rep = gather_reports(rep, dist, group)
    return rep
