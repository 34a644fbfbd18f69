"""Benchmark of the full-amplitude hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Metric: amplitude-gate updates/s = G * 2^n / time, G = gate instructions of
the expanded program.  Workload at N=1: BASELINE config 2 -
the 30-qubit 5x6 grid RQC, 24 cycles, eight cycled CZ patterns, seed 0
(16 GiB complex128 state, fused schedule with the product-state start).  A
step = reset to |0..0> and run the whole circuit.  Inputs (the 16 GiB state)
are far larger than the 126 MB L2, so no explicit flush is needed between steps.

`value` is device-timed with the state resident in HBM (CUDA events on the
engine's stream, barrier + synchronize around the K timed steps, max over
ranks).  `e2e` is the same metric through the public API (statevector.run_batch:
program text in, the full 2^n amplitude vector downloaded to pinned host memory
inside the timed region); `e2e.cold` is the first call on an unseen circuit
(planning + kernel compilation included).

N > 1 (torchrun): the state is sharded by global qubits (distributed.py).
Weak scaling (default): 2^30 amplitudes per GPU, n = 30 + log2 N (N = 1 is C2
itself, so `--gpus 1,2,4,8` is one ladder); `--local-qubits 32` gives BASELINE
C3's 64 GiB shards (n = 32 + log2 N); `--strong` fixes n (= --qubits, 32) for
every N, its N = 1 point being `--gpus 1 --strong`.

`--impl reference` times the reference CPU algorithm (the oracle port,
oracle/qsv_oracle.c, a restatement of qcsim/statevector.py) on the host
cores over a bounded sample of the same workload.

Other lines (not the driver's headline): `--workload qft` (C4), `traj` (C5,
pre-sampled depolarising trajectories), `partial` (partial-amplitude mode,
partition.py: n=36 RQC cut at 18), `noisy` (1024 general-channel trajectories,
noisy_batch.py: C1-shape RQC under amplitude damping), `--qubits 32` (C3's
single-GPU point).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "amplitude-gate updates/s"
UNIT = "amp-gate/s"
N_BASE = 30
C2 = (5, 6, 24)
SEED = 0


FP64_PEAK_GINSTR = 18050.0  # DFMA lane-instructions/s (36.1 TFLOP/s measured)


def ncu_traffic(args, passes: int):
    """DRAM bytes per pass-kernel launch, MEASURED: re-runs this bench (one warm-up +
    one timed step of the same workload) under `ncu --metrics dram__bytes_read.sum,
    dram__bytes_write.sum` and keeps the last step's `passes` launches.  Returns
    ({mean, per_launch, ...}, None) or (None, reason).  The child's own numbers are
    discarded (a number printed under ncu is never a bench value)."""
    import csv
    import shutil
    import tempfile

    if os.environ.get("QSV_BENCH_UNDER_NCU"):
        return None, "running under ncu"
    exe = shutil.which("ncu") or "/usr/local/cuda/bin/ncu"
    if not os.path.exists(exe):
        return None, "ncu not found"
    fwd = ["--workload", args.workload, "--product", str(args.product), "--jit", str(args.jit)]
    for flag, v in (("--qubits", args.qubits), ("--tile", args.tile), ("--regs", args.regs),
                    ("--low", args.low), ("--super", args.super)):
        if v:
            fwd += [flag, str(v)]
    with tempfile.TemporaryDirectory() as td:
        log = os.path.join(td, "traffic.csv")
        cmd = [exe, "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
               "--clock-control", "none", "--csv", "-k", "regex:qsv_pass|pass_kernel", "--log-file", log,
               sys.executable, str(ROOT / "bench.py"), "--steps", "1", "--warmup", "1", "--no-e2e",
               "--no-cpu-baseline", "--traffic", "off", *fwd]
        try:
            proc = subprocess.run(cmd, env=dict(os.environ, QSV_BENCH_UNDER_NCU="1"), capture_output=True,
                                  text=True, timeout=args.traffic_timeout)
        except subprocess.TimeoutExpired:
            return None, f"ncu run exceeded {args.traffic_timeout} s"
        if proc.returncode != 0 or not os.path.exists(log):
            return None, f"ncu exit {proc.returncode}: {(proc.stderr or proc.stdout)[-200:]}"
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
        rows = [r for r in csv.reader(open(log)) if len(r) > 10]
    if len(rows) < 2:
        return None, "ncu produced no launches"
    ix = {k: i for i, k in enumerate(rows[0])}
    per = {}
    for r in rows[1:]:
        rid = int(r[ix["ID"]])
        v = float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1.0)
        per.setdefault(rid, {})[r[ix["Metric Name"]]] = v
    ids = sorted(per)[-passes:]
    dram = [per[i].get("dram__bytes_read.sum", 0.0) + per[i].get("dram__bytes_write.sum", 0.0) for i in ids]
    return {"mean": sum(dram) / len(dram), "per_launch": dram,
            "read": [per[i].get("dram__bytes_read.sum", 0.0) for i in ids],
            "ncu_ms": [per[i].get("gpu__time_duration.sum", 0.0) for i in ids],
            "src": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none, "
                   "run by this bench on the same workload (last step's pass launches)"}, None


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d.get("hbm_gbs", 6650.0), "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int = 0):
        self.index = index
        self.proc = None
        self.path = Path(f"/tmp/qsv_clocks_{os.getpid()}.csv")

    _primed = False

    def __enter__(self):
        try:
            if not ClockSampler._primed:
                # the first nvidia-smi of a fresh box initialises NVML and pages the tool in,
                # which stalled host-timed launch loops (C5: 1.10-1.20 s instead of 0.79 s on
                # the first process of a box): one throwaway query before any timed region
                ClockSampler._primed = True
                subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm",
                                "--format=csv,noheader,nounits"], capture_output=True, timeout=30)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError, subprocess.TimeoutExpired):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self) -> dict:
        if self.proc is None or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lines = self.path.read_text().splitlines()
        if not lines:  # a timed region shorter than the sampling period: one query right after it
            try:
                lines = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                        "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                       timeout=20).stdout.splitlines()
            except (OSError, subprocess.TimeoutExpired):
                lines = []
        for line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower() == "active":
                    reasons.add(name)
        self.path.unlink(missing_ok=True)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("QSV_SHARE_GPU"):  # tests: every rank on GPU 0 (no kernel waits on another rank)
        local = 0
    return rank, world, local


def workloads_rqc(n: int, seed: int) -> str:
    from paper_2008_07140_b200 import workloads

    return workloads.rqc_text(*C2, seed=seed) if n == N_BASE else workloads.rqc_for_qubits(n, C2[2], seed)


def workload(n: int, kind: str = "rqc"):
    from paper_2008_07140_b200 import workloads
    from paper_2008_07140_b200.program import parse_program

    if kind == "qft":  # BASELINE config 4: QFT then DAGGER-QFT on a random state
        text = workloads.qft_text(n, round_trip=True)
    elif n == N_BASE:
        text = workloads.rqc_text(*C2, seed=SEED)
    else:
        text = workloads.rqc_for_qubits(n, C2[2], SEED)
    return text, parse_program(text)


# --------------------------------------------------------------------------
# CPU baseline (oracle port of the reference algorithm; test infrastructure)
# --------------------------------------------------------------------------


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def gate_sample(prog, stride: int):
    """Every stride-th gate of the whole circuit: the sample keeps the circuit's gate
    mix (H layer, CZ patterns, RX/RY/T) instead of its first cycle only."""
    insts = [i for i in prog.instructions if i.is_gate]
    return insts[::max(1, stride)], len(insts)


def _mix(insts) -> str:
    from collections import Counter

    return ", ".join(f"{k} {v}" for k, v in sorted(Counter(i.name for i in insts).items()))


def cpu_reference_sample(prog, budget_s: float, threads: int | None = None) -> dict:
    """The oracle port (oracle/qsv_oracle.c, restating qcsim/statevector.py:73-247
    with pthreads = WorkerPool) on a strided gate sample of the whole circuit, the
    stride chosen from a 3-gate calibration so the sample takes about `budget_s`."""
    from oracle import oracle as O

    threads = threads or O.cpu_threads()
    n = prog.qubit_count
    st = O.init_state(n, workers=threads, max_qubits=n)
    st.amplitudes[:] = 0  # first touch outside the timed region
    st.amplitudes[0] = 1
    allg = [i for i in prog.instructions if i.is_gate]
    t0 = time.perf_counter()
    for inst in (allg[0], allg[len(allg) // 2], allg[-1]):
        O.apply_instruction(st, inst, workers=threads)
    per_gate = (time.perf_counter() - t0) / 3
    stride = max(1, math.ceil(len(allg) * per_gate / max(budget_s, 1e-3)))
    sample, total = gate_sample(prog, stride)
    t0 = time.perf_counter()
    for inst in sample:
        O.apply_instruction(st, inst, workers=threads)
    dt = time.perf_counter() - t0
    del st
    return {"value": len(sample) * float(1 << n) / dt, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"gates at stride {stride} over the whole n={n} circuit: {len(sample)} of {total} gates ({_mix(sample)}), "
                      f"{dt:.1f} s, oracle/qsv_oracle.c restating qcsim/statevector.py:73-247, "
                      f"{threads} threads = WorkerPool({threads}) on {cpu_model()}",
            "seconds": dt, "gates": len(sample), "stride": stride}


def qcsim_reference_sample(text: str, stride: int, threads: int) -> dict | None:
    """The reference itself (qcsim, numba kernels, installed unmodified in
    baseline/_ref) on the same strided gate sample: its `apply_instruction`
    (statevector.py:360-394) over a WorkerPool(threads) state, after a small warm-up
    run that JIT-compiles the numba kernels.  None when it cannot be imported."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "qcsim").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/qsv_numba_cache")
    sys.path.insert(0, str(ref))
    try:
        from qcsim import statevector as QS
        from qcsim.parallel import WorkerPool
        from qcsim.program import parse_program as qparse
    except Exception as e:  # noqa: BLE001 - report why the second figure is missing
        return {"unavailable": f"{type(e).__name__}: {e}"}
    finally:
        sys.path.remove(str(ref))
    prog = qparse(text)
    n = prog.qubit_count
    pool = WorkerPool(threads)
    small = qparse("QINIT 12\n" + "\n".join(f"H {q}\nCZ {q},{(q + 1) % 12}\nRX {q},\"pi/2\"\nT {q}\n"
                                             f"SWAP {q},{(q + 5) % 12}" for q in range(12)) + "\n")
    QS.run_full(small, pool=pool, workers=threads)  # numba JIT outside the timed region
    st = QS.init_state(n, chunk_log2=QS.default_chunk_log2(n, threads), max_qubits=n)
    st.amplitudes[:] = 0
    st.amplitudes[0] = 1
    insts = [i for i in prog.instructions if i.name not in ("MEASURE", "PMEASURE")][::max(1, stride)]
    t0 = time.perf_counter()
    for inst in insts:
        QS.apply_instruction(st, inst, pool)
    dt = time.perf_counter() - t0
    del st
    return {"value": len(insts) * float(1 << n) / dt, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"qcsim (baseline/_ref, numba) apply_instruction on the same stride-{stride} gate sample: "
                      f"{len(insts)} gates, {dt:.1f} s, WorkerPool({threads})"}


def run_reference(args) -> None:
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O

    n = N_BASE
    text, prog = workload(n)
    threads = O.cpu_threads()
    per_step = args.ref_step_seconds
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference_sample(prog, per_step, threads)
        if i >= args.warmup:
            vals.append(r)
    value = statistics.median(v["value"] for v in vals)
    ms = statistics.median(v["seconds"] for v in vals) * 1e3
    qc = None if args.no_qcsim else qcsim_reference_sample(text, vals[-1]["stride"], threads)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic",
        "config": {"workload": f"C2: RQC 5x6 grid, 24 cycles, n={n}, seed {SEED} (bounded CPU sample)",
                   "n_qubits": n, "gates": len(prog.gate_instructions()), "cpu_model": cpu_model(),
                   "workers": threads},
        "cpu_baseline": {k: vals[-1][k] for k in ("kind", "cores", "sample")} | {"value": value, "unit": UNIT},
        "qcsim_numba": qc,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
# GPU arm
# --------------------------------------------------------------------------


def run_traj(args) -> None:
    """BASELINE config 5: 1024 depolarising trajectories of the 4x6, 20-cycle RQC
    (n=24, p=1e-3), split over ranks as independent replicas (no collective but
    the final result gather)."""
    import torch

    from paper_2008_07140_b200 import workloads
    from paper_2008_07140_b200.program import parse_program
    from paper_2008_07140_b200.trajectories import run_trajectories

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    prog = parse_program(workloads.rqc_text(4, 6, 20, seed=SEED))
    n_traj = args.trajectories
    bc = args.batch_clean
    topts = planner_options(args)
    run_trajectories(prog, 1e-3, min(8, n_traj), base_seed=SEED, device=local, rank=rank, world=world,
                     batch_clean=bc, options=topts)  # compiles the clean plan (and the batched one if bc > 0)
    # one whole untimed batch: the first batch of a process on a fresh box measured 0.94-1.20 s
    # against 0.77-0.79 s for every later one (host-side first-run costs of the launch loop)
    run_trajectories(prog, 1e-3, n_traj, base_seed=SEED, device=local, rank=rank, world=world,
                     streams=int(os.environ.get("QSV_TRAJ_STREAMS", "2")), dedup=args.dedup, batch_clean=bc,
                     options=topts)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        rep = run_trajectories(prog, 1e-3, n_traj, base_seed=SEED, device=local, rank=rank, world=world,
                               streams=int(os.environ.get("QSV_TRAJ_STREAMS", "2")),
                               dedup=args.dedup, batch_clean=bc, options=topts)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    # rank 0's report holds the whole batch (run_trajectories gathers the per-trajectory
    # tables there); the time is the max over ranks
    if world > 1:
        import torch.distributed as dist

        tt = torch.tensor([dt], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    updates, unique = float(rep.gate_updates), int(rep.unique_runs)
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        # the reference algorithm per trajectory (oracle port of statevector.py:73-247 on
        # the explicit-Pauli program that replays noise.py:188-222), trajectories in id
        # order until the budget is spent; the rate x 1024 trajectories is the CPU batch
        from oracle import oracle as O
        from paper_2008_07140_b200.workloads import noisy_trajectory_program, trajectory_seed

        threads = O.cpu_threads()
        done, work, t0 = 0, 0.0, time.perf_counter()
        while time.perf_counter() - t0 < args.cpu_seconds and done < n_traj:
            traj = noisy_trajectory_program(prog, 1e-3, trajectory_seed(SEED, done))
            O.run_full(traj, workers=threads)
            work += len(traj.gate_instructions()) * float(1 << prog.qubit_count)
            done += 1
        cdt = time.perf_counter() - t0
        cpu = {"value": work / cdt, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"trajectories 0..{done - 1} of the batch through oracle run_full on their explicit-Pauli "
                         f"programs ({cdt:.1f} s, {threads} threads on {cpu_model()}); the 1024-trajectory batch "
                         f"at this rate: {n_traj * cdt / done:.0f} s"}
    if rank == 0:
        line = {"metric": METRIC, "value": updates / dt, "unit": UNIT, "n_gpus": world, "steps": 1,
                "warmup": 1, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic",
                "config": {"workload": f"C5: {n_traj} depolarising trajectories, RQC 4x6 20 cycles, p=1e-3",
                           "n_qubits": 24, "trajectories": n_traj, "unique_simulations": unique,
                           "dedup": bool(args.dedup), "batch_clean": bc, "timing": "host wall clock around the batch"},
                "cpu_baseline": cpu, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)


def planner_options(args):
    """--tile/--regs/--low/--super for the traj and partial workloads (None = their defaults)."""
    if not (args.tile or args.regs or args.low or args.super):
        return None
    from paper_2008_07140_b200 import _native as N

    return N.options(tile_qubits=args.tile, reg_qubits=args.regs, low_qubits=args.low,
                     super_qubits=args.super)


PARTIAL = (6, 6, 12)  # partial-mode workload: n=36 RQC, cut 18


def partial_workload():
    from paper_2008_07140_b200 import workloads
    from paper_2008_07140_b200.partition import plan_partition
    from paper_2008_07140_b200.program import parse_program

    prog = parse_program(workloads.rqc_text(*PARTIAL, seed=SEED))
    n = prog.qubit_count
    cut = n // 2
    plan = plan_partition(prog, cut)
    rng = np.random.default_rng(SEED)
    targets = [format(int(i), f"0{n}b") for i in rng.integers(0, 1 << n, 256)]
    return prog, cut, plan, targets


def partial_updates(plan) -> float:
    """Amplitude-gate updates of the reference's 2*2^c branch sub-circuits
    (partition.py:96-140: every branch runs all non-crossing gates of its half,
    a projector per crossing gate and the target action where its bit is 1)."""
    n, cut, c = plan.qubit_count, plan.cut, plan.c
    size = {"lower": float(1 << cut), "upper": float(1 << (n - cut))}
    where = {cg.position for cg in plan.crossing_gates}
    tot = 0.0
    for pos, inst in enumerate(plan.program.instructions):
        if inst.is_gate and pos not in where:
            tot += size["lower" if all(q < cut for q in inst.all_qubits()) else "upper"] * (1 << c)
    for cg in plan.crossing_gates:
        tot += size["lower" if cg.control < cut else "upper"] * (1 << c)
        tot += size["lower" if cg.target < cut else "upper"] * (1 << (c - 1))
    return tot


def run_partial_bench(args) -> None:
    """Partial-amplitude mode (reference partition.py:151-192): 256 amplitudes of an
    n=36 RQC cut at qubit 18.  The metric counts the reference's branch
    sub-circuit work (2^c branches x both halves); each step is one full
    `run_partial` call through the public API (program in, amplitudes out on the
    host, device states allocated, run and freed inside the step)."""
    import torch

    from paper_2008_07140_b200.partition import batch_bits, decompose_crossing, run_partial

    rank, _, local = dist_env()
    torch.cuda.set_device(local)
    prog, cut, plan, targets = partial_workload()
    work = partial_updates(plan)
    popts = planner_options(args)
    for _ in range(args.warmup):
        run_partial(prog, cut, targets, device=local, options=popts)
    # the first call's kernels compile in the background (interpreted meanwhile): the timed
    # calls are warm
    from paper_2008_07140_b200 import _native as N

    N.check(N.lib().qsv_jit_wait())
    run_partial(prog, cut, targets, device=local, options=popts)
    torch.cuda.synchronize()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            run_partial(prog, cut, targets, device=local, options=popts)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
    dt = statistics.median(times)
    cb = batch_bits(plan)
    cpu = None
    if not args.no_cpu_baseline and rank == 0:
        from oracle import oracle as O

        threads = O.cpu_threads()
        done, t0 = 0.0, time.perf_counter()
        nb = 0
        for br in decompose_crossing(plan):
            for half in (br.lower_program, br.upper_program):
                O.run_full(half, workers=threads)
                done += len(half.instructions) * float(1 << half.qubit_count)
            nb += 1
            if time.perf_counter() - t0 >= args.cpu_seconds:
                break
        cdt = time.perf_counter() - t0
        cpu = {"value": done / cdt, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{nb} of {plan.branch_count} branches (both halves) through oracle run_full "
                         f"({cdt:.1f} s, {threads} threads)"}
    if rank == 0:
        line = {"metric": METRIC, "value": work / dt, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic",
                "config": {"workload": f"partial mode: RQC {PARTIAL[0]}x{PARTIAL[1]} {PARTIAL[2]} cycles, "
                                       f"n={plan.qubit_count}, cut {cut}, {len(targets)} targets",
                           "crossing_gates": plan.c, "branch_qubits": cb,
                           "half_states_qubits": [cut + cb, plan.qubit_count - cut + cb],
                           "reference_branch_updates": work,
                           "timing": "host wall clock around run_partial (public API, e2e)"},
                "e2e": {"value": work / dt, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 2 * len(targets) * (16 << cb)},
                "cpu_baseline": cpu, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)


NOISY = (4, 5, 20)  # general-channel trajectories: C1-shape RQC (n=20)


def run_noisy_bench(args) -> None:
    """General-channel noisy trajectories (noisy_batch.py): the C1-shape RQC
    (4x5, 20 cycles, n=20) under amplitude damping p=1e-3 on EVERY gate
    (state-dependent branch weights, reference noise.py:188-222), 1024 trajectories
    in one batched state.  Each step is one `run_noisy_batch` call through the
    public API; the metric counts trajectories x gates x 2^n."""
    import torch

    from paper_2008_07140_b200 import workloads
    from paper_2008_07140_b200.noise import make_noise_model
    from paper_2008_07140_b200.noisy_batch import run_noisy_batch
    from paper_2008_07140_b200.program import parse_program

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:  # replicas: each rank runs its B/world trajectories, no collective but the timing
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    prog = parse_program(workloads.rqc_text(*NOISY, seed=SEED))
    n = prog.qubit_count
    G = len(prog.gate_instructions())
    B = args.trajectories  # default 1024, as C5 (one 16 GiB batched state at n=20)
    kind, p = "ampdamp", 1e-3
    model = make_noise_model(kind, p)

    mine = range(rank * B // world, (rank + 1) * B // world)

    def once(step):
        rngs = [np.random.default_rng((SEED, step, t)) for t in mine]
        r = run_noisy_batch(prog, model, rngs, device=local)
        r.close()
        return r

    for w in range(args.warmup):
        once(10_000 + w)
    from paper_2008_07140_b200 import _native as N

    N.check(N.lib().qsv_jit_wait())  # background compiles of the first call done: timed calls are warm
    once(10_100)
    torch.cuda.synchronize()
    times = []
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            r = once(k)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
    if world > 1:  # max over ranks
        tt = torch.tensor(times, dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        times = tt.cpu().tolist()
    dt = statistics.median(times)
    work = float(B) * G * float(1 << n)
    cpu = None
    if not args.no_cpu_baseline and rank == 0:
        from oracle import oracle as O

        threads = O.cpu_threads()
        done, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < args.cpu_seconds:
            O.run_full(prog, np.random.default_rng(done), (kind, p), workers=threads)
            done += 1
        cdt = time.perf_counter() - t0
        cpu = {"value": done * G * float(1 << n) / cdt, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{done} trajectories through oracle run_full with ampdamp noise "
                         f"({cdt:.1f} s, {threads} threads; #Kraus + 2 state sweeps per noisy gate as "
                         f"reference noise.py:188-222)"}
    if rank == 0:
        line = {"metric": METRIC, "value": work / dt, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic",
                "config": {"workload": f"general-channel trajectories: RQC {NOISY[0]}x{NOISY[1]} "
                                       f"{NOISY[2]} cycles, n={n}, {kind} p={p} on every gate",
                           "trajectories": B, "gates": G, "noisy_steps": r.stats["noisy_steps"],
                           "step_ms": [round(t * 1e3, 1) for t in times],
                           "batched_state_gib": (B << n) * 16 / 2**30,
                           "timing": "host wall clock around run_noisy_batch (public API, e2e)"},
                "e2e": {"value": work / dt, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": None},
                "cpu_baseline": cpu, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def sharded_qubits(args, world: int) -> int:
    """Workload ladder.  Weak scaling (default): n_local = --local-qubits (30) on every
    GPU, n = n_local + log2 N - N = 1 is C2 itself.  Strong scaling (--strong): n =
    --qubits (32) on every N."""
    g = world.bit_length() - 1
    if args.strong:
        return args.qubits or 32
    return (args.local_qubits or N_BASE) + g


def run_sharded(args) -> None:
    """`bench.py --gpus N` under torchrun (N > 1): the state sharded over N GPUs by its
    top log2 N qubits (paper_2008_07140_b200/distributed.py), global<->local qubit
    swaps fused into the last pass's stores over CUDA-IPC-mapped peer memory (NVLink).
    Timed steps: set_basis(0) + the whole circuit, CUDA events on each rank's
    compute stream between barriers + synchronize, max over ranks.  One extra
    profiled step (after the timed region) gives the per-GPU HBM roofline and the
    exchange-out pass time; e2e = the same run through ShardedSimulator.run plus
    every rank's download of its shard into pinned host memory."""
    import torch
    import torch.distributed as dist

    from paper_2008_07140_b200 import _native as N
    from paper_2008_07140_b200.distributed import CudaShard, ShardedSimulator, make_transport
    from paper_2008_07140_b200.program import parse_program

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    # QSV_DIST_BACKEND=gloo (tests: several ranks sharing one GPU, which NCCL refuses);
    # the bookkeeping tensors then live on the host
    backend = os.environ.get("QSV_DIST_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        dist.init_process_group(backend)
    dev = f"cuda:{local}" if backend == "nccl" else "cpu"
    g = world.bit_length() - 1
    n = sharded_qubits(args, world)
    nl = n - g
    text = workloads_rqc(n, SEED)
    prog = parse_program(text)
    G = len(prog.gate_instructions())
    opts = N.options(tile_qubits=args.tile, reg_qubits=args.regs, low_qubits=args.low)
    shard = CudaShard(nl, local, options=opts)
    shard.reduce_device = dev
    kind = os.environ.get("QSV_TRANSPORT", "p2p")
    transport = make_transport(kind, dist, shard)
    sim = ShardedSimulator(n, shard, transport=transport)

    def step(stats=None):
        sim.set_basis(0)
        sim.run(prog, stats)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sim.stats.swaps.clear()
    timed = {}
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        ev0.record(shard.stream)
        for _ in range(args.steps):
            step(timed)
        ev1.record(shard.stream)
        torch.cuda.synchronize()
        dist.barrier()
    ms = torch.tensor([ev0.elapsed_time(ev1) / args.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_step = float(ms.item())
    swaps = list(sim.stats.swaps)
    # profiled step: per-launch times -> per-GPU HBM roofline and the exchange-out pass
    shard.options.profile = 1
    prof = {}
    step(prof)
    torch.cuda.synchronize()
    shard.options.profile = 0
    pk = peaks()
    mine = torch.tensor([prof.get("algorithmic_bytes", 0.0), prof.get("kernel_ms", 0.0),
                         float(timed.get("launches", 0))], dtype=torch.float64, device=dev)
    allr = [torch.zeros_like(mine) for _ in range(world)]
    dist.all_gather(allr, mine)
    per_gpu = [(float(a[0]) / (float(a[1]) / 1e3) / 1e9) if float(a[1]) > 0 else None for a in allr]
    xfer = {"swaps_per_step": len(swaps) / max(1, args.steps),
            "fused_exchanges_per_step": sum(x.fused for x in swaps) / max(1, args.steps),
            "swap_bytes_per_rank_per_step": sum(x.bytes_sent for x in swaps) / max(1, args.steps),
            "nvlink_peak_gbs": 900.0}
    lf = getattr(transport, "last_fused", None)
    if lf is not None:
        x_ms, others = lf
        t = torch.tensor([x_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sent = next((x.bytes_sent for x in reversed(swaps) if x.fused), None)
        if sent:
            gbs = sent / (float(t.item()) / 1e3) / 1e9
            xfer |= {"exchange_pass_ms": float(t.item()),
                     "other_pass_ms_median": statistics.median(others) if others else None,
                     "exchange_bytes_per_rank": sent, "nvlink_gbs_per_rank": gbs, "nvlink_frac": gbs / 900.0,
                     "nvlink_note": "remote bytes of the fused exchange-out pass / that pass's duration "
                                    "(the pass also computes: a lower bound on the link rate)"}
    elif kind == "p2p" and swaps and not all(x.fused for x in swaps):
        t = torch.tensor([transport.exchange_ms()], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        last = swaps[-1].bytes_sent
        xfer |= {"last_exchange_ms": float(t.item()), "last_exchange_bytes_per_rank": last,
                 "nvlink_gbs_per_rank": last / (float(t.item()) / 1e3) / 1e9,
                 "nvlink_frac": last / (float(t.item()) / 1e3) / 1e9 / 900.0}
    # end to end through the public API: run + every rank downloads its shard (pinned)
    e2e = None
    if not args.no_e2e:
        host = torch.empty(1 << nl, dtype=torch.complex128, pin_memory=True)
        times = []
        for _ in range(2):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            step()
            with torch.cuda.stream(shard.stream):
                host.copy_(shard.buf, non_blocking=True)
            shard.stream.synchronize()
            times.append(time.perf_counter() - t0)
        tt = torch.tensor([min(times)], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": G * float(1 << n) / float(tt.item()), "unit": UNIT, "ms_per_step": float(tt.item()) * 1e3,
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": (1 << nl) * 16 * world,
               "api": "ShardedSimulator.run(program) + every rank's shard -> pinned host (host wall clock, max over ranks)"}
        del host
    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        _, cprog = workload(N_BASE)
        cpu = cpu_reference_sample(cprog, min(args.cpu_seconds, 10.0))
        cpu.pop("seconds", None)
        cpu.pop("gates", None)
    dist.barrier()
    clocks = clk.summary()
    if rank == 0:
        ok = [x for x in per_gpu if x]
        line = {
            "metric": METRIC, "value": G * float(1 << n) / (ms_step / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic",
            "config": {"workload": (f"C3 {'strong' if args.strong else 'weak'} scaling: RQC n={n} on grid "
                                    f"{workloads_grid(n)}, 24 cycles, seed {SEED}"),
                       "n_qubits": n, "n_local": nl, "gates": G, "parallelism": f"sharded x{world} (top {g} qubits global)",
                       "transport": kind, "chunks": 1 << sim.chunk_log2, **xfer,
                       "l2": f"shard ({16 << nl >> 30} GiB) >> 126 MB L2: no flush needed"},
            "roofline": {"bound": "hbm", "achieved": statistics.mean(ok) if ok else None, "peak": pk["hbm_gbs"],
                         "unit": "GB/s", "frac": statistics.mean(ok) / pk["hbm_gbs"] if ok else None,
                         "per_gpu_gbs": per_gpu, "traffic": None, "peak_src": pk["src"],
                         "kernel": "qsv_pass (specialised fused pass, incl. exchange-out passes)",
                         "note": "per GPU: algorithmic bytes / event-timed kernel ms of one profiled step"},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(max(float(a[2]) for a in allr)),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    transport.close() if hasattr(transport, "close") else None
    dist.destroy_process_group()


def workloads_grid(n: int):
    from paper_2008_07140_b200 import workloads

    return workloads.grid_shape(n)


def run_gpu(args) -> None:
    rank, world, local = dist_env()
    if args.workload == "traj":
        run_traj(args)
        return
    if args.workload == "partial":
        run_partial_bench(args)
        return
    if args.workload == "noisy":
        run_noisy_bench(args)
        return
    if world > 1:
        run_sharded(args)
        return

    import torch

    from paper_2008_07140_b200 import _native as N
    from paper_2008_07140_b200 import statevector as SV

    torch.cuda.set_device(local)
    n = (args.qubits or 32) if args.strong else (args.qubits or N_BASE)
    text, prog = workload(n, args.workload)
    gates_list = prog.gate_instructions()
    G = len(gates_list)
    rec = SV.compile_gates(gates_list)
    L = N.lib()
    # RQC steps start from |0..0> (set_basis): the plan takes the product-state start
    # (leading single-qubit gates synthesised by the first pass), as qsv_run does for
    # run_full; the QFT round trip starts from an uploaded state
    product = 1 if (args.product and args.workload == "rqc" and not args.unfused and args.jit >= 0) else -1
    opts = N.options(fuse=not args.unfused, tile_qubits=args.tile, reg_qubits=args.regs,
                     low_qubits=args.low, profile=True, super_qubits=args.super, jit=args.jit,
                     product_start=product)

    stream = torch.cuda.Stream(device=local)
    state = SV.init_state(n, max_qubits=n, device=local, stream=stream.cuda_stream)
    plan = C.c_void_p()
    N.check(L.qsv_plan_create(rec.ctypes.data, len(rec), n, C.byref(opts), C.byref(plan)))
    info = N.qsv_plan_info()
    N.check(L.qsv_plan_summary(plan, C.byref(info)))

    psi0 = None
    if args.workload == "qft":
        from paper_2008_07140_b200 import workloads

        psi0 = workloads.gaussian_state(n, SEED)
        state.amplitudes = psi0

    def step(stats):
        if psi0 is None:
            state.set_basis(0)  # RQC starts from |0..0>; the QFT round trip maps psi0 back to psi0
        if args.unfused:
            N.check(L.qsv_run(state.handle, rec.ctypes.data, len(rec), C.byref(opts), C.byref(stats)))
        else:
            N.check(L.qsv_plan_execute(state.handle, plan, C.byref(opts), C.byref(stats)))

    for _ in range(args.warmup):
        step(N.qsv_run_stats())
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    stats = N.qsv_run_stats()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step(stats)
        ev1.record(stream)
        torch.cuda.synchronize()
    total_ms = ev0.elapsed_time(ev1)
    ms_step = total_ms / args.steps
    value = G * float(1 << n) / (ms_step / 1e3)

    # roofline of the dominant kernel (the fused pass kernel).  Algorithmic bytes
    # per launch as libqsv counts them: 2 x 16 x 2^n for a pass (read + write every
    # amplitude once), 16 x 2^n for the first pass after set_basis (it synthesises
    # |0..0> and only writes); unfused: 2 x 16 x 2^(n - #controls) per gate.
    # achieved = sum(bytes) / sum(event-timed launch ms) over the K timed steps
    # = mean bytes per launch / mean launch duration.
    launches = stats.launches
    avg_launch_ms = stats.kernel_ms / max(1, launches)
    pk = peaks()
    bytes_per_launch = stats.algorithmic_bytes / max(1, launches)
    achieved = bytes_per_launch / (avg_launch_ms / 1e3) / 1e9
    # per pass of the last timed step: ms, algorithmic bytes, HBM fraction and the
    # generator's FP64 instructions per amplitude (the heavy passes are FP64-issue
    # bound: against the measured DFMA rate)
    pass_ms, pass_bytes = N.last_launches(state.handle)
    per_pass, fp64_per_amp = [], 0.0
    for pi in range(len(pass_ms)):
        f = C.c_double(0.0)
        if not args.unfused:
            L.qsv_plan_pass_cost(plan, pi, C.byref(f))
            fp64_per_amp += f.value
        if args.unfused and pi >= 8:
            continue
        gbs = pass_bytes[pi] / (pass_ms[pi] / 1e3) / 1e9
        per_pass.append({"pass": pi, "ms": round(float(pass_ms[pi]), 3), "algorithmic_bytes": float(pass_bytes[pi]),
                         "hbm_gbs": round(gbs, 1), "hbm_frac": round(gbs / pk["hbm_gbs"], 3),
                         "fp64_per_amp": round(f.value, 1),
                         "fp64_frac": round(f.value * float(1 << n) / (pass_ms[pi] / 1e3) / 1e9 / FP64_PEAK_GINSTR, 3)})
    fp64_rate = fp64_per_amp * float(1 << n) / (ms_step / 1e3)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": pk["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / pk["hbm_gbs"], "traffic": None,
                "peak_src": pk["src"],
                "kernel": "qsv_pass (specialised fused pass)" if not args.unfused else "gate_kernel",
                "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_launch_ms,
                "kernel_share_of_step": stats.kernel_ms / total_ms,
                "per_pass": per_pass,
                "fp64": None if args.unfused else {
                    "instr_per_amplitude": fp64_per_amp, "achieved_ginstr_s": fp64_rate / 1e9,
                    "peak_ginstr_s": FP64_PEAK_GINSTR, "frac": fp64_rate / 1e9 / FP64_PEAK_GINSTR,
                    "peak_src": "scripts/fp64_pipes.cu: DFMA 36.1 TFLOP/s measured on B200 = 18.05e12 FP64 lane-instructions/s"}}

    # end to end through the public API: program text in, amplitudes out
    # (pinned host).  statevector.run_batch: every step parses the program,
    # plans/launches it and downloads the whole 2^n state; two device states
    # alternate so step i's download (PCIe) overlaps step i+1's simulation.
    e2e = None
    if not args.no_e2e:
        hosts = [torch.empty(1 << n, dtype=torch.complex128, pin_memory=True) for _ in range(2)]
        outs = [h.numpy() for h in hosts]
        states = [state, SV.init_state(n, max_qubits=n, device=local)]
        kw = dict(max_qubits=n, tile_qubits=args.tile, reg_qubits=args.regs, low_qubits=args.low, jit=args.jit,
                  fuse=not args.unfused, initial_state=psi0, device=local, states=states)
        SV.run_batch([text, text], outs, **kw)  # warm-up: plan cache, specialised kernels
        N.check(L.qsv_jit_wait())  # background compiles of the first call finished: the timed calls are warm
        SV.run_batch([text, text], outs, **kw)
        K = args.e2e_steps
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        SV.run_batch([text] * K, [outs[i % 2] for i in range(K)], **kw)
        torch.cuda.synchronize()
        e2e_t = (time.perf_counter() - t0) * 1e3 / K
        h2d = 0 if psi0 is None else psi0.nbytes
        e2e = {"value": G * float(1 << n) / (e2e_t / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": (1 << n) * 16, "ms_per_step": e2e_t, "steps": K,
               "api": "paper_2008_07140_b200.statevector.run_batch(program texts) -> pinned host amplitudes",
               "note": ("each step: parse + plan lookup + fused passes + full 2^n complex128 download; "
                        "gates reach the device as specialised-kernel code (cached per circuit), the "
                        "|0..0> input is synthesised by the first pass (no host buffer to copy); "
                        "downloads overlap the next step's passes (host wall clock over K steps)")}
        # COLD end to end: the first call on a circuit this process has never seen (same
        # C2 construction, another seed; the on-disk kernel cache is off, QSV_CACHE_DIR=0):
        # parse + look-ahead planning + kernel specialisation/NVRTC + passes + download
        if args.workload == "rqc" and not args.unfused:
            cold = []
            for k in range(args.cold_steps):
                ctext = workloads_rqc(n, SEED + 1000 + k)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = SV.run_batch([ctext], [outs[0]], **kw)
                torch.cuda.synchronize()
                cold.append((time.perf_counter() - t0) * 1e3)
                st = res[0].stats
                cold_plan = st.get("plan_ms", 0.0)
                cold_jit = st.get("jit_ms", 0.0)
                cold_compiled = st.get("compiled_passes", 0)
                N.check(L.qsv_jit_wait())
            cms = statistics.median(cold)
            e2e["cold"] = {"value": G * float(1 << n) / (cms / 1e3), "unit": UNIT, "ms_per_step": cms,
                           "ms_each": [round(c, 1) for c in cold], "plan_ms_last": cold_plan,
                           "jit_ms_last": cold_jit, "compiled_passes_last": cold_compiled,
                           "passes_last": st.get("passes", 0), "vs_warm": cms / e2e_t,
                           "h2d_bytes_per_step": 0, "d2h_bytes_per_step": (1 << n) * 16,
                           "note": "first run_batch call on an unseen circuit (C2 construction, seeds "
                                   f"{SEED + 1000}..{SEED + 999 + args.cold_steps}), QSV_CACHE_DIR=0: parse, "
                                   "planning, passes (compiled as their NVRTC compiles finish in the background, "
                                   "interpreted before), 16 GiB download"}
        states[1].close()
        del hosts, outs
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_reference_sample(prog, args.cpu_seconds)
        cpu.pop("seconds", None)
        cpu.pop("gates", None)

    clocks = clk.summary()
    L.qsv_plan_destroy(plan)
    state.close()
    if args.traffic == "auto" and not args.unfused:
        tr, why = ncu_traffic(args, len(pass_ms))
        if tr is None:
            roofline["traffic_note"] = why
        else:
            roofline["traffic"] = tr["mean"]
            roofline["traffic_src"] = tr["src"]
            for row, b, rd in zip(per_pass, tr["per_launch"], tr["read"]):
                row["dram_bytes"] = b
                row["dram_read_bytes"] = rd
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128 (f64)", "data": "synthetic",
        "config": {"workload": (f"C4: QFT + DAGGER-QFT round trip, n={n}, Gaussian state seed {SEED}"
                                if args.workload == "qft" else
                                f"C2: RQC {C2[0]}x{C2[1]} grid, {C2[2]} cycles, 8 CZ patterns, seed {SEED}"
                                if n == N_BASE else f"RQC n={n}"),
                   "n_qubits": n, "gates": G, "fused": not args.unfused, "passes": int(info.passes),
                   "stages": int(info.stages), "tile_qubits": int(info.tile_qubits),
                   "super_passes": int(info.super_passes), "super_qubits": int(info.super_qubits),
                   "reg_qubits": int(info.reg_qubits), "low_qubits": int(info.low_qubits),
                   "product_start": bool(info.product_start),
                   "l2": f"state ({16 << n >> 30} GiB) >> 126 MB L2: no flush needed", "parallelism": "single GPU"},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": int(launches),  # fused pass kernels (|0..0> is synthesised by the first pass)
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)


def main():
    # the on-disk kernel cache stays off in the bench: every specialised kernel of a
    # circuit is compiled by this process (the cold e2e number depends on it)
    os.environ.setdefault("QSV_CACHE_DIR", "0")
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--qubits", type=int, default=0, help="total qubits (N=1, or with --strong)")
    ap.add_argument("--local-qubits", type=int, default=0, help="weak scaling: qubits per GPU (default 30)")
    ap.add_argument("--strong", action="store_true", help="fixed total n (--qubits, default 32) for every N")
    ap.add_argument("--workload", default="rqc", choices=("rqc", "qft", "traj", "partial", "noisy"))
    ap.add_argument("--trajectories", type=int, default=1024)
    ap.add_argument("--dedup", action="store_true")
    ap.add_argument("--batch-clean", type=int, default=0,
                    help="traj: run error-free trajectories 2^b per (n+b)-qubit state (0 = one by one)")
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--regs", type=int, default=0)
    ap.add_argument("--low", type=int, default=0)
    ap.add_argument("--super", type=int, default=0, help="L2 super-tile qubits (0 = default)")
    ap.add_argument("--unfused", action="store_true")
    ap.add_argument("--jit", type=int, default=0, help="pass kernels: 0 auto, 1 specialised, -1 interpreted")
    ap.add_argument("--cold-steps", type=int, default=3)
    ap.add_argument("--product", type=int, default=1, help="1: product-state start for basis-state runs, 0: off")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-step-seconds", type=float, default=12.0)
    ap.add_argument("--no-qcsim", action="store_true", help="reference arm: skip the qcsim (numba) figure")
    ap.add_argument("--traffic", default="auto", choices=("auto", "off"),
                    help="auto: measure DRAM bytes per pass launch with an ncu child run of this workload")
    ap.add_argument("--traffic-timeout", type=float, default=240.0)
    args = ap.parse_args()
    if not args.product:
        os.environ["QSV_PRODUCT_START"] = "0"  # run_full / run_batch (qsv_run's automatic choice)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
