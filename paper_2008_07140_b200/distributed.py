"""Sharded full-amplitude state across P = 2^g GPUs (one process per GPU).

Layout.  The state of n logical qubits is split by the top g
PHYSICAL index bits: rank r holds the 2^(n-g) amplitudes whose global bits
equal r, contiguously, in a device buffer driven by libqsv.  A
logical->physical qubit map `perm` records where every logical qubit lives;
physical positions [0, n_local) are local, [n_local, n) are global (rank
bits).  The reference has no distributed mode (MPI is a SPEC.md:233
non-goal); the nearest analogue is its cross-chunk ownership
(statevector.py:5-8, 185-187), where a global qubit plays the role of a
chunk-index bit.

Per gate, on every rank:
* a control on a global qubit is a per-rank constant - the gate is skipped
  where it is 0 and the control dropped where it is 1 (cf. the reference's
  high-control chunk skip, statevector.py:170-172);
* a diagonal factor on a global qubit is a per-rank constant (cf. _k_scale,
  statevector.py:128-132): no communication;
* a non-diagonal target on a global qubit triggers a GLOBAL<->LOCAL QUBIT SWAP
  with the top local qubits: each rank cuts its buffer into 2^s contiguous
  blocks and exchanges them with the 2^s ranks that differ in the swapped
  global bits (all-to-all of contiguous blocks, NCCL over NVLink on the GPU
  path), after which `perm` is updated.

Runs of local gates between swaps go to the native fused scheduler (one
`qsv_run` per run).  The local engine is pluggable: `CudaShard` (libqsv on
this rank's GPU, the product path) or any object with the same methods (the
gloo CPU tests plug in the oracle).
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

from . import gates
from .errors import UnsupportedGate


def _is_diag(u) -> bool:
    return gates.is_diagonal(u)


@dataclass
class SwapRecord:
    global_positions: tuple
    local_positions: tuple
    bytes_sent: int
    seconds: float = 0.0


@dataclass
class ShardStats:
    swaps: list = field(default_factory=list)
    gate_runs: int = 0
    local_gates: int = 0
    skipped_gates: int = 0


class CudaShard:
    """This rank's 2^n_local amplitudes in device memory, driven by libqsv.

    The buffer is a torch tensor (so torch.distributed/NCCL can exchange it
    in place); libqsv wraps the same memory with `qsv_create_on`."""

    def __init__(self, n_local: int, device: int, stream=None, options=None):
        import torch

        from . import _native as N

        self.torch = torch
        self.N = N
        self.n_local = n_local
        self.device = device
        self.stream = stream or torch.cuda.Stream(device=device)
        self.options = options or N.options()
        self.buf = torch.zeros(1 << n_local, dtype=torch.complex128, device=f"cuda:{device}")
        self.spare = torch.empty_like(self.buf)
        self._wrap()

    def _wrap(self):
        h = C.c_void_p()
        self.N.check(self.N.lib().qsv_create_on(self.n_local, self.device, C.c_void_p(self.stream.cuda_stream),
                                                C.c_void_p(self.buf.data_ptr()), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            self.N.lib().qsv_destroy(self.h)
            self.h = C.c_void_p()

    def set_basis(self, index: int | None):
        """|index> restricted to this shard (None: all zeros)."""
        # torch work goes on the engine's stream, ordered with the libqsv kernels
        with self.torch.cuda.stream(self.stream):
            self.buf.zero_()
            if index is not None:
                self.buf[index] = 1.0

    def upload(self, host: np.ndarray):
        with self.torch.cuda.stream(self.stream):
            self.buf.copy_(self.torch.from_numpy(np.ascontiguousarray(host)))
        self.stream.synchronize()

    def download(self) -> np.ndarray:
        self.N.check(self.N.lib().qsv_synchronize(self.h))
        with self.torch.cuda.stream(self.stream):
            out = self.buf.cpu().numpy()
        return out

    def run(self, items, stats: dict | None = None):
        if not items:
            return
        rec = self.N.gate_records(items)
        st = self.N.qsv_run_stats()
        self.N.check(self.N.lib().qsv_run(self.h, rec.ctypes.data, len(rec), C.byref(self.options), C.byref(st)))
        if stats is not None:
            for k, v in st.as_dict().items():
                stats[k] = stats.get(k, 0) + v

    def exchange_buffers(self):
        """(send, recv) float64 views for an all-to-all; libqsv is drained first."""
        self.N.check(self.N.lib().qsv_synchronize(self.h))
        self.torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return self.torch.view_as_real(self.buf).reshape(-1), self.torch.view_as_real(self.spare).reshape(-1)

    def commit_exchange(self):
        """The receive buffer becomes the state."""
        self.torch.cuda.current_stream(self.device).synchronize()
        self.buf, self.spare = self.spare, self.buf
        self.close()
        self._wrap()

    def norm_sq(self) -> float:
        out = C.c_double()
        self.N.check(self.N.lib().qsv_norm_sq(self.h, C.byref(out)))
        return out.value


class ShardedSimulator:
    """Runs expanded gate streams on a state sharded over a process group."""

    def __init__(self, n: int, shard, group=None, rank: int | None = None, world: int | None = None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        g = int(round(math.log2(self.world)))
        if 1 << g != self.world:
            raise ValueError("the number of ranks must be a power of two")
        if n - g < 2:
            raise ValueError(f"{n} qubits cannot be sharded over {self.world} ranks")
        self.n, self.g, self.n_local = n, g, n - g
        self.shard = shard
        # gloo cannot exchange device tensors: stage the blocks through host memory
        self.stage_host = dist.get_backend(group) == "gloo"
        self.perm = list(range(n))  # logical qubit -> physical position
        self.stats = ShardStats()

    # -- bookkeeping ----------------------------------------------------------
    def _rank_bit(self, phys: int) -> int:
        return (self.rank >> (phys - self.n_local)) & 1

    def _logical_at(self, phys: int) -> int:
        return self.perm.index(phys)

    def set_basis(self, index: int = 0):
        """|index> (logical basis index) with the identity layout."""
        self.perm = list(range(self.n))
        local = index & ((1 << self.n_local) - 1)
        self.shard.set_basis(local if (index >> self.n_local) == self.rank else None)

    # -- the global <-> local qubit swap ------------------------------------------
    def swap_in(self, need_global: list[int], keep: set[int] = frozenset()):
        """Exchange global physical positions `need_global` with the top local
        positions (all-to-all of contiguous blocks within each 2^s-rank group)."""
        import time

        G = sorted(need_global)
        s = len(G)
        top = list(range(self.n_local - s, self.n_local))
        # a top local position holding a qubit the current gate needs locally is
        # first moved down with a local SWAP gate
        for p in top:
            lq = self._logical_at(p)
            if lq in keep:
                free = next(q for q in range(self.n_local - s - 1, -1, -1)
                            if self._logical_at(q) not in keep)
                self.shard.run([(gates.SWAP, (p, free), ())])
                lf = self._logical_at(free)
                self.perm[lq], self.perm[lf] = free, p
        chunk = 1 << (self.n_local - s)
        send, recv = self.shard.exchange_buffers()
        gbits = [q - self.n_local for q in G]
        mask = sum(1 << b for b in gbits)
        splits = []
        for r in range(self.world):
            splits.append(2 * chunk if (r & ~mask) == (self.rank & ~mask) else 0)
        t0 = time.perf_counter()
        if self.stage_host and send.device.type != "cpu":
            hs, hr = send.cpu(), send.new_empty(send.shape, device="cpu")
            self.dist.all_to_all_single(hr, hs, output_split_sizes=splits, input_split_sizes=splits,
                                        group=self.group)
            recv.copy_(hr)
        else:
            self.dist.all_to_all_single(recv, send, output_split_sizes=splits, input_split_sizes=splits,
                                        group=self.group)
        self.shard.commit_exchange()
        dt = time.perf_counter() - t0
        # physical positions G[i] <-> top[i] exchange their logical qubits
        for gp, lp in zip(G, top):
            a, b = self._logical_at(gp), self._logical_at(lp)
            self.perm[a], self.perm[b] = lp, gp
        self.stats.swaps.append(SwapRecord(tuple(G), tuple(top), 16 * chunk * ((1 << s) - 1), dt))

    # -- gate stream ------------------------------------------------------------
    def _localise(self, u, targets, controls):
        """Map one controlled-form gate onto this shard, or None when it is a
        no-op here.  Targets must already be local when the gate is not diagonal."""
        u = np.asarray(u, dtype=np.complex128)
        ctl = []
        for c in controls:
            pc = self.perm[c]
            if pc >= self.n_local:
                if not self._rank_bit(pc):
                    return None  # a global control is 0 on this rank
            else:
                ctl.append(pc)
        pt = [self.perm[t] for t in targets]
        glob = [i for i, p in enumerate(pt) if p >= self.n_local]
        if not glob:
            return (u, tuple(pt), tuple(ctl))
        if not _is_diag(u):
            raise AssertionError("non-diagonal gate on a global qubit must be swapped in first")
        d = np.diag(u)
        anchor = next(q for q in range(self.n_local) if q not in ctl)
        if len(pt) == 1:
            f = d[self._rank_bit(pt[0])]
            return None if f == 1 else (np.diag([f, f]), (anchor,), tuple(ctl))
        b = [self._rank_bit(p) if p >= self.n_local else None for p in pt]
        if len(glob) == 2:
            f = d[2 * b[0] + b[1]]
            return None if f == 1 else (np.diag([f, f]), (anchor,), tuple(ctl))
        if glob == [0]:  # first target (matrix MSB) global
            return (np.diag([d[2 * b[0]], d[2 * b[0] + 1]]), (pt[1],), tuple(ctl))
        return (np.diag([d[b[1]], d[2 + b[1]]]), (pt[0],), tuple(ctl))

    def run(self, program, stats: dict | None = None):
        """Apply every gate of an expanded Program (MEASURE / PMEASURE are
        not supported on the sharded path)."""
        batch = []
        for inst in program.instructions:
            if not inst.is_gate:
                raise UnsupportedGate(f"{inst.name} is not supported on a sharded state", inst.line)
            u, targets, controls = gates.controlled_form(inst)
            if len(targets) > 2:
                raise UnsupportedGate(f"{inst.name} targets {targets}", inst.line)
            if not _is_diag(u):
                need = [self.perm[t] for t in targets if self.perm[t] >= self.n_local]
                if need:
                    self.shard.run(batch, stats)
                    self.stats.gate_runs += bool(batch)
                    batch = []
                    self.swap_in(need, keep={t for t in targets})
            item = self._localise(u, targets, controls)
            if item is None:
                self.stats.skipped_gates += 1
                continue
            batch.append(item)
            self.stats.local_gates += 1
        self.shard.run(batch, stats)
        self.stats.gate_runs += bool(batch)

    # -- readout ----------------------------------------------------------------
    def norm_sq(self) -> float:
        import torch

        v = torch.tensor([self.shard.norm_sq()], dtype=torch.float64,
                         device="cpu" if self.stage_host else getattr(self.shard, "reduce_device", "cpu"))
        self.dist.all_reduce(v, group=self.group)
        return float(v.item())

    def gather_amplitudes(self) -> np.ndarray | None:
        """All 2^n amplitudes in LOGICAL order on rank 0 (None elsewhere)."""
        import torch

        # complex128 travels as float64 pairs (gloo/NCCL reductions are real)
        local = torch.from_numpy(self.shard.download().copy().view(np.float64))
        dev = "cpu" if self.stage_host else getattr(self.shard, "reduce_device", "cpu")
        local = local.to(dev)
        parts = [torch.empty_like(local) for _ in range(self.world)] if self.rank == 0 else None
        self.dist.gather(local, parts, dst=0, group=self.group)
        if self.rank != 0:
            return None
        phys = torch.cat(parts).cpu().numpy().view(np.complex128)  # index = rank << n_local | local
        idx = np.arange(1 << self.n, dtype=np.int64)
        src = np.zeros_like(idx)
        for q in range(self.n):  # logical bit q lives at physical position perm[q]
            src |= ((idx >> q) & 1) << self.perm[q]
        return phys[src]


def bench_main(args) -> None:
    """`bench.py --gpus N` under torchrun: weak-scaled RQC, n = 30 + log2(N)."""
    import json
    import time

    import torch
    import torch.distributed as dist

    from . import workloads
    from . import _native as N
    from .program import parse_program

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    g = int(round(math.log2(world)))
    n = (args.qubits or 30) + g
    prog = parse_program(workloads.rqc_for_qubits(n, 24, 0))
    G = len(prog.gate_instructions())
    shard = CudaShard(n - g, local, options=N.options(tile_qubits=args.tile, reg_qubits=args.regs,
                                                      low_qubits=args.low))
    shard.reduce_device = f"cuda:{local}"
    sim = ShardedSimulator(n, shard)

    def step():
        sim.set_basis(0)
        sim.run(prog)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sim.stats.swaps.clear()
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([ev0.elapsed_time(ev1) / args.steps], device=f"cuda:{local}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_step = float(ms.item())
    swaps = sim.stats.swaps
    swap_bytes = sum(s.bytes_sent for s in swaps) / max(1, args.steps)
    if rank == 0:
        line = {
            "metric": "amplitude-gate updates/s", "value": G * float(1 << n) / (ms_step / 1e3),
            "unit": "amp-gate/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c128 (f64)", "data": "synthetic",
            "config": {"workload": f"C3-style weak scaling: RQC n={n} on grid {workloads.grid_shape(n)}, 24 cycles",
                       "n_qubits": n, "n_local": n - g, "gates": G, "parallelism": f"sharded x{world}",
                       "swaps_per_step": len(swaps) / max(1, args.steps),
                       "swap_bytes_per_rank_per_step": swap_bytes},
            "gpu_launches": None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
