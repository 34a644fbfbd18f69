"""Sharded full-amplitude state across P = 2^g GPUs (one process per GPU).

Layout.  The state of n qubits is split by the top g
PHYSICAL index bits: rank r holds the 2^(n-g) amplitudes whose global bits
equal r, contiguously, in a device buffer driven by libqsv.  The reference has
no distributed mode (MPI is a SPEC.md:233 non-goal); the nearest analogue is
its cross-chunk ownership (statevector.py:5-8, 185-187), where a global qubit
plays the role of a chunk-index bit.

Two maps are kept on every rank:
* `dq`: logical qubit -> DATA qubit.  An uncontrolled SWAP moves no data: it
  exchanges two entries of `dq` (QFT's bit-reversal layer is free);
* `perm`: data qubit -> physical position; [0, n_local) are local positions,
  [n_local, n) global (rank bits).

Schedule.  libqsv's segment planner (`qsv_plan_segments`, C++) cuts the
gate stream into SEGMENTS that each run with one fixed set of n_local local
data qubits, taking every gate the set admits under the fused scheduler's
commutation rule (gates acting diagonally on a shared qubit commute); the set
changes only when no further gate fits (C3 random circuits: ONE exchange of
g qubits per circuit).  Within a segment:
* a control on a global qubit is a per-rank constant - the gate is skipped
  where it is 0 and the control dropped where it is 1 (cf. the reference's
  high-control chunk skip, statevector.py:170-172);
* a diagonal factor on a global qubit is a per-rank constant (cf. _k_scale,
  statevector.py:128-132);
* runs of local gates go to the native fused scheduler (`qsv_run`).

Exchange (global <-> local qubit swap), preferred form - FUSED into the
previous run's last pass (`P2PTransport.fused_exchange`, `qsv_run_exchange`):
that pass's kernel stores every output amplitude straight into the receive
buffer of the rank selected by its bits at the leaving qubits' positions
(remote stores over NVLink to CUDA-IPC-mapped peer memory), so the exchange
costs no extra HBM pass and overlaps the pass's math tile by tile; the
entering qubits take the leaving qubits' positions.  All ranks agree first
(it needs the specialised kernels on every rank).

Otherwise (copy form): leaving qubits V are first moved
(SWAP gates appended to the previous run - the fused planner turns them into
relabellings materialised by its last pass) onto the exchange positions
X = [n_local - c - s, n_local - c) just below the c CHUNK positions at the
top.  Chunk i (the contiguous quarter/eighth/... of the buffer with top bits
= i) is then exchanged as 2^s contiguous blocks with the 2^s ranks that differ
in the entering qubits' global bits, and the next segment's gates that do not
act non-diagonally on chunk positions (its PREFIX) run on chunk i as soon as
chunk i has arrived, while chunk i+1 is in flight.  Transports:
* `P2PTransport` - CUDA IPC mappings of the peers' buffers; the copy engines
  push every block straight into the peer's receive buffer over NVLink
  (no SM taken from the pass kernels), cross-process events order chunk i's
  arrival before its prefix on the compute stream;
* `AllToAllTransport` - `torch.distributed.all_to_all_single` per chunk
  (NCCL on GPUs; gloo on CPU tensors for the tests, or staged through host
  memory for GPU buffers under gloo).

The local engine is pluggable: `CudaShard` (libqsv on this rank's GPU, the
product path) or any object with the same methods (the gloo CPU tests plug
in the oracle).
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


def _is_plain_swap(u, controls) -> bool:
    return not controls and u.shape == (4, 4) and np.array_equal(u, gates.SWAP)


@dataclass
class SwapRecord:
    global_positions: tuple
    local_positions: tuple
    bytes_sent: int
    chunks: int = 1
    prefix_gates: int = 0
    fused: bool = False  # carried by the last pass's stores (qsv_run_exchange)


@dataclass
class ShardStats:
    swaps: list = field(default_factory=list)
    gate_runs: int = 0
    local_gates: int = 0
    skipped_gates: int = 0
    relabelled_swaps: int = 0
    placement_swaps: int = 0
    segments: int = 0


def plan_segments(items, n: int, n_local: int, local_mask: int, free_initial: bool):
    """libqsv segment planner over (u, targets, controls) items on DATA qubits.
    Returns (segment of every item, local data-qubit mask of every segment)."""
    from . import _native as N

    rec = N.gate_records(items)
    seg = np.zeros(max(1, len(rec)), dtype=np.int32)
    loc = np.zeros(max(1, len(rec)), dtype=np.uint64)
    ns = C.c_int64()
    N.check(N.lib().qsv_plan_segments(rec.ctypes.data, len(rec), n, n_local, C.c_uint64(local_mask),
                                      int(free_initial), seg.ctypes.data, loc.ctypes.data, C.byref(ns)))
    return seg[:len(rec)].tolist(), [int(x) for x in loc[:ns.value]]


class CudaShard:
    """This rank's 2^n_local amplitudes in device memory, driven by libqsv.

    Two equally sized buffers (torch tensors, so torch.distributed/NCCL can
    exchange them in place) alternate as state and receive buffer; libqsv
    wraps each (and each chunk of each) with `qsv_create_on` handles that all
    run on this shard's compute stream."""

    def __init__(self, n_local: int, device: int, stream=None, options=None):
        import torch

        from . import _native as N

        self.torch = torch
        self.N = N
        self.n_local = n_local
        self.device = device
        self.stream = stream or torch.cuda.Stream(device=device)
        self.options = options or N.options()
        self.bufs = [torch.zeros(1 << n_local, dtype=torch.complex128, device=f"cuda:{device}"),
                     torch.empty(1 << n_local, dtype=torch.complex128, device=f"cuda:{device}")]
        self.cur = 0  # index of the state buffer
        self._handles = {}  # (buffer, chunk_log2, chunk) -> qsv handle

    @property
    def buf(self):
        return self.bufs[self.cur]

    def handle(self, chunk=None):
        c, i = chunk if chunk else (0, 0)
        key = (self.cur, c, i)
        h = self._handles.get(key)
        if h is None:
            h = C.c_void_p()
            nsub = self.n_local - c
            ptr = self.buf.data_ptr() + (i << nsub) * 16
            self.N.check(self.N.lib().qsv_create_on(nsub, self.device, C.c_void_p(self.stream.cuda_stream),
                                                    C.c_void_p(ptr), C.byref(h)))
            self._handles[key] = h
        return h

    @property
    def h(self):
        return self.handle()

    def close(self):
        for h in self._handles.values():
            if h.value:
                self.N.lib().qsv_destroy(h)
        self._handles.clear()

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
        self.stream.synchronize()
        with self.torch.cuda.stream(self.stream):
            out = self.buf.cpu().numpy()
        return out

    def run(self, items, stats: dict | None = None, chunk=None):
        if not items:
            return
        rec = self.N.gate_records(items)
        st = self.N.qsv_run_stats()
        self.N.check(self.N.lib().qsv_run(self.handle(chunk), rec.ctypes.data, len(rec), C.byref(self.options),
                                          C.byref(st)))
        if stats is not None:
            for k, v in st.as_dict().items():
                stats[k] = stats.get(k, 0) + v

    def exchange_buffers(self):
        """(send, recv) float64 views for an all-to-all, ordered after the
        compute stream's pending work on the caller's current stream."""
        self.torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return (self.torch.view_as_real(self.bufs[self.cur]).reshape(-1),
                self.torch.view_as_real(self.bufs[1 - self.cur]).reshape(-1))

    def commit_exchange(self):
        """The receive buffer becomes the state (no synchronisation: later
        work is ordered by the transport's stream waits)."""
        self.cur = 1 - self.cur

    def norm_sq(self) -> float:
        out = C.c_double()
        self.N.check(self.N.lib().qsv_norm_sq(self.h, C.byref(out)))
        return out.value

    def pmeasure_local(self, positions) -> np.ndarray:
        q = np.asarray(positions, dtype=np.int32)
        table = np.empty(1 << q.size)
        self.N.check(self.N.lib().qsv_pmeasure(self.h, q.ctypes.data, int(q.size), table.ctypes.data))
        return table

    def prob_bit0(self, position: int) -> float:
        out = C.c_double()
        self.N.check(self.N.lib().qsv_prob_bit0(self.h, int(position), C.byref(out)))
        return out.value

    def collapse(self, position: int, outcome: int, scale: float):
        self.N.check(self.N.lib().qsv_collapse(self.h, int(position), int(outcome), float(scale)))

    def scale(self, s: float):
        self.N.check(self.N.lib().qsv_scale(self.h, float(s)))


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------


class AllToAllTransport:
    """One `all_to_all_single` per chunk: NCCL over NVLink for device buffers,
    gloo for CPU buffers (tests), or gloo staged through host memory."""

    def __init__(self, dist, group=None):
        self.dist = dist
        self.group = group
        self.gloo = dist.get_backend(group) == "gloo"

    def exchange(self, sim, G, chunk_log2, on_chunk):
        import torch

        shard = sim.shard
        s = len(G)
        nl = sim.n_local
        chunk = 2 << (nl - chunk_log2)  # float64 per chunk
        blk = chunk >> s
        gmask = sum(1 << (p - nl) for p in G)
        splits = [blk if (r & ~gmask) == (sim.rank & ~gmask) else 0 for r in range(sim.world)]
        send, recv = shard.exchange_buffers()
        stream = getattr(shard, "stream", None)
        on_device = send.device.type != "cpu"
        works = []
        for i in range(1 << chunk_log2):
            sl = slice(i * chunk, (i + 1) * chunk)
            if self.gloo and on_device:
                hs, hr = send[sl].cpu(), torch.empty(chunk, dtype=send.dtype)
                self.dist.all_to_all_single(hr, hs, output_split_sizes=splits, input_split_sizes=splits,
                                            group=self.group)
                recv[sl].copy_(hr)
                works.append(None)
            else:
                works.append(self.dist.all_to_all_single(recv[sl], send[sl], output_split_sizes=splits,
                                                         input_split_sizes=splits, group=self.group,
                                                         async_op=True))
        shard.commit_exchange()
        for i, w in enumerate(works):
            if w is not None:
                if on_device and stream is not None:
                    with torch.cuda.stream(stream):
                        w.wait()  # the compute stream waits for chunk i
                else:
                    w.wait()
            elif on_device and stream is not None:
                stream.wait_stream(torch.cuda.current_stream(send.device))
            on_chunk(i)


class P2PTransport:
    """Copy-engine pushes into CUDA-IPC-mapped peer buffers (NVLink P2P).

    Setup shares both buffers of every rank (qsv_ipc_mem_handle) and one
    interprocess event per chunk (torch.cuda.Event(interprocess=True)).  An
    exchange: wait until every rank's previous pushes completed (host
    barrier) so every receive buffer is free; push chunk by chunk on the copy
    stream, recording chunk i's event after its blocks; host barrier (every
    rank has ENQUEUED its records); the compute stream then waits for chunk i's
    events of all partner ranks before running the prefix on chunk i."""

    def __init__(self, dist, shard, group=None, max_chunk_log2: int = 3):
        import torch

        from . import _native as N

        self.dist, self.group, self.shard, self.N = dist, group, shard, N
        self.torch = torch
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.copy_stream = torch.cuda.Stream(device=shard.device)
        L = N.lib()
        mine = []
        for b in shard.bufs:
            hbuf = C.create_string_buffer(64)
            off = C.c_uint64()
            N.check(L.qsv_ipc_mem_handle(C.c_void_p(b.data_ptr()), hbuf, C.byref(off)))
            mine.append((hbuf.raw, off.value))
        self.events = [torch.cuda.Event(interprocess=True) for _ in range(1 << max_chunk_log2)]
        # recorded on the compute stream before an exchange: completes when this rank is
        # done with its receive buffer (last read by its previous exchange's sends)
        self.free_event = torch.cuda.Event(interprocess=True)
        ev_handles = [e.ipc_handle() for e in self.events]
        allh = [None] * self.world
        dist.all_gather_object(allh, (mine, ev_handles, self.free_event.ipc_handle()), group=group)
        self.peer_ptr = []  # [rank][buffer] -> device pointer (own buffers: local pointers)
        self.peer_events = []
        self.peer_free = []
        self._opened = []
        for r, (bufs, evh, freeh) in enumerate(allh):
            if r == self.rank:
                self.peer_ptr.append([b.data_ptr() for b in shard.bufs])
                self.peer_events.append(self.events)
                self.peer_free.append(self.free_event)
                continue
            self.peer_free.append(torch.cuda.Event.from_ipc_handle(shard.device, freeh))
            ptrs = []
            for raw, off in bufs:
                p = C.c_void_p()
                N.check(L.qsv_ipc_mem_open(raw, off, shard.device, C.byref(p)))
                self._opened.append(p)
                ptrs.append(p.value)
            self.peer_ptr.append(ptrs)
            self.peer_events.append([torch.cuda.Event.from_ipc_handle(shard.device, h) for h in evh])
        self.max_chunk_log2 = max_chunk_log2
        self.last_exchange_ms = 0.0
        self.last_fused = None  # (exchange-out pass ms, the run's other pass ms) when profiled
        self._t0 = torch.cuda.Event(enable_timing=True)
        self._t1 = torch.cuda.Event(enable_timing=True)

    def close(self):
        for p in self._opened:
            self.N.lib().qsv_ipc_mem_close(p)
        self._opened.clear()

    def exchange(self, sim, G, chunk_log2, on_chunk):
        torch, L = self.torch, self.N.lib()
        shard = self.shard
        assert chunk_log2 <= self.max_chunk_log2
        s, nl = len(G), sim.n_local
        gbits = [p - nl for p in G]
        gmask = sum(1 << b for b in gbits)
        my_g = sum(((self.rank >> b) & 1) << i for i, b in enumerate(gbits))
        chunk = 1 << (nl - chunk_log2)  # amplitudes
        blk = chunk >> s
        src_base = shard.bufs[shard.cur].data_ptr()
        spare = 1 - shard.cur
        partners = []
        for j in range(1 << s):
            peer = self.rank & ~gmask
            for i, b in enumerate(gbits):
                peer |= ((j >> i) & 1) << b
            partners.append(peer)
        self.copy_stream.wait_stream(shard.stream)  # this rank's send data is final
        self._wait_partners_free(self.copy_stream, partners)
        self._t0.record(self.copy_stream)
        for i in range(1 << chunk_log2):
            for j, peer in enumerate(partners):
                src = src_base + (i * chunk + j * blk) * 16
                dst = self.peer_ptr[peer][spare] + (i * chunk + my_g * blk) * 16
                self.N.check(L.qsv_copy_async(C.c_void_p(dst), C.c_void_p(src), blk * 16,
                                              C.c_void_p(self.copy_stream.cuda_stream)))
            self.events[i].record(self.copy_stream)
        self._t1.record(self.copy_stream)
        self.dist.barrier(group=self.group)  # every partner has enqueued its chunk events
        shard.commit_exchange()
        for i in range(1 << chunk_log2):
            for peer in partners:
                shard.stream.wait_event(self.peer_events[peer][i])
            on_chunk(i)

    def fused_exchange(self, sim, run, vpos, G, stats=None) -> bool:
        """The global<->local swap FUSED into the run's last pass: its kernel
        stores every output amplitude straight into the partner rank's receive
        buffer over NVLink (qsv_run_exchange).  All ranks decide together (a
        rank whose last pass holds an exchanged position in its tile cannot
        fuse); False = nothing was run, the caller exchanges by copies."""
        torch, L, N = self.torch, self.N.lib(), self.N
        shard = self.shard
        rec = N.gate_records(run) if run else None
        ok = C.c_int(0)
        vmask = sum(1 << p for p in vpos)
        if run:
            N.check(L.qsv_exchange_fusable(shard.handle(), rec.ctypes.data, len(rec), C.byref(shard.options),
                                           C.c_uint64(vmask), C.byref(ok)))
        flag = torch.tensor([int(ok.value)], dtype=torch.int32,
                            device="cpu" if self.dist.get_backend(self.group) == "gloo" else f"cuda:{shard.device}")
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=self.group)
        if not int(flag.item()):
            return False
        nl = sim.n_local
        gbits = [p - nl for p in G]
        gmask = sum(1 << b for b in gbits)
        my_g = sum(((self.rank >> b) & 1) << i for i, b in enumerate(gbits))
        spare = 1 - shard.cur
        ex = N.qsv_exchange()
        ex.positions = vmask
        ex.self_bits = sum(((my_g >> i) & 1) << p for i, p in enumerate(vpos))
        partners = []
        for j in range(1 << len(G)):
            peer = self.rank & ~gmask
            for i, b in enumerate(gbits):
                peer |= ((j >> i) & 1) << b
            partners.append(peer)
            ex.dst[j] = self.peer_ptr[peer][spare]
        # the partners' receive buffers are free once their streams pass their free
        # events (no host synchronisation: only event waits on the compute stream)
        self._wait_partners_free(shard.stream, partners)
        st = N.qsv_run_stats()
        rc = L.qsv_run_exchange(shard.handle(), rec.ctypes.data, len(rec), C.byref(shard.options), C.byref(ex),
                                C.byref(st))
        if rc == 0:
            self.events[0].record(shard.stream)
            if shard.options.profile:
                ms, _ = N.last_launches(shard.handle())
                self.last_fused = (float(ms[-1]), [float(x) for x in ms[:-1]])
        # the status vote doubles as the barrier after which every partner's event
        # record has been enqueued; a failure on any rank raises on every rank
        good = torch.tensor([int(rc == 0)], dtype=torch.int32,
                            device="cpu" if self.dist.get_backend(self.group) == "gloo" else f"cuda:{shard.device}")
        self.dist.all_reduce(good, op=self.dist.ReduceOp.MIN, group=self.group)
        if not int(good.item()):
            N.check(rc, shard.handle())
            raise RuntimeError("fused exchange failed on another rank; the sharded state is invalid")
        if stats is not None:
            for k, v in st.as_dict().items():
                stats[k] = stats.get(k, 0) + v
        shard.commit_exchange()
        for peer in partners:
            shard.stream.wait_event(self.peer_events[peer][0])
        return True

    def _wait_partners_free(self, stream, partners):
        """`stream` waits until every partner is done with the receive buffer this
        exchange writes into: each rank records its free event on its compute stream
        (after all its work so far, including copy-stream pushes), a host barrier makes
        every record visible, then the waits are enqueued."""
        shard = self.shard
        shard.stream.wait_stream(self.copy_stream)
        self.free_event.record(shard.stream)
        self.dist.barrier(group=self.group)
        for peer in partners:
            if peer != self.rank:
                stream.wait_event(self.peer_free[peer])

    def exchange_ms(self) -> float:
        """Copy-stream time of the last exchange (this rank's pushes)."""
        self._t1.synchronize()
        return self._t0.elapsed_time(self._t1)


# ---------------------------------------------------------------------------
# the sharded simulator
# ---------------------------------------------------------------------------


class ShardedSimulator:
    """Runs expanded gate streams on a state sharded over a process group."""

    def __init__(self, n: int, shard, group=None, rank: int | None = None, world: int | None = None,
                 chunk_log2: int | None = None, transport=None):
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
        if chunk_log2 is None:
            chunk_log2 = int(os.environ.get("QSV_SWAP_CHUNKS_LOG2", "2" if self.n_local >= 16 else "0"))
        self.chunk_log2 = chunk_log2
        self.transport = transport or AllToAllTransport(dist, group)
        self.fuse_exchange = os.environ.get("QSV_FUSED_EXCHANGE", "1") != "0"
        self.dq = list(range(n))    # logical -> data qubit
        self.perm = list(range(n))  # data qubit -> physical position
        self._basis = None          # pending basis index (layout still free)
        self.stats = ShardStats()

    # -- bookkeeping ----------------------------------------------------------
    def _rank_bit(self, phys: int) -> int:
        return (self.rank >> (phys - self.n_local)) & 1

    def _occupant(self, phys: int) -> int:
        return self.perm.index(phys)

    def _local_mask(self) -> int:
        return sum(1 << q for q in range(self.n) if self.perm[q] < self.n_local)

    def set_basis(self, index: int = 0):
        """|index> (logical basis index).  Materialised lazily: a basis state
        fits any layout, so the first segment picks its local qubits freely."""
        self.dq = list(range(self.n))
        self.perm = list(range(self.n))
        self._basis = index

    def upload_local(self, host_slice: np.ndarray):
        """This rank's slice of a logical-order state (identity layout)."""
        self.dq = list(range(self.n))
        self.perm = list(range(self.n))
        self._basis = None
        self.shard.upload(host_slice)

    def _materialize(self):
        if self._basis is None:
            return
        phys = 0
        for q in range(self.n):  # logical q = data q right after set_basis
            if (self._basis >> q) & 1:
                phys |= 1 << self.perm[q]
        nl = self.n_local
        self.shard.set_basis(phys & ((1 << nl) - 1) if (phys >> nl) == self.rank else None)
        self._basis = None

    # -- localisation -----------------------------------------------------------
    def _localise(self, item, chunk=None):
        """Map one gate on physical positions onto this shard (or onto chunk
        `chunk` = (c, i) of it), or None when it is a no-op here.  Positions at or
        above the view's size are fixed bits: chunk bits, then rank bits."""
        u, pt, pc = item
        nv = self.n_local - (chunk[0] if chunk else 0)

        def fixed(p):
            if p >= self.n_local:
                return self._rank_bit(p)
            return (chunk[1] >> (p - nv)) & 1

        ctl = []
        for p in pc:
            if p >= nv:
                if not fixed(p):
                    return None  # a fixed control is 0 here
            else:
                ctl.append(p)
        glob = [i for i, p in enumerate(pt) if p >= nv]
        if not glob:
            return (u, tuple(pt), tuple(ctl))
        if not _is_diag(u):
            raise AssertionError("non-diagonal gate on a fixed qubit must be exchanged in first")
        d = np.diag(u)
        anchor = next(q for q in range(nv) if q not in ctl)
        if len(pt) == 1:
            f = d[fixed(pt[0])]
            return None if f == 1 else (np.diag([f, f]), (anchor,), tuple(ctl))
        b = [fixed(p) if p >= nv else None for p in pt]
        if len(glob) == 2:
            f = d[2 * b[0] + b[1]]
            return None if f == 1 else (np.diag([f, f]), (anchor,), tuple(ctl))
        if glob == [0]:  # first target (matrix MSB) fixed
            return (np.diag([d[2 * b[0]], d[2 * b[0] + 1]]), (pt[1],), tuple(ctl))
        return (np.diag([d[b[1]], d[2 + b[1]]]), (pt[0],), tuple(ctl))

    def _physical(self, item):
        u, t, c = item
        return (u, tuple(self.perm[q] for q in t), tuple(self.perm[q] for q in c))

    def _flush(self, run, stats):
        self.shard.run(run, stats)
        self.stats.gate_runs += bool(run)

    # -- the global <-> local qubit swap ------------------------------------------
    def _transition(self, new_local: int, seg_items, run, stats):
        """Exchange into local set `new_local`; returns the segment's gates not
        already run on the chunks (the part after its prefix)."""
        nl = self.n_local
        E = [q for q in range(self.n) if (new_local >> q) & 1 and self.perm[q] >= nl]
        V = [q for q in range(self.n) if not (new_local >> q) & 1 and self.perm[q] < nl]
        s = len(E)
        if hasattr(self.transport, "fused_exchange") and self.fuse_exchange:
            vpos = sorted(self.perm[v] for v in V)
            G = sorted(self.perm[e] for e in E)
            if self.transport.fused_exchange(self, run, vpos, G, stats):
                self.stats.gate_runs += bool(run)
                for gp, vp in zip(G, vpos):  # bit i at vpos[i] <-> the partner's global bit G[i]
                    a, b = self._occupant(gp), self._occupant(vp)
                    self.perm[a], self.perm[b] = vp, gp
                self.stats.swaps.append(SwapRecord(tuple(G), tuple(vpos), 16 * (1 << nl) * ((1 << s) - 1) >> s, 0,
                                                   0, True))
                return seg_items
        c = max(0, min(self.chunk_log2, nl - s - 2))
        X = list(range(nl - c - s, nl - c))
        # leaving qubits onto the exchange positions (SWAPs fused into the run)
        for v in V:
            if self.perm[v] in X:
                continue
            x = next(p for p in X if self._occupant(p) not in V)
            w = self._occupant(x)
            run.append((gates.SWAP, (self.perm[v], x), ()))
            self.perm[v], self.perm[w] = x, self.perm[v]
            self.stats.placement_swaps += 1
        self._flush(run, stats)
        G = sorted(self.perm[e] for e in E)
        Xs = sorted(self.perm[v] for v in V)
        assert Xs == X
        for gp, xp in zip(G, X):  # bit i of the block index <-> bit i of the partner's global index
            a, b = self._occupant(gp), self._occupant(xp)
            self.perm[a], self.perm[b] = xp, gp
        # prefix: gates of the segment that never act non-diagonally on chunk positions
        nv = nl - c
        prefix, rest = [], []
        bN = bD = 0
        for it in seg_items:
            u, pt, pc = self._physical(it)
            diag = _is_diag(u)
            nmask = 0 if diag else sum(1 << p for p in pt)
            dmask = sum(1 << p for p in pc) | (sum(1 << p for p in pt) if diag else 0)
            blocked = ((nmask | dmask) & bN) or (nmask & bD)
            if c and not blocked and not any(p >= nv for p in (pt if not diag else ())):
                prefix.append((u, pt, pc))
            else:
                rest.append(it)
                bN |= nmask
                bD |= dmask

        def on_chunk(i):
            items = [x for x in (self._localise(p, (c, i)) for p in prefix) if x is not None]
            self.shard.run(items, stats, chunk=(c, i))

        self.transport.exchange(self, G, c, on_chunk)
        self.stats.swaps.append(SwapRecord(tuple(G), tuple(X), 16 * (1 << nl) * ((1 << s) - 1) >> s, 1 << c,
                                           len(prefix)))
        return rest

    # -- gate stream ------------------------------------------------------------
    def run(self, program, stats: dict | None = None, rng=None):
        """Execute an expanded Program: gates (segment-planned, fused), and the
        readouts PMEASURE (table appended to `self.tables`) and MEASURE
        (collapse, bit into `self.cregs`; `rng` lives on rank 0, which draws
        and broadcasts the outcome - the reference draws on its coordinator,
        statevector.py:304)."""
        self.cregs = [0] * program.creg_count
        self.tables = []
        items = []
        for inst in program.instructions:
            if inst.name in ("PMEASURE", "MEASURE"):
                self._run_items(items, stats)
                items = []
                if inst.name == "PMEASURE":
                    self.tables.append((inst.qubits, self.pmeasure(inst.qubits)))
                else:
                    self.cregs[inst.creg] = self.measure(inst.qubits[0], rng, inst.line)
                continue
            if not inst.is_gate:
                raise UnsupportedGate(f"{inst.name} is not supported on a sharded state", inst.line)
            u, targets, controls = gates.controlled_form(inst)
            if len(targets) > 2:
                raise UnsupportedGate(f"{inst.name} targets {targets}", inst.line)
            u = np.asarray(u, dtype=np.complex128)
            if _is_plain_swap(u, controls):
                a, b = targets
                self.dq[a], self.dq[b] = self.dq[b], self.dq[a]
                self.stats.relabelled_swaps += 1
                continue
            items.append((u, tuple(self.dq[t] for t in targets), tuple(self.dq[c] for c in controls)))
        self._run_items(items, stats)

    def _run_items(self, items, stats=None):
        """Gates on DATA qubits: segment planning, exchanges, fused local runs."""
        if not items:
            self._materialize()
            return
        free = self._basis is not None
        seg, seg_local = plan_segments(items, self.n, self.n_local, self._local_mask(), free)
        if free:
            # qubits leaving at the first exchange sit at the TOP local positions:
            # outside the forced low tile qubits, so the exchange can ride on the
            # last pass's stores (fused exchange)
            nxt = seg_local[1] if len(seg_local) > 1 else seg_local[0]
            loc = [q for q in range(self.n) if (seg_local[0] >> q) & 1 and (nxt >> q) & 1]
            loc += [q for q in range(self.n) if (seg_local[0] >> q) & 1 and not (nxt >> q) & 1]
            glo = [q for q in range(self.n) if not (seg_local[0] >> q) & 1]
            for p, q in enumerate(loc + glo):
                self.perm[q] = p
        self._materialize()
        by_seg = [[] for _ in seg_local]
        for it, k in zip(items, seg):
            by_seg[k].append(it)
        self.stats.segments += len(seg_local)
        run = []
        for k, seg_items in enumerate(by_seg):
            if seg_local[k] != self._local_mask():
                seg_items = self._transition(seg_local[k], seg_items, run, stats)
                run = []
            for it in seg_items:
                loc_it = self._localise(self._physical(it))
                if loc_it is None:
                    self.stats.skipped_gates += 1
                    continue
                run.append(loc_it)
                self.stats.local_gates += 1
        self._flush(run, stats)

    # -- readout ----------------------------------------------------------------
    def _allreduce(self, values) -> np.ndarray:
        import torch

        v = torch.tensor(np.asarray(values, dtype=np.float64), device=getattr(self.shard, "reduce_device", "cpu"))
        self.dist.all_reduce(v, group=self.group)
        return v.cpu().numpy()

    def pmeasure(self, qubits) -> np.ndarray:
        """Probability table over logical `qubits` (first listed = MSB,
        statevector.py:311-328): each rank tabulates its shard over the probe
        qubits that are local (global ones are fixed by its rank bits), the
        tables are summed over ranks."""
        self._materialize()
        M = len(qubits)
        pos = [self.perm[self.dq[q]] for q in qubits]
        loc = [i for i, p in enumerate(pos) if p < self.n_local]
        fixed = sum(self._rank_bit(p) << (M - 1 - i) for i, p in enumerate(pos) if p >= self.n_local)
        part = self.shard.pmeasure_local([pos[i] for i in loc]) if loc else np.array([self.shard.norm_sq()])
        full = np.zeros(1 << M)
        for kl in range(len(part)):
            key = fixed
            for j, i in enumerate(loc):  # bit j of kl (MSB first over loc) -> probe bit i
                if (kl >> (len(loc) - 1 - j)) & 1:
                    key |= 1 << (M - 1 - i)
            full[key] = part[kl]
        return self._allreduce(full)

    def measure(self, qubit: int, rng, line: int = 0) -> int:
        """MEASURE (statevector.py:298-308): global bit-0 probability, outcome
        drawn on rank 0 and broadcast, collapse + renormalisation per rank."""
        import torch

        from .errors import DegenerateState

        import torch as _t

        # the stream lives on rank 0; every rank learns whether it is there before any
        # collective, so a missing stream raises everywhere instead of hanging the others
        has = _t.tensor([int(rng is not None)], dtype=_t.int64, device=getattr(self.shard, "reduce_device", "cpu"))
        self.dist.broadcast(has, src=0, group=self.group)
        if not int(has.item()):
            raise UnsupportedGate("MEASURE needs a random stream", line)
        self._materialize()
        p = self.perm[self.dq[qubit]]
        norm = self.shard.norm_sq()
        if p < self.n_local:
            p0 = self.shard.prob_bit0(p)
        else:
            p0 = norm if self._rank_bit(p) == 0 else 0.0
        p0, tot = self._allreduce([p0, norm])
        p1 = tot - p0
        if p0 < 1e-12 and p1 < 1e-12:
            raise DegenerateState(f"both outcomes of qubit {qubit} have ~zero probability")
        out = torch.tensor([0], dtype=torch.int64, device=getattr(self.shard, "reduce_device", "cpu"))
        if self.rank == 0:
            out[0] = 0 if rng.random() < p0 else 1
        self.dist.broadcast(out, src=0, group=self.group)
        outcome = int(out.item())
        scale = 1.0 / math.sqrt(p0 if outcome == 0 else p1)
        if p < self.n_local:
            self.shard.collapse(p, outcome, scale)
        else:
            self.shard.scale(scale if self._rank_bit(p) == outcome else 0.0)
        return outcome

    def norm_sq(self) -> float:
        import torch

        self._materialize()
        v = torch.tensor([self.shard.norm_sq()], dtype=torch.float64,
                         device=getattr(self.shard, "reduce_device", "cpu"))
        self.dist.all_reduce(v, group=self.group)
        return float(v.item())

    def gather_amplitudes(self) -> np.ndarray | None:
        """All 2^n amplitudes in LOGICAL order on rank 0 (None elsewhere)."""
        import torch

        self._materialize()
        # complex128 travels as float64 pairs (gloo/NCCL reductions are real)
        local = torch.from_numpy(self.shard.download().copy().view(np.float64))
        dev = getattr(self.shard, "reduce_device", "cpu")
        local = local.to(dev)
        parts = [torch.empty_like(local) for _ in range(self.world)] if self.rank == 0 else None
        self.dist.gather(local, parts, dst=0, group=self.group)
        if self.rank != 0:
            return None
        phys = torch.cat(parts).cpu().numpy().view(np.complex128)  # index = rank << n_local | local
        idx = np.arange(1 << self.n, dtype=np.int64)
        src = np.zeros_like(idx)
        for q in range(self.n):  # logical bit q lives at physical position perm[dq[q]]
            src |= ((idx >> q) & 1) << self.perm[self.dq[q]]
        return phys[src]


def make_transport(kind: str, dist, shard, group=None):
    if kind == "p2p":
        return P2PTransport(dist, shard, group)
    return AllToAllTransport(dist, group)
