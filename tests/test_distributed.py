"""Sharded layout (paper_2008_07140_b200/distributed.py) over gloo, CPU only.

Every rank runs the product host logic - logical->physical qubit map,
per-rank handling of controls/diagonals on global qubits, the global<->local
qubit swap as an all-to-all of contiguous blocks (torch.distributed) - with
the local gate runs executed by the oracle instead of libqsv (no GPU here).
Rank 0 gathers the amplitudes in logical order and compares with the oracle
on the unsharded state."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2008_07140_b200 import workloads
from paper_2008_07140_b200.distributed import ShardedSimulator
from paper_2008_07140_b200.program import parse_program


class OracleShard:
    """Local engine for the CPU tests: numpy buffer + the oracle's kernels."""

    def __init__(self, n_local):
        self.n_local = n_local
        self.buf = np.zeros(1 << n_local, dtype=np.complex128)
        self.spare = np.empty_like(self.buf)

    def set_basis(self, index):
        self.buf[:] = 0
        if index is not None:
            self.buf[index] = 1

    def upload(self, host):
        self.buf[:] = host

    def run(self, items, stats=None):
        st = O.OracleState(self.n_local, self.buf, 0)
        for u, t, c in items:
            O.apply_gate(st, u, t, c)

    def exchange_buffers(self):
        return torch.from_numpy(self.buf.view(np.float64)), torch.from_numpy(self.spare.view(np.float64))

    def commit_exchange(self):
        self.buf, self.spare = self.spare, self.buf

    def download(self):
        return self.buf.copy()

    def norm_sq(self):
        return float(np.vdot(self.buf, self.buf).real)


def _worker(rank, world, port, cases, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    results = {}
    try:
        for name, text, psi0_seed in cases:
            prog = parse_program(text)
            n = prog.qubit_count
            g = world.bit_length() - 1
            sim = ShardedSimulator(n, OracleShard(n - g))
            if psi0_seed is None:
                sim.set_basis(0)
            else:
                psi0 = workloads.gaussian_state(n, psi0_seed)
                nl = n - g
                sim.shard.upload(psi0[rank << nl:(rank + 1) << nl])
            sim.run(prog)
            amps = sim.gather_amplitudes()
            norm = sim.norm_sq()
            if rank == 0:
                results[name] = (amps, norm, len(sim.stats.swaps))
    finally:
        dist.destroy_process_group()
    if rank == 0:
        np.save(out_path, np.array([results], dtype=object), allow_pickle=True)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(world, cases, tmp_path):
    out = str(tmp_path / f"res{world}.npy")
    mp.spawn(_worker, args=(world, _free_port(), cases, out), nprocs=world, join=True)
    return np.load(out, allow_pickle=True)[0]


def _reference(text, seed):
    prog = parse_program(text)
    init = None if seed is None else workloads.gaussian_state(prog.qubit_count, seed)
    return O.run_full(prog, initial=init).state.amplitudes


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_matches_oracle(world, golden, tmp_path):
    cases = [
        ("rqc", workloads.rqc_for_qubits(10, 12, 3), None),
        ("qft", workloads.qft_text(9), 4),
        ("qft_rt", workloads.qft_text(8, round_trip=True), 5),
    ]
    for name in ("random0", "random3", "random6", "random9"):
        text = golden["random_programs"][name]["text"]
        if parse_program(text).qubit_count >= world.bit_length() + 2:
            cases.append((name, text, 6))
    res = _run(world, cases, tmp_path)
    for name, text, seed in cases:
        amps, norm, swaps = res[name]
        ref = _reference(text, seed)
        assert np.abs(amps - ref).max() <= 1e-12, (world, name)
        assert abs(norm - np.vdot(ref, ref).real) <= 1e-12
    assert res["rqc"][2] > 0  # global-qubit gates really exchanged blocks
