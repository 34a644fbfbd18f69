"""C5 replicas over ranks (trajectories.py), CPU only: two gloo ranks each run
their share of the trajectories (t = rank, rank + P, ...; no collective while
they run) and rank 0 gathers the per-trajectory probe tables, error counts,
norms and kept amplitudes (`gather_reports`).  The native steps run on the
numpy stand-in of libqsv (tests/fake_qsv.py); the gathered batch must equal a
single-process run and the oracle's reference noisy trajectories
(noise.py:188-222) for every trajectory id."""

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2008_07140_b200 import workloads
from paper_2008_07140_b200.program import parse_program

P = 0.05
N_TRAJ = 9
PROBE = (0, 3, 5)


def _program():
    return parse_program(workloads.rqc_text(2, 3, 6, seed=4))


def _run(rank, world, port, out):
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    from fake_qsv import FakeLib
    from paper_2008_07140_b200 import _native as N
    from paper_2008_07140_b200.trajectories import run_trajectories

    fake = FakeLib()
    N.lib = lambda: fake
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rep = run_trajectories(_program(), P, N_TRAJ, base_seed=3, probe_qubits=PROBE, keep=(1, 4), rank=rank,
                               world=world, streams=1)
        if rank == 0:
            np.save(out, np.array([rep], dtype=object), allow_pickle=True)
        else:
            assert rep.trajectories == list(range(rank, N_TRAJ, world))
    finally:
        dist.destroy_process_group()


def test_replica_split_gathers_on_rank0(tmp_path, monkeypatch):
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    from fake_qsv import FakeLib
    from paper_2008_07140_b200 import _native as N
    from paper_2008_07140_b200.trajectories import run_trajectories
    from paper_2008_07140_b200.workloads import trajectory_seed

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "rep.npy")
    mp.spawn(_run, args=(2, port, out), nprocs=2, join=True)
    got = np.load(out, allow_pickle=True)[0]
    fake = FakeLib()
    monkeypatch.setattr(N, "lib", lambda: fake)
    one = run_trajectories(_program(), P, N_TRAJ, base_seed=3, probe_qubits=PROBE, keep=(1, 4), streams=1)
    assert got.trajectories == list(range(N_TRAJ)) == one.trajectories
    assert got.errors == one.errors and sum(e > 0 for e in got.errors) >= 2
    assert np.abs(got.tables - one.tables).max() <= 1e-14
    assert got.gate_updates == one.gate_updates
    assert sorted(got.kept) == [1, 4]
    prog = _program()
    for t in range(N_TRAJ):
        ref = O.run_full(prog, np.random.default_rng(trajectory_seed(3, t)), noise=("depolarizing", P))
        assert np.abs(got.tables[t] - O.pmeasure(ref.state, PROBE)).max() <= 1e-12
        if t in got.kept:
            assert np.abs(got.kept[t] - ref.state.amplitudes).max() <= 1e-12
