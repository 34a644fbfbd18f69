"""GPU parity: the CUDA path (libqsv through its C ABI) vs the oracle and the
reference golden vectors.  Tolerances (north_star): max|d amplitude| <= 1e-10
and 1 - |<psi_ref|psi>| <= 1e-12 in complex128."""

import math

import numpy as np
import pytest

from conftest import program_text
from oracle import oracle as O
from paper_2008_07140_b200 import errors, gates, workloads
from paper_2008_07140_b200 import statevector as SV
from paper_2008_07140_b200.noise import make_noise_model
from paper_2008_07140_b200.program import parse_program

pytestmark = pytest.mark.gpu

ATOL = 1e-10
FID = 1e-12


def assert_parity(got, want):
    got = np.asarray(got)
    want = np.asarray(want)
    assert np.abs(got - want).max() <= ATOL
    ov = abs(np.vdot(want, got)) / math.sqrt(np.vdot(want, want).real * np.vdot(got, got).real)
    assert 1.0 - ov <= FID


CONFIGS = [dict(), dict(fuse=False), dict(tile_qubits=3, reg_qubits=2, low_qubits=1),
           dict(tile_qubits=5, reg_qubits=3, low_qubits=2), dict(tile_qubits=8, reg_qubits=4),
           dict(tile_qubits=6, reg_qubits=1), dict(jit=1), dict(jit=1, tile_qubits=5, reg_qubits=3, low_qubits=2)]


@pytest.mark.parametrize("cfg", CONFIGS)
def test_run_full_golden_programs(golden, golden_arrays, cfg):
    for name, rec in golden["runs"].items():
        prog = parse_program(program_text(golden, name))
        res = SV.run_full(prog, np.random.default_rng(rec["seed"]), **cfg)
        assert_parity(res.state.amplitudes, golden_arrays[f"run/{name}"])
        assert res.cregs == rec["cregs"], name
        for t_i, _ in enumerate(rec["tables"]):
            assert np.abs(res.tables[t_i][1] - golden_arrays[f"run/{name}/table{t_i}"]).max() <= 1e-12
        res.state.close()


def test_golden_table_appendix_a2(golden):
    res = SV.run_full(parse_program(golden["programs"]["golden"]["text"]))
    want = {0: 0.820082, 2: 0.106694, 4: 0.0549175, 6: 0.0183058}
    table = res.tables[0][1]
    for i in range(8):
        assert abs(table[i] - want.get(i, 0.0)) <= 1e-4


def test_kernel_api_streams(golden, golden_arrays):
    """apply_single_qubit / apply_controlled / apply_two_qubit / apply_projector (unfused kernels)."""
    for s_idx, rec in enumerate(golden["kernel_streams"]):
        st = SV.StateVector(rec["n"], golden_arrays[f"stream{s_idx}/psi0"], rec["chunk_log2"])
        for o_idx, op in enumerate(rec["ops"]):
            u = golden_arrays[f"stream{s_idx}/u{o_idx}"]
            if op["kind"] == "single":
                SV.apply_single_qubit(st, u, op["targets"][0])
            elif op["kind"] == "controlled":
                SV.apply_controlled(st, u, op["controls"], op["targets"][0])
            elif op["kind"] == "two":
                SV.apply_two_qubit(st, u, *op["targets"], controls=tuple(op["controls"]))
            else:
                SV.apply_projector(st, u, op["targets"][0])
        assert np.abs(st.amplitudes - golden_arrays[f"stream{s_idx}/final"]).max() <= ATOL
        st.close()


@pytest.mark.parametrize("n", [3, 6, 9])
def test_qft_random_state_golden(golden, golden_arrays, n):
    psi0 = golden_arrays[f"qft{n}/psi0"]
    for tag in ("forward", "round_trip"):
        res = SV.run_full(parse_program(golden["qft"][str(n)][tag]), initial_state=psi0)
        assert_parity(res.state.amplitudes, golden_arrays[f"qft{n}/{tag}"])


@pytest.mark.parametrize("engine", ["fused", "sequential"])
def test_reference_noise_semantics(golden, golden_arrays, engine):
    """run_full with a depolarising NoiseModel reproduces the reference trajectory
    (fused: batch-of-one noisy steps; sequential: weights pass + gate per noisy gate)."""
    for rec in golden["noise"]:
        res = SV.run_full(parse_program(rec["text"]), np.random.default_rng(rec["traj_seed"]),
                          make_noise_model("depolarizing", rec["p"]), noise_engine=engine)
        assert_parity(res.state.amplitudes, golden_arrays[rec["key"]])


def test_presampled_pauli_trajectories_match_reference(golden, golden_arrays):
    """BASELINE C5 semantics: explicit Pauli insertion + fused noiseless run."""
    for rec in golden["noise"]:
        prog = parse_program(rec["text"])
        traj = workloads.noisy_trajectory_program(prog, rec["p"], rec["traj_seed"])
        res = SV.run_full(traj)
        assert_parity(res.state.amplitudes, golden_arrays[rec["key"]])


@pytest.mark.parametrize("cfg", [dict(), dict(fuse=False), dict(tile_qubits=10, reg_qubits=3, low_qubits=4),
                                 dict(tile_qubits=13, reg_qubits=4), dict(jit=-1)])
def test_c1_twenty_qubits_vs_oracle(golden, golden_arrays, cfg):
    prog = parse_program(golden["c1"]["text"])
    res = SV.run_full(prog, **cfg)
    got = res.state.amplitudes
    idx = golden_arrays["c1/idx"]
    assert np.abs(got[idx] - golden_arrays["c1/amps"]).max() <= ATOL
    ref = O.run_full(prog, workers=O.cpu_threads())
    assert_parity(got, ref.state.amplitudes)
    assert np.abs(SV.pmeasure(res.state, (0, 7, 13, 19)) - golden_arrays["c1/pm_0_7_13_19"]).max() <= 1e-12


@pytest.mark.parametrize("n,depth,seed", [(22, 12, 1), (24, 20, 0)])
def test_rqc_vs_oracle_larger(n, depth, seed):
    prog = parse_program(workloads.rqc_for_qubits(n, depth, seed))
    ref = O.run_full(prog, workers=O.cpu_threads())
    for jit in (1, -1):
        res = SV.run_full(prog, jit=jit)
        assert_parity(res.state.amplitudes, ref.state.amplitudes)
        res.state.close()


def test_run_batch_overlapped_downloads():
    """run_batch (two device states, downloads overlapping the next run) returns
    the same amplitudes as run_full for each program, incl. a reused buffer."""
    import torch

    n = 18
    texts = [workloads.rqc_for_qubits(n, 10, s) for s in (1, 2, 3)]
    bufs = [torch.empty(1 << n, dtype=torch.complex128, pin_memory=True).numpy() for _ in range(2)]
    outs = [bufs[0], bufs[1], bufs[0]]
    res = SV.run_batch(texts, outs)
    assert all(r.amplitudes is outs[i] and r.state is None for i, r in enumerate(res))
    # buffers 0 and 1 hold programs 2 and 1 (program 0's result was overwritten in order)
    for i, buf in ((1, bufs[1]), (2, bufs[0])):
        ref = O.run_full(parse_program(texts[i]), workers=O.cpu_threads())
        assert_parity(buf, ref.state.amplitudes)
    with pytest.raises(ValueError):
        SV.run_batch(texts[:1], [np.zeros(4, np.complex128)])


def test_qft_round_trip_22():
    n = 22
    psi0 = workloads.gaussian_state(n, 11)
    fwd = SV.run_full(parse_program(workloads.qft_text(n)), initial_state=psi0)
    assert_parity(fwd.state.amplitudes, math.sqrt(1 << n) * np.fft.ifft(psi0))
    fwd.state.close()
    rt = SV.run_full(parse_program(workloads.qft_text(n, round_trip=True)), initial_state=psi0)
    assert_parity(rt.state.amplitudes, psi0)


def test_random_programs_all_configs(golden):
    rng = np.random.default_rng(5)
    for name, rec in golden["random_programs"].items():
        prog = parse_program(rec["text"])
        psi0 = workloads.gaussian_state(prog.qubit_count, int(rng.integers(1 << 30)))
        ref = O.run_full(prog, initial=psi0)
        for cfg in CONFIGS:
            res = SV.run_full(prog, initial_state=psi0, **cfg)
            assert_parity(res.state.amplitudes, ref.state.amplitudes)
            res.state.close()


def test_readouts():
    n = 12
    psi = workloads.gaussian_state(n, 4)
    st = SV.StateVector(n, psi)
    ref = O.OracleState(n, psi.copy(), 0)
    assert st.norm_sq() == pytest.approx(ref.norm_sq(), abs=1e-14)
    for k in (0, 5, 11):
        assert SV.probability_bit0(st, k) == pytest.approx(O.probability_bit0(ref, k), abs=1e-14)
    for qs in [(0,), (11, 0), (3, 7, 1), tuple(range(n - 1, -1, -1)), (2, 9, 4, 6, 0, 11, 8, 1, 5, 3, 10, 7)]:
        assert np.abs(SV.pmeasure(st, qs) - O.pmeasure(ref, qs)).max() <= 1e-14
    rho = st.reduced_density((3, 8))
    t = psi.reshape((2,) * n)
    sub = np.moveaxis(t, [n - 1 - 3, n - 1 - 8], [0, 1]).reshape(4, -1)
    assert np.abs(rho - sub @ sub.conj().T).max() <= 1e-14
    other = SV.StateVector(n, psi * np.exp(0.3j))
    assert st.inner(other) == pytest.approx(np.exp(0.3j), abs=1e-13)
    assert st.max_abs_diff(other) == pytest.approx(np.abs(psi * np.exp(0.3j) - psi).max(), abs=1e-15)


def test_measure_collapse_and_statistics():
    rng = np.random.default_rng(1)
    st = SV.StateVector(2, np.array([1, 0, 0, 1], dtype=complex) / math.sqrt(2))
    bit = SV.measure(st, 0, rng)
    want = np.zeros(4)
    want[3 * bit] = 1
    assert np.abs(st.amplitudes - want).max() <= 1e-15
    ones = 0
    rng = np.random.default_rng(42)
    for _ in range(2000):
        st.amplitudes = np.array([1, 1, 0, 0], dtype=complex) / math.sqrt(2)
        ones += SV.measure(st, 0, rng)
    assert abs(ones - 1000) < 3 * math.sqrt(500)
    st.amplitudes = np.zeros(4, dtype=complex)
    with pytest.raises(errors.DegenerateState):
        SV.measure(st, 0, rng)


def test_errors_and_ceiling():
    with pytest.raises(errors.TooManyQubits):
        SV.init_state(31)
    with pytest.raises(errors.TooManyQubits):
        SV.init_state(0)
    st = SV.init_state(3)
    with pytest.raises(errors.ParseError):
        SV.apply_single_qubit(st, gates.H, 7)
    assert np.array_equal(SV.init_state(3).amplitudes, [1, 0, 0, 0, 0, 0, 0, 0])


def test_trajectories_vs_oracle():
    """C5 semantics on a small grid with many errors: every trajectory equals the
    oracle running the reference noisy-gate rule with the same seed."""
    from paper_2008_07140_b200.noise import make_noise_model
    from paper_2008_07140_b200.trajectories import run_trajectories
    from paper_2008_07140_b200.workloads import trajectory_seed

    prog = parse_program(workloads.rqc_text(3, 4, 8, seed=2))
    keep = tuple(range(12))
    rep = run_trajectories(prog, 0.05, 12, base_seed=7, probe_qubits=(0, 5, 11), keep=keep)
    assert sum(e > 0 for e in rep.errors) >= 3
    for t in keep:
        ref = O.run_full(prog, np.random.default_rng(trajectory_seed(7, t)), noise=("depolarizing", 0.05))
        assert_parity(rep.kept[t], ref.state.amplitudes)
        assert np.abs(rep.tables[t] - O.pmeasure(ref.state, (0, 5, 11))).max() <= 1e-12


@pytest.mark.slow
def test_trajectories_full_size_c5():
    """BASELINE C5 shape (n=24, 4x6, 20 cycles, p=1e-3): 16 trajectories of the
    1024-trajectory batch - 8 error-free and the first 8 that drew errors - vs the
    oracle running the same explicit-Pauli programs (the replay of the reference
    draw rule, noise.py:188-222, is pinned in test_program.py); every kept state at
    the north-star tolerances and every probe table to 1e-12.  Error-free
    trajectories share one oracle run (they are the noiseless circuit)."""
    from paper_2008_07140_b200.trajectories import run_trajectories
    from paper_2008_07140_b200.workloads import noisy_trajectory_program, trajectory_seed

    prog = parse_program(workloads.rqc_text(4, 6, 20, seed=0))
    probe = run_trajectories(prog, 1e-3, 64, base_seed=0, probe_qubits=(0, 23))
    noisy = [t for t, e in zip(probe.trajectories, probe.errors) if e > 0]
    clean = [t for t, e in zip(probe.trajectories, probe.errors) if e == 0]
    assert len(noisy) >= 8 and len(clean) >= 8
    check = clean[:8] + noisy[:8]
    rep = run_trajectories(prog, 1e-3, max(check) + 1, base_seed=0, keep=tuple(check), probe_qubits=(0, 23))
    clean_ref = None
    for t in check:
        traj = noisy_trajectory_program(prog, 1e-3, trajectory_seed(0, t))
        if rep.errors[t] == 0:
            if clean_ref is None:
                clean_ref = O.run_full(traj, workers=O.cpu_threads()).state
            ref = clean_ref
        else:
            ref = O.run_full(traj, workers=O.cpu_threads()).state
        assert_parity(rep.kept[t], ref.amplitudes)
        assert np.abs(rep.tables[t] - O.pmeasure(ref, (0, 23))).max() <= 1e-12


# readouts on the sharded state too: tables summed over ranks, MEASURE drawn on rank 0
_SHARDED_RQC = workloads.rqc_for_qubits(16, 12, 4).replace("QINIT 16", "QINIT 16\nCREG 2", 1) + (
    "PMEASURE 0,15,7\nMEASURE 15,$0\nH 15\nPMEASURE 15,3\nMEASURE 3,$1\n")


def _sharded_gpu_worker(rank, world, port, out, transport):
    import os

    import torch
    import torch.distributed as dist

    from paper_2008_07140_b200.distributed import CudaShard, ShardedSimulator, make_transport
    from paper_2008_07140_b200 import _native as N

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for name, text in (("rqc", _SHARDED_RQC), ("qft", workloads.qft_text(15, True))):
            prog = parse_program(text)
            g = world.bit_length() - 1
            kind, _, variant = transport.partition("-")
            # specialised kernels at this small size (the fused exchange needs them); 8-qubit tiles
            # leave the leaving qubits outside the last pass's tile often enough to fuse
            opts = N.options(jit=1, tile_qubits=8, reg_qubits=4) if kind == "p2p" else None
            shard = CudaShard(prog.qubit_count - g, 0, options=opts)
            tr = make_transport(kind, dist, shard)
            sim = ShardedSimulator(prog.qubit_count, shard, chunk_log2=2, transport=tr)
            sim.fuse_exchange = variant == "fused"
            for _ in range(2):  # twice: the second run reuses buffers, handles and plans
                sim.set_basis(1)
                sim.run(prog, rng=np.random.default_rng(5) if rank == 0 else None)
            amps = sim.gather_amplitudes()
            if rank == 0:
                res[name] = (amps, len(sim.stats.swaps), sum(x.fused for x in sim.stats.swaps), sim.cregs,
                             [t for _, t in sim.tables])
            if hasattr(tr, "close"):
                tr.close()
            dist.barrier()
            sim.shard.close()
        if rank == 0:
            np.save(out, np.array([res], dtype=object), allow_pickle=True)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,transport", [(2, "gloo"), (4, "gloo"), (2, "p2p-copy"), (4, "p2p-copy"),
                                             (2, "p2p-fused"), (4, "p2p-fused")])
def test_sharded_path_on_gpu(world, transport, tmp_path):
    """CudaShard (libqsv on the GPU) + chunked global<->local qubit swaps, P ranks
    sharing the one GPU of this box.  Blocks travel over gloo through host
    memory, or as copy-engine pushes into CUDA-IPC-mapped peer buffers ordered
    by interprocess events (the P2PTransport used over NVLink on a multi-GPU
    box); no kernel ever waits on another rank."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "sharded.npy")
    mp.spawn(_sharded_gpu_worker, args=(world, port, out, transport), nprocs=world, join=True)
    res = np.load(out, allow_pickle=True)[0]
    for name, text in (("rqc", _SHARDED_RQC), ("qft", workloads.qft_text(15, True))):
        prog = parse_program(text)
        init = np.zeros(1 << prog.qubit_count, complex)
        init[1] = 1
        ref_run = O.run_full(prog, np.random.default_rng(5), initial=init)
        ref = ref_run.state.amplitudes
        amps, swaps, fused, cregs, tables = res[name]
        assert swaps > 0
        assert_parity(amps, ref)
        assert list(cregs) == list(ref_run.cregs)
        for t, (_, t2) in zip(tables, ref_run.tables):
            assert np.abs(t - t2).max() <= 1e-12
    if transport.endswith("fused"):
        assert sum(res[k][2] for k in res) > 0  # at least one exchange rode on a pass's stores


@pytest.mark.gpu
@pytest.mark.parametrize("positions", [(17,), (3, 12), (0, 9, 17)])
def test_exchange_out_pass_single_process(positions):
    """qsv_run_exchange on one GPU with local destinations: the last pass's stores
    land at dst[bits at positions] + (index with those bits replaced by self_bits);
    here dst[j] = receive buffer + j-th slot so the receive buffer must equal the
    plain run's state exactly (layout identity when self_bits = 0)."""
    import ctypes as C

    import torch

    from paper_2008_07140_b200 import _native as N

    n = 18
    prog = parse_program(workloads.rqc_for_qubits(n, 12, 5))
    rec = SV.compile_gates(prog.gate_instructions())
    L = N.lib()
    st = SV.init_state(n, max_qubits=n, device=0)
    recv = torch.zeros(1 << n, dtype=torch.complex128, device="cuda:0")
    o = N.options(jit=1)
    ex = N.qsv_exchange()
    ex.positions = sum(1 << p for p in positions)
    ex.self_bits = 0
    for j in range(1 << len(positions)):
        off = sum(((j >> i) & 1) << p for i, p in enumerate(positions))
        ex.dst[j] = recv.data_ptr() + off * 16
    ok = C.c_int()
    N.check(L.qsv_exchange_fusable(st.handle, rec.ctypes.data, len(rec), C.byref(o), ex.positions, C.byref(ok)))
    assert ok.value == 1
    st.set_basis(0)
    N.check(L.qsv_run_exchange(st.handle, rec.ctypes.data, len(rec), C.byref(o), C.byref(ex), C.byref(N.qsv_run_stats())))
    torch.cuda.synchronize()
    ref = O.run_full(prog).state.amplitudes
    assert_parity(recv.cpu().numpy(), ref)
    st.close()


@pytest.mark.gpu
@pytest.mark.parametrize("probe", [(0, 1, 2), (5,), (19, 3), (7, 0, 12, 18)])
def test_probe_out_last_pass(probe):
    """qsv_plan_execute_probe: the probe table accumulated by the last pass while
    it stores (clean run and runs with Pauli errors) equals pmeasure of the
    oracle's final state; the stored state is untouched by the probe."""
    import ctypes as C

    import torch

    from paper_2008_07140_b200 import _native as N

    n = 20
    prog = parse_program(workloads.rqc_for_qubits(n, 14, 8))
    gl = prog.gate_instructions()
    rec = SV.compile_gates(gl)
    L = N.lib()
    o = N.options()
    plan = C.c_void_p()
    N.check(L.qsv_plan_create(rec.ctypes.data, len(rec), n, C.byref(o), C.byref(plan)))
    st = SV.init_state(n, max_qubits=n, device=0)
    pq = np.asarray(probe, dtype=np.int32)
    table = torch.zeros(1 << len(probe), dtype=torch.float64, device="cuda:0")
    try:
        for errs in ([], [(10, 3, 1)], [(len(gl) - 1, 0, 2), (40, 7, 3)]):
            pa = np.zeros(len(errs), dtype=N.PAULI_DTYPE)
            for i, e in enumerate(errs):
                pa[i] = e
            st.set_basis(0)
            N.check(L.qsv_plan_execute_probe(st.handle, plan, pa.ctypes.data, len(pa), pq.ctypes.data, len(pq),
                                             C.c_void_p(table.data_ptr()), C.byref(o), C.byref(N.qsv_run_stats())))
            st.synchronize()
            got = table.cpu().numpy()
            by = {}
            for g, q, k in errs:
                by.setdefault(g, []).append(gates_mod_instruction("_XYZ"[k], q))
            insts = []
            for i, inst in enumerate(gl):
                insts += by.get(i, [])
                insts.append(inst)
            from paper_2008_07140_b200.program import Program

            ref = O.run_full(Program(n, prog.creg_count, tuple(insts))).state
            assert np.abs(got - O.pmeasure(ref, probe)).max() <= 1e-12, (probe, errs)
            assert_parity(st.amplitudes, ref.amplitudes)
    finally:
        L.qsv_plan_destroy(plan)
        st.close()


def gates_mod_instruction(name, q):
    from paper_2008_07140_b200.program import Instruction

    return Instruction(name, (q,))


def test_trajectories_clean_batches_match_single_runs():
    """Error-free trajectories run 2^b per batched state give the same probe tables
    as one-by-one runs (and the noisy ones are untouched)."""
    from paper_2008_07140_b200.trajectories import run_trajectories

    prog = parse_program(workloads.rqc_text(3, 4, 8, seed=5))
    a = run_trajectories(prog, 0.01, 100, base_seed=3, probe_qubits=(0, 6, 11), batch_clean=3)
    b = run_trajectories(prog, 0.01, 100, base_seed=3, probe_qubits=(0, 6, 11), batch_clean=0)
    assert sum(e == 0 for e in a.errors) >= 20 and sum(e > 0 for e in a.errors) >= 5
    assert a.errors == b.errors
    assert np.abs(a.tables - b.tables).max() <= 1e-12
    assert np.abs(a.norms - 1).max() <= 1e-10


def test_trajectories_fallback_when_plan_cannot_take_paulis(monkeypatch):
    """When the clean plan cannot carry a trajectory's Paulis (QSV_E_UNSUPPORTED, e.g. a
    super-pass plan) the trajectory runs as its explicit noisy program; states and probe
    tables still match the oracle with the same seeds."""
    from paper_2008_07140_b200 import _native as N
    from paper_2008_07140_b200.trajectories import run_trajectories
    from paper_2008_07140_b200.workloads import trajectory_seed

    lib = N.lib()
    monkeypatch.setattr(lib, "qsv_plan_execute_probe", lambda *a: N.QSV_E_UNSUPPORTED)
    prog = parse_program(workloads.rqc_text(3, 4, 8, seed=2))
    keep = tuple(range(6))
    rep = run_trajectories(prog, 0.05, 6, base_seed=7, probe_qubits=(0, 5, 11), keep=keep)
    assert sum(e > 0 for e in rep.errors) >= 1
    for t in keep:
        ref = O.run_full(prog, np.random.default_rng(trajectory_seed(7, t)), noise=("depolarizing", 0.05))
        assert_parity(rep.kept[t], ref.state.amplitudes)
        assert np.abs(rep.tables[t] - O.pmeasure(ref.state, (0, 5, 11))).max() <= 1e-12


def test_cold_call_runs_while_kernels_compile():
    """The first run of a new circuit (jit auto) does not wait for NVRTC: passes whose
    specialised kernel is still compiling run on the interpreted kernel (plus the scale op
    the compiled chain expects), the product-start plan's first pass reads the state of
    product_state_kernel; after qsv_jit_wait every pass runs compiled.  Both vs the oracle."""
    from paper_2008_07140_b200 import _native as N

    import time

    # a circuit no earlier run compiled (the on-disk kernel cache survives on a reused box)
    seed = 10_000 + int(time.time() * 1000) % 1_000_000
    prog = parse_program(workloads.rqc_for_qubits(22, 16, seed))
    ref = O.run_full(prog, workers=O.cpu_threads()).state.amplitudes
    cold = SV.run_full(prog)
    assert cold.stats["compiled_passes"] < cold.stats["passes"]
    assert_parity(cold.state.amplitudes, ref)
    cold.state.close()
    N.check(N.lib().qsv_jit_wait())
    warm = SV.run_full(prog)
    assert warm.stats["compiled_passes"] in (0, warm.stats["passes"])  # 0: the plan was already fully loaded
    assert_parity(warm.state.amplitudes, ref)
    # an uploaded (non-basis) start: no product start, the same mixed/compiled machinery
    psi0 = workloads.gaussian_state(22, 5)
    prog2 = parse_program(workloads.rqc_for_qubits(22, 12, seed + 1))
    ref2 = O.run_full(prog2, initial=psi0).state.amplitudes
    assert_parity(SV.run_full(prog2, initial_state=psi0).state.amplitudes, ref2)


EDGE_PROGRAMS = {
    "no_gates_1": "QINIT 1\n",
    "no_gates_5": "QINIT 5\nCREG 1\n",
    "only_readout": "QINIT 3\nCREG 3\nMEASURE 0,$0\nMEASURE 2,$2\nPMEASURE 2,1,0\n",
    "one_qubit_chain": "QINIT 1\nH 0\nT 0\nRX 0,\"0.3\"\nS 0\nH 0\n",
    "diagonal_only": "QINIT 6\nT 0\nS 3\nCZ 1,4\nCR 0,5,\"pi/8\"\nRZ 2,\"0.7\"\nZ 5\n",
    "many_controls": ("QINIT 10\n" + "".join(f"H {q}\n" for q in range(10))
                      + "".join(f"CONTROL {q}\n" for q in range(1, 9)) + "RY 0,\"0.9\"\nSWAP 0,9\n"
                      + "".join(f"ENDCONTROL {q}\n" for q in range(8, 0, -1)) + "iSWAP 9,0\n"),
    "top_and_bottom": "QINIT 16\nH 15\nH 0\nCNOT 15,0\nRX 15,\"1.1\"\nCZ 0,15\nSWAP 0,15\nT 15\nH 0\n",
}


@pytest.mark.parametrize("name", sorted(EDGE_PROGRAMS))
def test_edge_programs_all_configs(name):
    """Gate-less programs, readout-only programs, a single qubit, diagonal-only streams, the
    deepest control nesting the parser takes and gates on the extreme qubits, in every planner
    configuration, against the oracle (statevector.py:360-430)."""
    prog = parse_program(EDGE_PROGRAMS[name])
    ref = O.run_full(prog, np.random.default_rng(7))
    for cfg in CONFIGS:
        res = SV.run_full(prog, np.random.default_rng(7), **cfg)
        assert_parity(res.state.amplitudes, ref.state.amplitudes)
        assert res.cregs == ref.cregs
        assert len(res.tables) == len(ref.tables)
        for (_, got), (_, want) in zip(res.tables, ref.tables):
            assert np.abs(np.asarray(got) - np.asarray(want)).max() <= 1e-12
        res.state.close()
