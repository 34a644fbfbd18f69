"""The runtime kernel specialiser (csrc/qsv_jit.cpp), checked on CPU.

Every fused pass is emitted as straight-line CUDA with compile-time register
positions, smem offsets, matrices and control classes.  The generator can
render the same pass as plain C++; compiling that with gcc and running it
against the oracle validates the generated code without a GPU.  The device
rendering is compiled with NVRTC for sm_100a (no GPU needed either)."""

import ctypes as C

import numpy as np
import pytest

from conftest import program_text
from jit_host import kernel_source, plan_handle, run_plan_host
from oracle import oracle as O
from paper_2008_07140_b200 import _native as N
from paper_2008_07140_b200 import workloads
from paper_2008_07140_b200.program import parse_program
from paper_2008_07140_b200.statevector import compile_gates

CONFIGS = [dict(), dict(tile_qubits=5, reg_qubits=3, low_qubits=2), dict(tile_qubits=4, reg_qubits=2),
           dict(tile_qubits=6, reg_qubits=4, low_qubits=3)]


@pytest.mark.parametrize("cfg", CONFIGS)
def test_generated_passes_match_oracle_golden(golden, cfg):
    for name in golden["runs"]:
        prog = parse_program(program_text(golden, name))
        if any(not i.is_gate for i in prog.instructions):
            continue
        n = prog.qubit_count
        psi = workloads.gaussian_state(n, 3)
        ref = O.run_full(prog, initial=psi).state.amplitudes
        out = run_plan_host(compile_gates(prog.gate_instructions()), n, psi, **cfg)
        assert np.abs(out - ref).max() <= 1e-12, (name, cfg)


@pytest.mark.parametrize("seed", range(4))
def test_generated_passes_random_streams(seed):
    """Dense / permutation / diagonal 1q and 2q gates with controls on register,
    thread and external qubits, multi-tile (external bits + tile base)."""
    rng = np.random.default_rng(100 + seed)
    n = 9
    items = []
    for _ in range(60):
        qs = [int(q) for q in rng.permutation(n)]
        kind = int(rng.integers(0, 6))
        z = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
        q4, _ = np.linalg.qr(z)
        ctrl = tuple(qs[2:2 + int(rng.integers(0, 3))])
        if kind == 0:
            items.append((q4[:2, :2] / np.abs(np.linalg.det(q4[:2, :2])) ** 0.5, (qs[0],), ctrl))
        elif kind == 1:
            items.append((np.diag(np.exp(1j * rng.uniform(0, 6, 2))), (qs[0],), ctrl))
        elif kind == 2:
            items.append((q4, (qs[0], qs[1]), ctrl))
        elif kind == 3:
            items.append((np.diag(np.exp(1j * rng.uniform(0, 6, 4))), (qs[0], qs[1]), ctrl))
        elif kind == 4:
            perm = np.zeros((4, 4), complex)
            for r, c in enumerate(rng.permutation(4)):
                perm[r, c] = [1, -1, 1j, -1j, np.exp(0.3j)][int(rng.integers(0, 5))]
            items.append((perm, (qs[0], qs[1]), ctrl))
        else:
            items.append((np.array([[0, 1], [1, 0]], complex), (qs[0],), ctrl))
    recs = N.gate_records(items)
    psi = workloads.gaussian_state(n, seed)
    ref = O.OracleState(n, psi.copy(), 0)
    for u, t, c in items:
        O.apply_gate(ref, u, t, c)
    for cfg in CONFIGS:
        out = run_plan_host(recs, n, psi, **cfg)
        assert np.abs(out - ref.amplitudes).max() <= 1e-12, cfg


def test_generated_rqc_multi_tile():
    prog = parse_program(workloads.rqc_for_qubits(14, 10, 2))
    psi = workloads.gaussian_state(14, 5)
    ref = O.run_full(prog, initial=psi).state.amplitudes
    out = run_plan_host(compile_gates(prog.gate_instructions()), 14, psi, tile_qubits=8, reg_qubits=4,
                        low_qubits=3)
    assert np.abs(out - ref).max() <= 1e-12


def test_device_source_compiles_for_sm100a():
    prog = parse_program(workloads.rqc_text(5, 6, 24, 0))
    h = plan_handle(compile_gates(prog.gate_instructions()), 30)
    try:
        src = kernel_source(h, 0, False)
    finally:
        N.lib().qsv_plan_destroy(h)
    assert "qsv_pass" in src and "__launch_bounds__(" in src and "prefetch_l2" in src
    size = C.c_int64()
    N.check(N.lib().qsv_jit_compile(src.encode(), C.byref(size)))
    assert size.value > 1000


@pytest.mark.parametrize("n,m,s,budget", [(12, 6, 9, 64 << 20), (12, 6, 9, 16 << 9), (14, 7, 10, 16 << 11),
                                          (13, 6, 13, 64 << 20)])
def test_generated_super_pass_kernels(n, m, s, budget):
    """Two-level schedule: persistent super-pass kernels (inner passes on
    super-tiles, batches of super-tiles, grid barrier) vs the oracle."""
    from jit_host import run_plan_host_super

    prog = parse_program(workloads.rqc_for_qubits(n, 10, n))
    psi = workloads.gaussian_state(n, 5)
    ref = O.run_full(prog, initial=psi).state.amplitudes
    out = run_plan_host_super(compile_gates(prog.gate_instructions()), n, psi, budget=budget, tile_qubits=m,
                              reg_qubits=4, low_qubits=3, super_qubits=s)
    assert np.abs(out - ref).max() <= 1e-12


def test_super_plan_reduces_hbm_passes():
    prog = parse_program(workloads.rqc_text(5, 6, 24, 0))
    recs = compile_gates(prog.gate_instructions())
    for s, most in ((21, 5), (0, 16)):
        h = plan_handle(recs, 30, super_qubits=s)
        info = N.qsv_plan_info()
        N.check(N.lib().qsv_plan_summary(h, C.byref(info)))
        N.lib().qsv_plan_destroy(h)
        assert info.super_passes <= most, (s, info.super_passes)
    src_h = plan_handle(recs, 30, super_qubits=21)
    try:
        from jit_host import super_source

        src = super_source(src_h, 0, False)
    finally:
        N.lib().qsv_plan_destroy(src_h)
    assert "grid_sync" in src and "qsv_super" in src
    size = C.c_int64()
    N.check(N.lib().qsv_jit_compile(src.encode(), C.byref(size)))


@pytest.mark.parametrize("cfg", [dict(tile_qubits=6, reg_qubits=4, low_qubits=3),
                                 dict(tile_qubits=7, reg_qubits=3, low_qubits=2, super_qubits=10)])
def test_generated_qft_runtime_diagonals(cfg):
    """QFT: controlled phases between register, thread and tile qubits go
    through the runtime diagonal accumulators of the generated kernels."""
    from jit_host import run_plan_host_super

    n = 12
    psi = workloads.gaussian_state(n, 9)
    fwd = parse_program(workloads.qft_text(n))
    out = run_plan_host_super(compile_gates(fwd.gate_instructions()), n, psi, **cfg)
    assert np.abs(out - np.sqrt(1 << n) * np.fft.ifft(psi)).max() <= 1e-12
    rt = parse_program(workloads.qft_text(n, round_trip=True))
    out = run_plan_host_super(compile_gates(rt.gate_instructions()), n, psi, **cfg)
    assert np.abs(out - psi).max() <= 1e-12


@pytest.mark.parametrize("seed,n_pos", [(0, 2), (1, 1), (2, 3), (3, 2)])
def test_exchange_out_pass_host(seed, n_pos):
    """Exchange-out variant of a run's last pass (qsv_run_exchange): every output
    amplitude lands in dst[bits at `positions`] at its index with those bits
    replaced by this rank's own bits - the global<->local qubit swap fused into
    the pass's stores.  Host rendering of the generated kernel vs the oracle."""
    import ctypes as C2

    from jit_host import _compile, kernel_source, plan_handle

    n = 12
    prog = parse_program(workloads.rqc_for_qubits(n, 8, seed))
    recs = compile_gates(prog.gate_instructions())
    psi = workloads.gaussian_state(n, seed)
    ref = O.run_full(prog, initial=psi).state.amplitudes
    h = plan_handle(recs, n, tile_qubits=6, reg_qubits=3, low_qubits=2)
    try:
        info = N.qsv_plan_info()
        N.check(N.lib().qsv_plan_summary(h, C2.byref(info)))
        last = info.passes - 1
        pi = N.qsv_pass_info()
        N.check(N.lib().qsv_plan_pass(h, last, C2.byref(pi)))
        # outside the tile (per-tile destination) or inside it (per-store destination)
        pool = [q for q in range(n) if bool((pi.tile_mask >> q) & 1) == bool(seed % 2)]
        positions = tuple(sorted(pool[-n_pos:]))
        vmask = sum(1 << p for p in positions)
        out = psi.copy()
        for p in range(last):
            q = N.qsv_pass_info()
            N.check(N.lib().qsv_plan_pass(h, p, C2.byref(q)))
            _compile(kernel_source(h, p, True)).qsv_pass_host(out.ctypes.data, 1 << (n - q.m))
        need = C2.c_int64()
        N.check(N.lib().qsv_plan_exchange_source(h, last, 1, vmask, None, 0, C2.byref(need)))
        buf = C2.create_string_buffer(need.value)
        N.check(N.lib().qsv_plan_exchange_source(h, last, 1, vmask, buf, need.value, C2.byref(need)))
        lib = _compile(buf.value.decode())

        class XDst(C2.Structure):
            _fields_ = [("p", C2.c_uint64 * 8), ("self", C2.c_uint64)]

        dsts = [np.zeros(1 << n, complex) for _ in range(1 << len(positions))]
        self_val = (1 << len(positions)) - 2 if len(positions) > 1 else 1
        self_bits = sum(((self_val >> i) & 1) << p for i, p in enumerate(positions))
        xd = XDst()
        for j, d in enumerate(dsts):
            xd.p[j] = d.ctypes.data
        xd.self = self_bits
        lib.qsv_pass_host.argtypes = [C2.c_void_p, C2.c_ulonglong, XDst]
        lib.qsv_pass_host(out.ctypes.data, 1 << (n - pi.m), xd)
    finally:
        N.lib().qsv_plan_destroy(h)
    idx = np.arange(1 << n)
    j = sum(((idx >> p) & 1) << i for i, p in enumerate(positions))
    dest = (idx & ~vmask) | self_bits
    got = np.array([dsts[a][b] for a, b in zip(j, dest)])
    assert np.abs(got - ref).max() <= 1e-12
    written = sum(int(np.count_nonzero(d)) for d in dsts)
    assert written == np.count_nonzero(ref)


@pytest.mark.parametrize("pattern", ["45", "54", "4", "5"])
def test_mixed_register_qubits_per_pass(pattern, monkeypatch):
    """Plans whose passes use different register-qubit counts (r = 4 / 5 per
    pass, build_plan_auto): the per-pass kernels and the uniform-scale chain
    across them, host rendering vs the oracle."""
    monkeypatch.setenv("QSV_MIXED_R_PATTERN", pattern)
    for text, seed in ((workloads.rqc_for_qubits(16, 14, 2), 3), (workloads.qft_text(16, round_trip=True), 4)):
        prog = parse_program(text)
        psi = workloads.gaussian_state(16, seed)
        ref = O.run_full(prog, initial=psi).state.amplitudes
        out = run_plan_host(compile_gates(prog.gate_instructions()), 16, psi, tile_qubits=9, jit=1)
        assert np.abs(out - ref).max() <= 1e-12, pattern


@pytest.mark.parametrize("basis", [0, 5, 0b101101])
@pytest.mark.parametrize("cfg", [dict(), dict(tile_qubits=5, reg_qubits=3, low_qubits=2), dict(tile_qubits=6, reg_qubits=4)])
def test_product_start_plan_matches_oracle(basis, cfg):
    """Product-state start (qsv_options.product_start): every qubit's leading
    single-qubit gates (the RQC's H layer and the idle qubits' first gates) leave the
    stream and the first pass synthesises prefix (x) e_b from host-built factor tables
    instead of reading the state; host rendering vs the oracle from |basis>."""
    from jit_host import run_product_plan_host

    prog = parse_program(workloads.rqc_text(3, 4, 10, seed=basis % 7))
    n = prog.qubit_count
    got = run_product_plan_host(compile_gates(prog.gate_instructions()), n, basis, **cfg)
    assert got is not None
    init = np.zeros(1 << n, complex)
    init[basis] = 1
    ref = O.run_full(prog, initial=init).state.amplitudes
    assert np.abs(got[0] - ref).max() <= 1e-12


def test_product_start_split_rules():
    """Absorption stops at the first gate on a qubit that is not an uncontrolled
    single-qubit gate; diagonal single-qubit gates are absorbed too; a stream with
    nothing to absorb gives an ordinary plan."""
    from jit_host import run_product_plan_host

    text = "QINIT 4\nH 0\nT 0\nCZ 0,1\nH 1\nX 0\nRY 2,\"0.3\"\nCNOT 2,3\nH 3\nRZ 2,\"0.7\"\n"
    prog = parse_program(text)
    got, passes = run_product_plan_host(compile_gates(prog.gate_instructions()), 4, 0, tile_qubits=3,
                                        reg_qubits=2, low_qubits=1)
    ref = O.run_full(prog).state.amplitudes
    assert np.abs(got - ref).max() <= 1e-13 and passes >= 1
    only2q = parse_program("QINIT 3\nCZ 0,1\nCNOT 1,2\n")
    assert run_product_plan_host(compile_gates(only2q.gate_instructions()), 3, 0, tile_qubits=3, reg_qubits=2,
                                 low_qubits=1) is None


@pytest.mark.parametrize("cfg", [dict(tile_qubits=5, reg_qubits=3, low_qubits=2), dict(tile_qubits=6, reg_qubits=4, low_qubits=3)])
def test_external_control_phase_tables(cfg):
    """Controlled phases whose controls lie outside the tile are uniform over a CTA: groups of
    up to six external qubits become one table lookup per accumulator (csrc/qsv_jit.cpp,
    materialize).  Scattered and contiguous external controls, more than six per target (two
    tables), 1- and 2-qubit diagonals, against the oracle; the tables must appear in the source."""
    rng = np.random.default_rng(77)
    n = 15
    items = []
    h = np.array([[1, 1], [1, -1]]) / np.sqrt(2)
    for t in (0, 1, 3):
        items.append((h, (t,), ()))
        for c in (5, 6, 7, 8, 9, 10, 11, 12, 13, 14):      # contiguous run: two tables
            items.append((np.diag([1, np.exp(1j * rng.uniform(0, 6))]), (t,), (c,)))
        items.append((h, (t,), ()))
    for t in (2, 4):
        items.append((h, (t,), ()))
        for c in (6, 9, 11, 14):                            # scattered controls
            items.append((np.diag([1, np.exp(1j * rng.uniform(0, 6))]), (t,), (c,)))
        items.append((np.diag(np.exp(1j * rng.uniform(0, 6, 4))), (t, 13), ()))   # 2-qubit diagonal, one end external
        items.append((np.diag([1, np.exp(1j * rng.uniform(0, 6))]), (t,), (8, 12)))  # two external controls
        items.append((h, (t,), ()))
    recs = N.gate_records(items)
    psi = workloads.gaussian_state(n, 5)
    ref = O.OracleState(n, psi.copy(), 0)
    for u, t, c in items:
        O.apply_gate(ref, u, t, c)
    out = run_plan_host(recs, n, psi, **cfg)
    assert np.abs(out - ref.amplitudes).max() <= 1e-12
    hnd = plan_handle(recs, n, **cfg)
    try:
        src = kernel_source(hnd, 0, False)
    finally:
        N.lib().qsv_plan_destroy(hnd)
    assert "(unsigned)(base >> " in src and "qtab" in src


def test_first_reading_pass_staggers_its_first_wave(monkeypatch):
    """A plan's first pass that reads its input (>= 2^16 tiles) delays the second CTA of every
    SM of its first residency wave (csrc/qsv_jit.cpp, kernel_head); later passes, small states,
    product-start (synthesising) first passes and the host rendering do not; QSV_JIT_STAGGER=0
    switches it off."""
    monkeypatch.delenv("QSV_JIT_STAGGER", raising=False)

    def sources(text, **opts):
        prog = parse_program(text)
        h = plan_handle(compile_gates(prog.gate_instructions()), prog.qubit_count, **opts)
        try:
            info = N.qsv_plan_info()
            N.check(N.lib().qsv_plan_summary(h, C.byref(info)))
            return [kernel_source(h, p, False) for p in range(info.passes)], kernel_source(h, 0, True)
        finally:
            N.lib().qsv_plan_destroy(h)

    big, host0 = sources(workloads.qft_text(30, round_trip=False), product_start=-1)
    assert len(big) >= 2 and "%nsmid" in big[0] and "clock64()" in big[0]
    assert all("%nsmid" not in s for s in big[1:]) and "%nsmid" not in host0
    small, _ = sources(workloads.qft_text(20, round_trip=False), product_start=-1)
    assert all("%nsmid" not in s for s in small)
    prod, _ = sources(workloads.rqc_text(5, 6, 8, seed=3), product_start=1)
    assert "%nsmid" not in prod[0]
    monkeypatch.setenv("QSV_JIT_STAGGER", "0")
    off, _ = sources(workloads.qft_text(30, round_trip=False), product_start=-1)
    assert all("%nsmid" not in s for s in off)
