"""Where C5 trajectory time goes (diagnostic): clean JIT plan vs interpreted noisy runs vs readout."""
import ctypes as C, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2008_07140_b200 import _native as N, statevector as SV, workloads
from paper_2008_07140_b200.program import parse_program

prog = parse_program(workloads.rqc_text(4, 6, 20, seed=0))
L = N.lib()
st = SV.init_state(24, device=0)
clean = SV.compile_gates([i for i in prog.instructions if i.is_gate])
oc = N.options(); plan = C.c_void_p()
N.check(L.qsv_plan_create(clean.ctypes.data, len(clean), 24, C.byref(oc), C.byref(plan)))
def timeit(f, k=20):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): f()
    N.check(L.qsv_synchronize(st.handle)); return (time.perf_counter() - t0) / k * 1e3
def clean_run():
    st.set_basis(0); N.check(L.qsv_plan_execute(st.handle, plan, C.byref(oc), C.byref(N.qsv_run_stats())))
print("clean JIT plan execute ms", timeit(clean_run))
noisy = [t for t in range(200) if workloads.sample_pauli_insertions(prog, 1e-3, workloads.trajectory_seed(0, t))][:20]
recs = [SV.compile_gates([i for i in workloads.noisy_trajectory_program(prog, 1e-3, workloads.trajectory_seed(0, t)).instructions if i.is_gate]) for t in noisy]
for jit in (-1, 1):
    o = N.options(fuse=True, jit=jit)
    for k, rec in enumerate(recs[:4]):
        t0 = time.perf_counter(); st.set_basis(0)
        N.check(L.qsv_run(st.handle, rec.ctypes.data, len(rec), C.byref(o), C.byref(N.qsv_run_stats())))
        N.check(L.qsv_synchronize(st.handle)); t1 = time.perf_counter()
        st.set_basis(0)
        N.check(L.qsv_run(st.handle, rec.ctypes.data, len(rec), C.byref(o), C.byref(N.qsv_run_stats())))
        N.check(L.qsv_synchronize(st.handle)); t2 = time.perf_counter()
        print(f"noisy jit={jit} traj {noisy[k]}: first {1e3*(t1-t0):.1f} ms, repeat {1e3*(t2-t1):.2f} ms")
pq = np.asarray((0, 1, 2), np.int32)
print("pmeasure ms", timeit(lambda: SV.pmeasure(st, pq)))
print("norm ms", timeit(lambda: st.norm_sq()))
t0 = time.perf_counter()
for t in range(1024): workloads.sample_pauli_insertions(prog, 1e-3, workloads.trajectory_seed(0, t))
print("sampling 1024 ms", 1e3 * (time.perf_counter() - t0))
