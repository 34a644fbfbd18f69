"""Cost of carrying a global<->local qubit swap in a pass's stores (exchange-out
variant, qsv_run_exchange) vs the plain pass, on ONE GPU: destinations are two
halves of a local receive buffer (what a 2-rank exchange writes, minus NVLink)."""
import ctypes as C, sys
sys.path.insert(0, ".")
import torch
import bench
from paper_2008_07140_b200 import _native as N, statevector as SV

n = 30
text, prog = bench.workload(n, "rqc")
rec = SV.compile_gates(prog.gate_instructions())
L = N.lib()
st = SV.init_state(n, max_qubits=n, device=0)
spare = torch.empty(1 << n, dtype=torch.complex128, device="cuda:0")
o = N.options(profile=1)
for pos in (29, 20, 11):
    ex = N.qsv_exchange()
    ex.positions = 1 << pos
    ex.self_bits = 0
    ex.dst[0] = spare.data_ptr()
    ex.dst[1] = spare.data_ptr() + (1 << pos) * 16
    res = {}
    for name in ("plain", "exchange"):
        for k in range(3):
            stats = N.qsv_run_stats()
            st.set_basis(0)
            if name == "plain":
                N.check(L.qsv_run(st.handle, rec.ctypes.data, len(rec), C.byref(o), C.byref(stats)))
            else:
                N.check(L.qsv_run_exchange(st.handle, rec.ctypes.data, len(rec), C.byref(o), C.byref(ex), C.byref(stats)))
            torch.cuda.synchronize()
        res[name] = (stats.kernel_ms, stats.max_launch_ms)
    # correctness of the layout: the spare must equal the plain run's state
    st.set_basis(0)
    N.check(L.qsv_run(st.handle, rec.ctypes.data, len(rec), C.byref(o), C.byref(N.qsv_run_stats())))
    d = C.c_double()
    N.check(L.qsv_max_abs_diff(st.handle, C.c_void_p(spare.data_ptr()), C.byref(d)))
    print(f"position {pos}: plain run {res['plain'][0]:.2f} ms, with exchange-out last pass {res['exchange'][0]:.2f} ms, "
          f"max|d| {d.value:.1e}")
