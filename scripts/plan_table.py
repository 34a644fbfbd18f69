"""Plan table on the CPU (planner + specialiser cost model are host code): passes, stages,
FP64/amp per pass and a modeled time.  usage: plan_table.py [--workload c2|qft|n32] [--low L]
[--tile m] [--regs r] [--product 0|1]"""
import argparse, ctypes as C, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_07140_b200 import _native as N, workloads
from paper_2008_07140_b200.program import parse_program
from paper_2008_07140_b200.statevector import compile_gates

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="c2")
ap.add_argument("--low", type=int, default=0)
ap.add_argument("--tile", type=int, default=0)
ap.add_argument("--regs", type=int, default=0)
ap.add_argument("--product", type=int, default=1)
ap.add_argument("--seed", type=int, default=None)
a = ap.parse_args()
if a.workload == "c2":
    text = workloads.rqc_text(5, 6, 24, seed=a.seed if a.seed is not None else 0)
elif a.workload == "n32":
    text = workloads.rqc_text(4, 8, 24, seed=a.seed if a.seed is not None else 0)
elif a.workload == "c5":
    text = workloads.rqc_text(4, 6, 20, seed=a.seed if a.seed is not None else 0)
else:
    text = workloads.qft_text(30, round_trip=True)
prog = parse_program(text)
recs = compile_gates(prog.gate_instructions())
n = prog.qubit_count
L = N.lib()
h = C.c_void_p()
o = N.options(tile_qubits=a.tile, reg_qubits=a.regs, low_qubits=a.low, jit=1, product_start=1 if (a.product and a.workload != "qft") else -1)
t0 = time.perf_counter()
N.check(L.qsv_plan_create(recs.ctypes.data, len(recs), n, C.byref(o), C.byref(h)))
t1 = time.perf_counter()
info = N.qsv_plan_info()
N.check(L.qsv_plan_summary(h, C.byref(info)))
print(f"n={n} gates={len(recs)} passes={info.passes} stages={info.stages} plan {1e3*(t1-t0):.0f} ms product={info.product_start}")
tot = 0.0; model = 0.0
for p in range(info.passes):
    pi = N.qsv_pass_info()
    N.check(L.qsv_plan_pass(h, p, C.byref(pi)))
    c = C.c_double()
    N.check(L.qsv_plan_pass_cost(h, p, C.byref(c)))
    tot += c.value
    hbm = 5.0 if (p or not info.product_start) else 2.6
    t = max(hbm, 0.7 * pi.n_stages + 0.066 * c.value - 0.7)
    model += t
    tq = [q for q in range(n) if (pi.tile_mask >> q) & 1]
    print(f"  pass {p}: ops={pi.n_ops:3d} stages={pi.n_stages} fp64/amp={c.value:6.1f} model {t:5.2f} ms  tile={tq}")
print(f"total fp64/amp {tot:.1f}  modeled {model:.1f} ms")
