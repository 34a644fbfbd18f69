"""Dumps the generated pass kernels of a workload's plan to a directory and compiles them with
nvcc (-Xptxas -v) so registers / spills can be read without a GPU.
usage: dump_kernels.py outdir [--workload c2|qft|n32|c5] [--no-compile]"""
import argparse, ctypes as C, subprocess, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2008_07140_b200 import _native as N, workloads
from paper_2008_07140_b200.program import parse_program
from paper_2008_07140_b200.statevector import compile_gates

ap = argparse.ArgumentParser()
ap.add_argument("outdir")
ap.add_argument("--workload", default="c2")
ap.add_argument("--no-compile", action="store_true")
ap.add_argument("--regs", type=int, default=0)
a = ap.parse_args()
text = {"c2": lambda: workloads.rqc_text(5, 6, 24, seed=0), "n32": lambda: workloads.rqc_text(4, 8, 24, seed=0),
        "c5": lambda: workloads.rqc_text(4, 6, 20, seed=0), "qft": lambda: workloads.qft_text(30, round_trip=True)}[a.workload]()
prog = parse_program(text)
recs = compile_gates(prog.gate_instructions())
n = prog.qubit_count
L = N.lib()
h = C.c_void_p()
o = N.options(jit=1, product_start=1 if a.workload != "qft" else -1, reg_qubits=a.regs)
N.check(L.qsv_plan_create(recs.ctypes.data, len(recs), n, C.byref(o), C.byref(h)))
info = N.qsv_plan_info()
N.check(L.qsv_plan_summary(h, C.byref(info)))
out = Path(a.outdir); out.mkdir(parents=True, exist_ok=True)
procs = []
for p in range(info.passes):
    need = C.c_int64()
    L.qsv_plan_kernel_source(h, p, 0, None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value + 1)
    N.check(L.qsv_plan_kernel_source(h, p, 0, buf, need.value + 1, C.byref(need)))
    f = out / f"pass{p}.cu"
    f.write_bytes(buf.value)
    if not a.no_compile:
        procs.append((p, subprocess.Popen(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-Xptxas", "-v",
                                           "-o", str(out / f"pass{p}.cubin"), str(f)], stderr=subprocess.PIPE, text=True)))
for p, pr in procs:
    err = pr.communicate()[1]
    lines = [l for l in err.splitlines() if "registers" in l or "spill" in l or "error" in l]
    print(p, " | ".join(l.split("ptxas info    : ")[-1] for l in lines))
