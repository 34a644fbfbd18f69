"""Latency of ONE run_full call launched on an idle GPU (sleep before every call) against the
same call issued back to back: does a pass that starts on an idle GPU run its CTA pairs in lock
step?  usage: idle_start_probe.py [c2|qft]   (QSV_JIT_STAGGER=... to compare)"""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
from paper_2008_07140_b200 import statevector as SV, workloads, _native as N
from paper_2008_07140_b200.program import parse_program

w = sys.argv[1] if len(sys.argv) > 1 else "c2"
if w == "c2":
    prog, psi0 = parse_program(workloads.rqc_text(5, 6, 24, seed=0)), None
else:
    prog = parse_program(workloads.qft_text(30, round_trip=True))
    psi0 = workloads.gaussian_state(30, 1)
n = prog.qubit_count
st = SV.init_state(n, max_qubits=n)
kw = dict(state=st, max_qubits=n, jit=1)
if psi0 is not None:
    kw["initial_state"] = psi0
for _ in range(3):
    SV.run_full(prog, **kw)
N.check(N.lib().qsv_jit_wait())
st.synchronize()
def once():
    t0 = time.perf_counter(); SV.run_full(prog, **kw); st.synchronize(); return (time.perf_counter() - t0) * 1e3
if psi0 is None:
    b2b = [once() for _ in range(6)]
    idle = []
    for _ in range(6):
        time.sleep(0.3); idle.append(once())
    print(w, "back-to-back ms", [round(x, 2) for x in b2b], "| from idle ms", [round(x, 2) for x in idle])
else:
    print(w, "per call ms (includes the 16 GiB upload)", [round(once(), 1) for _ in range(4)])
