"""First-call latency of the public API on a fresh process (NVRTC compiles included) vs warm."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
t0 = time.perf_counter()
from paper_2008_07140_b200 import statevector as SV, workloads
from paper_2008_07140_b200.program import parse_program
import torch; torch.cuda.init()
t1 = time.perf_counter()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
text = workloads.rqc_for_qubits(n, 24, 0)
for k in range(2):
    ta = time.perf_counter()
    res = SV.run_full(parse_program(text), max_qubits=n)
    res.state.synchronize() if hasattr(res.state, "synchronize") else None
    torch.cuda.synchronize()
    tb = time.perf_counter()
    print(f"n={n} call {k}: {1e3*(tb-ta):.1f} ms", flush=True)
    res.state.close()
print(f"import+init {1e3*(t1-t0):.0f} ms")
