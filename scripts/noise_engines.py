"""run_full(prog, rng, noise) on the C2 circuit (RQC 5x6, 24 cycles, n=30) under
depolarising p=1e-3 on every gate: the presampled fused engine (default for
mixed-unitary channels) vs the per-gate reference-shaped engine (weights pass +
gate pass per noisy gate), and amplitude damping (state-dependent) as a batch of
one.  Prints one JSON line per engine; the two depolarising runs must agree."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2008_07140_b200 import workloads  # noqa: E402
from paper_2008_07140_b200.noise import make_noise_model  # noqa: E402
from paper_2008_07140_b200.program import parse_program  # noqa: E402
from paper_2008_07140_b200.statevector import run_full  # noqa: E402

n_arg = int(sys.argv[1]) if len(sys.argv) > 1 else 30
prog = parse_program(workloads.rqc_text(5, 6, 24, seed=0) if n_arg == 30 else workloads.rqc_for_qubits(n_arg, 24, 0))
G = len(prog.gate_instructions())
n = prog.qubit_count
out = {}
for kind, engine in (("depolarizing", "fused"), ("depolarizing", "sequential"), ("ampdamp", "fused")):
    model = make_noise_model(kind, 1e-3)
    run_full(prog, np.random.default_rng(1), model, noise_engine=engine).state.close()  # warm-up / plan cache
    t0 = time.perf_counter()
    res = run_full(prog, np.random.default_rng(7), model, noise_engine=engine)
    res.state.synchronize()
    dt = time.perf_counter() - t0
    out[(kind, engine)] = res
    print(json.dumps({"n_qubits": n, "gates": G, "noise": f"{kind} p=1e-3 on every gate", "engine": engine,
                      "path": res.stats.get("noise_engine", "batch-of-one" if engine == "fused" else "sequential"),
                      "seconds": dt, "amp_gate_per_s": G * 2.0 ** n / dt}), flush=True)
a = out[("depolarizing", "fused")].state
b = out[("depolarizing", "sequential")].state
print(json.dumps({"depolarizing fused vs sequential max|d|": a.max_abs_diff(b)}))
