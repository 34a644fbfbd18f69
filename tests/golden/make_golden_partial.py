"""Generate tests/golden/partial.json: amplitudes from the REAL reference
partial-amplitude backend (`qcsim.partition.run_partial`, partition.py:151-192).

Run in the build container only (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden_partial.py
The GPU tests and CPU tests read the committed JSON; nothing reads the
reference at test time.
"""

import json
from pathlib import Path

import numpy as np
from qcsim import parse_program
from qcsim.partition import plan_partition, run_partial
from qcsim.rqc import RqcConfig, generate_rqc

CASES = [
    # (name, program text, cut, n_targets or None = all)
    ("cnot2", "QINIT 2\nH 0\nCNOT 0,1\n", 1, None),
    ("cz2", "QINIT 2\nH 0\nCZ 0,1\n", 1, None),
    ("ctrl_upper3", 'QINIT 3\nH 2\nH 0\nCR 2,0,"0.77"\nRY 2,"0.2"\n', 1, None),
    ("fig1_8", "QINIT 8\n" + "".join(f"H {q}\n" for q in range(8))
     + "CNOT 0,1\nCNOT 2,3\nCNOT 4,5\nCNOT 6,7\nT 2\nT 6\nCZ 3,4\nCZ 2,5\n"
     + "".join(f'RY {q},"0.3"\n' for q in range(8)), 4, None),
    ("rqc_1x8_s0", generate_rqc(RqcConfig(1, 8, depth=12, seed=0)), 4, None),
    ("rqc_1x8_s5", generate_rqc(RqcConfig(1, 8, depth=12, seed=5)), 4, None),
    ("rqc_1x12_s31", generate_rqc(RqcConfig(1, 12, depth=8, seed=31)), 6, 64),
    ("rqc_2x7_s2", generate_rqc(RqcConfig(2, 7, depth=10, seed=2)), 7, 64),
    ("rqc_1x16_s4", generate_rqc(RqcConfig(1, 16, depth=14, seed=4)), 8, 48),
]


def main():
    out = {}
    for name, text, cut, nt in CASES:
        prog = parse_program(text)
        n = prog.qubit_count
        if nt is None:
            idx = list(range(1 << n))
        else:
            rng = np.random.default_rng(len(name))
            idx = sorted({int(i) for i in rng.integers(0, 1 << n, nt)})
        targets = [format(i, f"0{n}b") for i in idx]
        amps = run_partial(prog, cut, targets)
        out[name] = {
            "text": text, "cut": cut, "c": plan_partition(prog, cut).c, "targets": targets,
            "re": [amps[t].real for t in targets], "im": [amps[t].imag for t in targets],
        }
        print(name, n, "c =", out[name]["c"], len(targets), "targets")
    Path(__file__).with_name("partial.json").write_text(json.dumps(out, indent=0))


if __name__ == "__main__":
    main()
