"""Command line for the full-amplitude path (reference `qcsim run --mode full`).

    python -m paper_2008_07140_b200.cli run script.qprog [--seed S] [--noise kind:p[:G,...]]
                                              [--out FILE] [--log FILE] [--max-qubits N]
                                              [--dump-state FILE] [--no-fuse]
    python -m paper_2008_07140_b200.cli run script.qprog --mode partial --targets 0101,...|FILE
                                              [--cut C] [--out FILE]
    python -m paper_2008_07140_b200.cli rqc --rows R --cols C --depth D [--seed S]
                                              [--pmeasure q,q] [--patterns 4|8] [--out FILE]

Output and error conventions follow reference `cli.py:23-34,122-161,233-248`:
PMEASURE tables print one line per basis string in ascending binary order
(first listed qubit leftmost) with 6 significant digits and exact zeros as
"0"; MEASURE results print as "creg j: v"; errors are logged as
"Class: message (line N)" and the process exits with the class's code
(2 parse, 3 resource, 4 numeric).  `--mode partial` (reference cli.py:163-174)
runs the batched branch decomposition of `partition.py` on the same engine and
prints "bits: re+imi" lines; single-amplitude graph contraction is a different
algorithm and out of scope.
"""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np

from . import noise, program, rqc
from .errors import SimulatorError


# Probabilities below this print as "0".  The reference prints exact zeros as
# "0" (cli.py:31-33); where it cancels exactly, FMA-contracted GPU arithmetic
# leaves residues of ~1e-34, i.e. amplitudes ~1e-17 - far below the 1e-10
# parity tolerance - so they are treated as zero when printed.
ZERO_PRINT = 1e-24


def format_pmeasure(table: np.ndarray, warn=None) -> str:
    m = (len(table) - 1).bit_length()
    total = float(table.sum())
    if warn is not None and abs(total - 1.0) > 1e-9:
        warn(f"probability table sums to {total!r}, expected 1")
    return "\n".join(f"{format(i, f'0{m}b')}: {'0' if abs(p) < ZERO_PRINT else f'{p:.6g}'}"
                     for i, p in enumerate(table))


class _Log:
    def __init__(self, path):
        self.path, self.lines = path, []

    def __call__(self, message: str) -> None:
        self.lines.append(message)
        if self.path is None:
            print(message, file=sys.stderr)

    def flush(self) -> None:
        if self.path and self.lines:
            Path(self.path).write_text("\n".join(self.lines) + "\n")


def format_amplitude(z: complex) -> str:
    """reference cli.py:19-20"""
    return f"{z.real:.6f}{z.imag:+.6f}i"


def _read_targets(value: str) -> list[str]:
    """Comma-separated bit strings or a whitespace-separated file (cli.py:59-64)."""
    path = Path(value)
    if path.is_file():
        return [t.strip() for t in path.read_text().split() if t.strip()]
    return [t.strip() for t in value.split(",") if t.strip()]


def _emit(text: str, out) -> None:
    if out:
        Path(out).write_text(text)
    else:
        sys.stdout.write(text)


def run_text(prog, seed: int = 0, noise_spec: str | None = None, max_qubits: int = 30, warn=None,
             fuse: bool = True):
    """Run a parsed program; returns (stdout text, RunResult)."""
    from .statevector import run_full

    rng = np.random.default_rng(seed)
    model = noise.parse_noise_spec(noise_spec) if noise_spec else None
    result = run_full(prog, rng, model, max_qubits=max_qubits, fuse=fuse)
    blocks = [format_pmeasure(table, warn=warn) for _, table in result.tables]
    if any(i.name == "MEASURE" for i in prog.instructions):
        blocks.append("\n".join(f"creg {j}: {v}" for j, v in enumerate(result.cregs)))
    return (("\n\n".join(blocks) + "\n") if blocks else ""), result


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="qsv", description="B200 full-amplitude quantum circuit simulator")
    sub = ap.add_subparsers(dest="command", required=True)
    run = sub.add_parser("run", help="execute an instruction script (full-amplitude mode)")
    run.add_argument("script")
    run.add_argument("--mode", choices=("full", "partial"), default="full")
    run.add_argument("--cut", type=int, default=None, help="partition boundary (partial)")
    run.add_argument("--targets", default=None, help="bit strings, comma-separated or a file (partial)")
    run.add_argument("--workers", type=int, default=1, help="accepted for compatibility; unused")
    run.add_argument("--seed", type=int, default=0)
    run.add_argument("--noise", default=None, help="kind:p[:MNEMONIC,...]")
    run.add_argument("--out", default=None)
    run.add_argument("--log", default=None)
    run.add_argument("--max-qubits", type=int, default=30)
    run.add_argument("--dump-state", default=None)
    run.add_argument("--no-fuse", action="store_true", help="one kernel per gate (reference-shaped)")
    gen = sub.add_parser("rqc", help="generate a layered grid random circuit")
    gen.add_argument("--rows", type=int, required=True)
    gen.add_argument("--cols", type=int, required=True)
    gen.add_argument("--depth", type=int, required=True)
    gen.add_argument("--seed", type=int, default=0)
    gen.add_argument("--pmeasure", default=None)
    gen.add_argument("--patterns", type=int, choices=(4, 8), default=4)
    gen.add_argument("--out", default=None)
    return ap


def main(argv=None) -> int:
    args = _parser().parse_args(argv)
    log = _Log(getattr(args, "log", None))
    try:
        if args.command == "rqc":
            pm = tuple(int(q) for q in args.pmeasure.split(",")) if args.pmeasure else ()
            cfg = rqc.RqcConfig(args.rows, args.cols, args.depth, args.seed, pmeasure=pm,
                                patterns=args.patterns, no_repeat=args.patterns == 8)
            _emit(rqc.generate_rqc(cfg), args.out)
            return 0
        prog = program.parse_program(Path(args.script).read_text())
        if args.mode == "partial":
            from . import partition
            from .errors import ParseError

            if not args.targets:
                raise ParseError("partial mode requires --targets")
            cut = args.cut if args.cut is not None else prog.qubit_count // 2
            amps = partition.run_partial(prog, cut, _read_targets(args.targets), workers=args.workers,
                                         max_qubits=args.max_qubits, fuse=not args.no_fuse)
            _emit("\n".join(f"{t}: {format_amplitude(a)}" for t, a in amps.items()) + "\n", args.out)
            return 0
        out, result = run_text(prog, args.seed, args.noise, args.max_qubits, warn=log, fuse=not args.no_fuse)
        if args.dump_state:
            from .dump import save_state

            save_state(result.state, args.dump_state)
        _emit(out, args.out)
        return 0
    except SimulatorError as exc:
        log(exc.render())
        return exc.exit_code
    finally:
        log.flush()


if __name__ == "__main__":
    sys.exit(main())
