"""B200-native full-amplitude state-vector engine (arXiv 2008.07140 hot path).

The public surface mirrors the reference package's full-amplitude API
(`qcsim/__init__.py:10-16`, `qcsim/statevector.py:292-430`): parse a script
into a `Program`, run it with `run_full`, read `RunResult.state`.  Gate
application, fusion/scheduling and the sharded layout live in the native
library `libqsv.so` (hand-written sm_100a CUDA + C++ scheduler) behind the
C ABI declared in `include/qsv.h`; there is no CPU execution path.
"""

from .program import Instruction, Program, eval_angle, parse_program, to_script
from .rqc import RqcConfig, generate_rqc

__version__ = "0.1.0"


def __getattr__(name):
    # the engine needs the native library; import it lazily so the parser and
    # generators stay usable on machines without the built .so
    if name in ("RunResult", "StateVector", "init_state", "run_full", "apply_instruction"):
        from . import statevector

        return getattr(statevector, name)
    raise AttributeError(name)


__all__ = ["Instruction", "Program", "eval_angle", "parse_program", "to_script",
           "RqcConfig", "generate_rqc", "RunResult", "StateVector", "init_state",
           "run_full", "apply_instruction", "__version__"]
