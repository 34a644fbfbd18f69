"""Typed errors of the state-vector engine.

Mirrors the reference exception taxonomy (`qcsim/errors.py:1-128`) so code
written against the reference catches the same classes, with the same CLI
exit codes: 2 = script/config validation, 3 = resource limit, 4 = numeric or
internal failure.  The C-ABI (`include/qsv.h`) returns negative status codes
that `raise_for_status` maps back onto these classes.
"""

from __future__ import annotations


class SimulatorError(Exception):
    """Base class; carries an optional 1-based source line."""

    exit_code = 4

    def __init__(self, message: str, line: int | None = None):
        super().__init__(message)
        self.message = message
        self.line = line

    def render(self) -> str:
        where = "" if self.line is None else f" (line {self.line})"
        return f"{type(self).__name__}: {self.message}{where}"


class ParseError(SimulatorError):
    exit_code = 2


class ResourceError(SimulatorError):
    exit_code = 3


class NumericError(SimulatorError):
    exit_code = 4


def _subclass(name: str, base: type) -> type:
    return type(name, (base,), {"__module__": __name__})


# Validation errors (exit 2).  Same names as the reference so `except X:` ports.
MissingQinit = _subclass("MissingQinit", ParseError)
UnknownMnemonic = _subclass("UnknownMnemonic", ParseError)
QubitOutOfRange = _subclass("QubitOutOfRange", ParseError)
CregOutOfRange = _subclass("CregOutOfRange", ParseError)
DuplicateQubitArg = _subclass("DuplicateQubitArg", ParseError)
UnbalancedBlock = _subclass("UnbalancedBlock", ParseError)
MalformedAngle = _subclass("MalformedAngle", ParseError)
MeasureInsideDagger = _subclass("MeasureInsideDagger", ParseError)
MeasureInsideControl = _subclass("MeasureInsideControl", ParseError)
ControlQubitCollision = _subclass("ControlQubitCollision", ParseError)
NonUnitaryU4 = _subclass("NonUnitaryU4", ParseError)
MalformedTarget = _subclass("MalformedTarget", ParseError)
UnsupportedGate = _subclass("UnsupportedGate", ParseError)
InvalidProbability = _subclass("InvalidProbability", ParseError)
UncuttableGate = _subclass("UncuttableGate", ParseError)  # partial mode (partition.py)

# Resource errors (exit 3).
TooManyQubits = _subclass("TooManyQubits", ResourceError)
BranchExplosion = _subclass("BranchExplosion", ResourceError)  # partial mode branch budget

# Numeric errors (exit 4).
DegenerateState = _subclass("DegenerateState", NumericError)
DegenerateBranch = _subclass("DegenerateBranch", NumericError)


class DeviceError(NumericError):
    """CUDA / NCCL failure inside the native library (no reference analogue)."""


class NativeLibraryMissing(SimulatorError):
    """The compiled libqsv.so is absent: there is deliberately no CPU fallback."""


# C-ABI status codes (include/qsv.h) -> exception class.
STATUS_CLASSES = {
    -2: ParseError,
    -3: TooManyQubits,
    -4: NumericError,
    -5: DeviceError,
    -6: UnsupportedGate,
    -7: DegenerateState,
}


def raise_for_status(status: int, message: str) -> None:
    if status == 0:
        return
    raise STATUS_CLASSES.get(status, SimulatorError)(message or f"status {status}")
