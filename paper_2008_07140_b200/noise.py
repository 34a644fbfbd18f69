"""Kraus channels and noise models (host side of the noisy-trajectory path).

Mirrors `qcsim/noise.py:25-137`: six single-qubit channels, two-qubit
channels as Kronecker products, first-matching-rule noise models and the CLI
spec syntax.  Intensity convention as in the reference: the flip channels
are noiseless at p = 1, damping and depolarising at p = 0.

Trajectory execution lives in `statevector._noisy` (branch weights from one
on-device reduced-density pass) and, for pre-sampled Pauli trajectories
(BASELINE config 5), in `workloads.sample_pauli_insertions` +
`trajectories.run_trajectories`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import gates
from .errors import InvalidProbability

KINDS = ("bitflip", "phaseflip", "bitphaseflip", "ampdamp", "phasedamp", "depolarizing")


def kraus_ops(kind: str, p: float) -> list[np.ndarray]:
    """Operator set of the named channel at intensity p (noise.py:35-64)."""
    if not 0.0 <= p <= 1.0:
        raise InvalidProbability(f"noise intensity {p} outside [0, 1]")
    sp, sq = math.sqrt(p), math.sqrt(1.0 - p)
    damp0 = np.array([[1, 0], [0, sq]], dtype=np.complex128)
    flips = {"bitflip": gates.X, "phaseflip": gates.Z, "bitphaseflip": gates.Y}
    if kind in flips:
        return [sp * gates.I2, sq * flips[kind]]
    if kind == "ampdamp":
        return [damp0, np.array([[0, sp], [0, 0]], dtype=np.complex128)]
    if kind == "phasedamp":
        return [damp0, np.array([[0, 0], [0, sp]], dtype=np.complex128)]
    if kind == "depolarizing":
        return [math.sqrt(1.0 - 0.75 * p) * gates.I2] + [0.5 * sp * P for P in (gates.X, gates.Y, gates.Z)]
    raise InvalidProbability(f"unknown noise kind {kind!r}")


@dataclass(frozen=True)
class NoiseChannel:
    kind: str
    p: float

    @property
    def kraus(self) -> list[np.ndarray]:
        return kraus_ops(self.kind, self.p)


def two_qubit_kraus(a: NoiseChannel, b: NoiseChannel) -> list[np.ndarray]:
    """{K_i (x) M_j} in i-major order; K acts on the first (MSB) qubit."""
    return [np.kron(k, m) for k in a.kraus for m in b.kraus]


@dataclass(frozen=True)
class NoiseRule:
    mnemonics: frozenset | None  # None = every gate
    channel_a: NoiseChannel
    channel_b: NoiseChannel


@dataclass
class NoiseModel:
    """Gate class -> channel assignment; the first matching rule wins."""

    rules: list

    def __post_init__(self):
        seen: set = set()
        for rule in self.rules:
            names = rule.mnemonics or frozenset({"*"})
            if seen & names:
                raise InvalidProbability(f"gate class {sorted(seen & names)} assigned noise more than once")
            seen |= names

    def kraus_for(self, inst, n_qubits: int):
        for rule in self.rules:
            if rule.mnemonics is None or inst.name in rule.mnemonics:
                if n_qubits == 1:
                    return rule.channel_a.kraus
                return two_qubit_kraus(rule.channel_a, rule.channel_b)
        return None


def make_noise_model(kind: str, p: float, mnemonics=None) -> NoiseModel:
    ch = NoiseChannel(kind, p)
    ch.kraus  # validate eagerly
    return NoiseModel([NoiseRule(frozenset(mnemonics) if mnemonics else None, ch, ch)])


def parse_noise_spec(spec: str) -> NoiseModel:
    """kind:p[:MNEMONIC,...] (noise.py:122-137)."""
    parts = spec.split(":")
    if len(parts) not in (2, 3):
        raise InvalidProbability(f"bad noise spec {spec!r}; want kind:p[:gates]")
    kind = parts[0].strip().lower()
    if kind not in KINDS:
        raise InvalidProbability(f"unknown noise kind {parts[0]!r}")
    try:
        p = float(parts[1])
    except ValueError:
        raise InvalidProbability(f"bad noise intensity {parts[1]!r}") from None
    names = [m.strip() for m in parts[2].split(",") if m.strip()] if len(parts) == 3 else None
    return make_noise_model(kind, p, names)
