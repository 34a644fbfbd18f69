"""Kraus channels and noise models (host side of the noisy-trajectory path).

Behaviour of `qcsim/noise.py:25-137` (the API and the error messages are part
of the reference interface): six single-qubit channels, two-qubit channels as
Kronecker products (operator index i*len(M) + j, K_i on the first / MSB
qubit), noise models whose first matching rule wins, and the CLI spec
`kind:p[:MNEMONIC,...]`.  Intensity convention: the flip channels are
noiseless at p = 1, damping and depolarising at p = 0.

The channels are kept as a table of (coefficient, operator) terms so the same
data drives the reference-shaped per-gate path (`statevector._noisy`, branch
weights from one on-device reduced-density pass), the batched general-channel
trajectories (`noisy_batch.py`) and the pre-sampled Pauli trajectories of
BASELINE config 5 (`workloads.sample_pauli_insertions`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import gates
from .errors import InvalidProbability

_P0_ONLY = np.array([[1, 0], [0, 0]], dtype=np.complex128)
_P1_ONLY = np.array([[0, 0], [0, 1]], dtype=np.complex128)
_LOWER = np.array([[0, 1], [0, 0]], dtype=np.complex128)  # |0><1|


def _terms(kind: str, p: float):
    """[(scalar a, matrix A, scalar b, matrix B)] per Kraus operator K = a A + b B."""
    sp, sq = math.sqrt(p), math.sqrt(1.0 - p)
    table = {
        # mixtures of a scaled identity and a scaled Pauli
        "bitflip": [(sp, gates.I2), (sq, gates.X)],
        "phaseflip": [(sp, gates.I2), (sq, gates.Z)],
        "bitphaseflip": [(sp, gates.I2), (sq, gates.Y)],
        "depolarizing": [(math.sqrt(1.0 - 0.75 * p), gates.I2), (0.5 * sp, gates.X), (0.5 * sp, gates.Y),
                         (0.5 * sp, gates.Z)],
        # damping: K0 = |0><0| + sqrt(1-p) |1><1|, K1 = sqrt(p) x (|0><1| or |1><1|)
        "ampdamp": [((1.0, _P0_ONLY), (sq, _P1_ONLY)), (sp, _LOWER)],
        "phasedamp": [((1.0, _P0_ONLY), (sq, _P1_ONLY)), (sp, _P1_ONLY)],
    }
    return table.get(kind)


KINDS = ("bitflip", "phaseflip", "bitphaseflip", "ampdamp", "phasedamp", "depolarizing")


def kraus_ops(kind: str, p: float) -> list[np.ndarray]:
    """Operator set of the named channel at intensity p (noise.py:35-64)."""
    if not 0.0 <= p <= 1.0:
        raise InvalidProbability(f"noise intensity {p} outside [0, 1]")
    spec = _terms(kind, p)
    if spec is None:
        raise InvalidProbability(f"unknown noise kind {kind!r}")
    ops = []
    for term in spec:
        parts = term if isinstance(term[0], tuple) else (term,)
        ops.append(sum((c * m for c, m in parts), np.zeros((2, 2), dtype=np.complex128)))
    return ops


@dataclass(frozen=True)
class NoiseChannel:
    kind: str
    p: float

    @property
    def kraus(self) -> list[np.ndarray]:
        return kraus_ops(self.kind, self.p)


def two_qubit_kraus(a: NoiseChannel, b: NoiseChannel) -> list[np.ndarray]:
    """{K_i (x) M_j}, index i * len(M) + j; K acts on the first (MSB) qubit."""
    mb = b.kraus
    return [np.kron(ka, mb[j]) for ka in a.kraus for j in range(len(mb))]


@dataclass(frozen=True)
class NoiseRule:
    mnemonics: frozenset | None  # None = every gate
    channel_a: NoiseChannel
    channel_b: NoiseChannel


@dataclass
class NoiseModel:
    """Gate class -> channel assignment; the first matching rule wins (a gate class
    may be assigned only once; the catch-all rule counts as the class "*")."""

    rules: list
    _claimed: dict = field(default_factory=dict, init=False, repr=False)

    def __post_init__(self):
        for idx, rule in enumerate(self.rules):
            names = rule.mnemonics if rule.mnemonics else frozenset({"*"})
            clash = sorted(n for n in names if n in self._claimed)
            if clash:
                raise InvalidProbability(f"gate class {clash} assigned noise more than once")
            self._claimed.update((n, idx) for n in names)

    def rule_for(self, name: str):
        for rule in self.rules:
            if rule.mnemonics is None or name in rule.mnemonics:
                return rule
        return None

    def kraus_for(self, inst, n_qubits: int):
        rule = self.rule_for(inst.name)
        if rule is None:
            return None
        return rule.channel_a.kraus if n_qubits == 1 else two_qubit_kraus(rule.channel_a, rule.channel_b)


def make_noise_model(kind: str, p: float, mnemonics=None) -> NoiseModel:
    channel = NoiseChannel(kind, p)
    kraus_ops(kind, p)  # reject a bad kind / intensity when the model is built
    return NoiseModel([NoiseRule(frozenset(mnemonics) if mnemonics else None, channel, channel)])


def parse_noise_spec(spec: str) -> NoiseModel:
    """kind:p[:MNEMONIC,...] (noise.py:122-137)."""
    fields = spec.split(":")
    if not 2 <= len(fields) <= 3:
        raise InvalidProbability(f"bad noise spec {spec!r}; want kind:p[:gates]")
    kind_txt, p_txt = fields[0], fields[1]
    kind = kind_txt.strip().lower()
    if kind not in KINDS:
        raise InvalidProbability(f"unknown noise kind {kind_txt!r}")
    try:
        p = float(p_txt)
    except ValueError:
        raise InvalidProbability(f"bad noise intensity {p_txt!r}") from None
    names = None
    if len(fields) == 3:
        names = [tok.strip() for tok in fields[2].split(",") if tok.strip()]
    return make_noise_model(kind, p, names)
