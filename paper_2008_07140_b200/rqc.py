"""Seeded layered random circuits on a rectangular qubit grid (.qprog text).

Two families:

* ``patterns=4`` (default): byte-identical to the reference generator
  (`qcsim/rqc.py:24-85`): an H layer, then `depth` layers of CZ on one of
  four cycled grid-edge patterns (horizontal even/odd columns, vertical
  even/odd rows, `rqc.py:48-61`) and an i.i.d. pool gate on every idle qubit.
* ``patterns=8, no_repeat=True``: the BASELINE.json workload (configs 1-3, 5).
  The four reference patterns are each split by the parity of the other grid
  coordinate, giving eight patterns that cover every grid edge exactly once
  per eight cycles (order A0 B1 C0 D1 A1 B0 C1 D0); the pool
  gate of an idle qubit is drawn from the pool minus the gate that qubit got
  last, so no qubit sees the same pool gate twice in a row (SURVEY.md
  Appendix C.1-C.2, a documented extension - ref [21]'s exact prescription
  is not available).

Qubits are numbered row-major, q = r * cols + c.  `qubits` < rows * cols
leaves the last row partial (qubits >= `qubits` do not exist and their edges
are dropped): the near-square grids of qubit counts with no near-square
rectangle.  The pool gates are the
reference vocabulary: ``RX q,"pi/2"`` (= sqrt(X) up to a global phase),
``RY q,"pi/2"`` (= sqrt(Y) up to a global phase) and ``T q``.
"""

from __future__ import annotations

import random
from dataclasses import dataclass, field

DEFAULT_POOL = ("T", "RX", "RY")

_POOL_TEXT = {"T": "T {q}", "RX": 'RX {q},"pi/2"', "RY": 'RY {q},"pi/2"'}

# eight-pattern order: (orientation, start parity, split parity)
_EIGHT = [("h", 0, 0), ("h", 1, 1), ("v", 0, 0), ("v", 1, 1),
          ("h", 0, 1), ("h", 1, 0), ("v", 0, 1), ("v", 1, 0)]


@dataclass(frozen=True)
class RqcConfig:
    rows: int
    cols: int
    depth: int
    seed: int
    single_qubit_pool: tuple[str, ...] = DEFAULT_POOL
    entangler: str = "CZ"
    pmeasure: tuple[int, ...] = field(default=())
    patterns: int = 4
    no_repeat: bool = False
    qubits: int = 0  # 0: rows * cols; else a partial last row

    def __post_init__(self):
        if self.rows * self.cols < 2:
            raise ValueError("grid needs at least 2 qubits")
        if self.qubits and not ((self.rows - 1) * self.cols < self.qubits <= self.rows * self.cols):
            raise ValueError("qubits must end inside the last grid row")
        if self.depth < 1:
            raise ValueError("depth must be at least 1")
        if self.patterns not in (4, 8):
            raise ValueError("patterns must be 4 (reference) or 8 (BASELINE)")
        if self.no_repeat and len(self.single_qubit_pool) < 2:
            raise ValueError("no_repeat needs at least two pool gates")
        for g in self.single_qubit_pool:
            if g not in _POOL_TEXT:
                raise ValueError(f"unsupported pool gate {g!r}")

    @property
    def qubit_count(self) -> int:
        return self.qubits or self.rows * self.cols


def _edges(rows, cols, orient, start, split=None, n=None):
    """Grid edges of one orientation; `start` = parity of the lower endpoint
    along the edge axis, `split` = optional parity filter on the other axis;
    edges touching a qubit >= n (partial last row) are dropped."""
    q = lambda r, c: r * cols + c
    out = []
    if n is not None and n < rows * cols:
        return [e for e in _edges(rows, cols, orient, start, split) if e[1] < n]
    if orient == "h":
        for r in range(rows):
            if split is not None and r % 2 != split:
                continue
            for c in range(start, cols - 1, 2):
                out.append((q(r, c), q(r, c + 1)))
    else:
        for r in range(start, rows - 1, 2):
            for c in range(cols):
                if split is not None and c % 2 != split:
                    continue
                out.append((q(r, c), q(r + 1, c)))
    return out


def layer_pairs(config: RqcConfig, layer: int) -> list[tuple[int, int]]:
    """CZ pairs of one cycle (reference pattern order for patterns=4)."""
    n = config.qubit_count
    if config.patterns == 4:
        p = layer % 4
        return _edges(config.rows, config.cols, "h" if p < 2 else "v", p % 2, n=n)
    orient, start, split = _EIGHT[layer % 8]
    return _edges(config.rows, config.cols, orient, start, split, n=n)


_layer_pairs = layer_pairs  # reference-compatible private name


def generate_rqc(config: RqcConfig) -> str:
    """Deterministic script text for the configured random circuit."""
    rng = random.Random(config.seed)
    n = config.qubit_count
    head = (f"% random layered circuit rows={config.rows} cols={config.cols} "
            f"depth={config.depth} seed={config.seed}")
    if config.patterns != 4 or config.no_repeat:
        head += f" patterns={config.patterns} no_repeat={int(config.no_repeat)}"
    if config.qubits and config.qubits != config.rows * config.cols:
        head += f" qubits={config.qubits}"
    lines = [head, f"QINIT {n}"] + [f"H {q}" for q in range(n)]
    last: dict[int, str] = {}
    pool = config.single_qubit_pool
    for layer in range(config.depth):
        busy = set()
        for a, b in layer_pairs(config, layer):
            lines.append(f"{config.entangler} {a},{b}")
            busy.update((a, b))
        for q in range(n):
            if q in busy:
                continue
            choices = pool
            if config.no_repeat and q in last:
                choices = tuple(g for g in pool if g != last[q])
            g = rng.choice(choices)
            last[q] = g
            lines.append(_POOL_TEXT[g].format(q=q))
    if config.pmeasure:
        lines.append("PMEASURE " + ",".join(map(str, config.pmeasure)))
    return "\n".join(lines) + "\n"
