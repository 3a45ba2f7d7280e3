"""Circuit data model and the optimized text format — host mirror of the
reference's `quokka.circuit` for the simulation path.

Names, fields, validation messages and the text grammar follow
/root/reference/pkg/src/quokka/circuit.py (cited per item). Parsing goes
through the native parser of libqkb200.so (`qk_parse_text`), the same code the
`Quokka` CLI path and `qk_load_text` use, so there is a single implementation
of the grammar. The reference's own objects are accepted everywhere these are
(duck-typed on `.gates`, `.out_set`, `.local_set`, `.kind.value`).
"""
from __future__ import annotations

import cmath
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .errors import ParseError

__all__ = ["DEFAULT_ANGLE", "GateKind", "Gate", "LayoutParams", "GateBlock", "InMemSwap",
           "CrossRankSwap", "RawCircuit", "OptimizedCircuit", "ParseError", "parse_optimized",
           "serialize_optimized", "gate_matrix", "replay_permutation",
           "apply_swap_to_permutation", "default_params", "DIAGONAL_KINDS"]

DEFAULT_ANGLE = math.pi / 4                   # circuit.py:21
_SQRT1_2 = 1.0 / math.sqrt(2.0)               # circuit.py:23


class GateKind(Enum):                         # circuit.py:34-45
    H = "H"
    X = "X"
    U = "U"
    CX = "CX"
    CP = "CP"
    SWAP = "SWAP"
    RX = "RX"
    RY = "RY"
    RZ = "RZ"
    RZZ = "RZZ"
    D = "D"


_TARGETS = {"H": 1, "X": 1, "U": 1, "RX": 1, "RY": 1, "RZ": 1, "CX": 2, "CP": 2, "SWAP": 2,
            "RZZ": 2}                          # circuit.py:50-54
_ANGLES = {"H": 0, "X": 0, "CX": 0, "SWAP": 0, "CP": 1, "RX": 1, "RY": 1, "RZ": 1, "RZZ": 1,
           "U": 3}                             # circuit.py:55-59
DIAGONAL_KINDS = frozenset({GateKind.RZ, GateKind.RZZ, GateKind.CP, GateKind.D})
SYMMETRIC_KINDS = frozenset({GateKind.SWAP, GateKind.RZZ, GateKind.CP, GateKind.D})


def default_params(kind: GateKind) -> tuple:  # circuit.py:114-115
    return (DEFAULT_ANGLE,) * _ANGLES[kind.value]


@dataclass(frozen=True)
class Gate:                                   # circuit.py:73-111
    kind: GateKind
    targets: tuple
    gid: int
    params: tuple = ()

    def __post_init__(self):
        name = self.kind.value
        if len(set(self.targets)) != len(self.targets):
            raise ValueError(f"duplicate targets in {name} gate {self.gid}")
        if self.kind is GateKind.D:
            k = len(self.targets)
            if k < 2:
                raise ValueError("fused diagonal needs at least 2 qubits")
            if len(self.params) != 1 << k:
                raise ValueError(f"D{k} needs {1 << k} diagonal entries, got {len(self.params)}")
            return
        if len(self.targets) != _TARGETS[name]:
            raise ValueError(f"{name} takes {_TARGETS[name]} targets")
        if len(self.params) != _ANGLES[name]:
            raise ValueError(f"{name} takes {_ANGLES[name]} parameters")

    @property
    def is_diagonal(self) -> bool:
        return self.kind in DIAGONAL_KINDS


@dataclass(frozen=True)
class RawCircuit:                             # circuit.py:118-128 (input of run_gate_by_gate)
    num_qubits: int
    gates: tuple


@dataclass(frozen=True)
class LayoutParams:                           # circuit.py:131-163
    n: int
    c: int
    r: int = 0
    cl: int = 2
    f: int = 0
    b: int | None = None

    def __post_init__(self):
        n, r = self.n, self.r
        if self.b is None:
            object.__setattr__(self, "b", n - r)
        checks = (
            (0 <= r <= n, f"need 0 <= R <= N, got R={r}, N={n}"),
            (0 < self.c <= n - r, f"need 0 < C <= N-R, got C={self.c}, N-R={n - r}"),
            (0 <= self.cl <= self.c, f"need CL <= C, got CL={self.cl}, C={self.c}"),
            (0 <= self.f <= self.c, f"need F <= C, got F={self.f}, C={self.c}"),
            (0 <= self.b <= n - r, f"need B <= N-R, got B={self.b}, N-R={n - r}"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    @property
    def local_qubits(self) -> int:
        return self.n - self.r

    @property
    def num_ranks(self) -> int:
        return 1 << self.r


@dataclass(frozen=True)
class GateBlock:                              # circuit.py:166-168
    gates: tuple


@dataclass(frozen=True)
class InMemSwap:                              # circuit.py:171-180
    out_set: tuple
    in_set: tuple

    def __post_init__(self):
        if len(self.out_set) != len(self.in_set):
            raise ValueError("swap sets must have equal size")
        if set(self.out_set) & set(self.in_set):
            raise ValueError("swap sets must be disjoint")


@dataclass(frozen=True)
class CrossRankSwap:                          # circuit.py:183-190
    local_set: tuple
    rank_set: tuple

    def __post_init__(self):
        if len(self.local_set) != len(self.rank_set):
            raise ValueError("swap sets must have equal size")


def apply_swap_to_permutation(perm: list, a, b) -> None:    # circuit.py:196-199
    for pa, pb in zip(sorted(a), sorted(b)):
        perm[pa], perm[pb] = perm[pb], perm[pa]


def replay_permutation(instructions, n: int) -> tuple:     # circuit.py:202-210
    perm = list(range(n))
    for ins in instructions:
        if hasattr(ins, "out_set"):
            apply_swap_to_permutation(perm, ins.out_set, ins.in_set)
        elif hasattr(ins, "local_set"):
            apply_swap_to_permutation(perm, ins.local_set, ins.rank_set)
    return tuple(perm)


@dataclass(frozen=True)
class OptimizedCircuit:                       # circuit.py:213-227
    num_qubits: int
    layout: LayoutParams
    instructions: tuple
    final_permutation: tuple = field(default=())

    def __post_init__(self):
        if not self.final_permutation:
            object.__setattr__(self, "final_permutation",
                               replay_permutation(self.instructions, self.num_qubits))

    def gate_blocks(self) -> list:
        return [i for i in self.instructions if isinstance(i, GateBlock)]


# ---------------------------------------------------------------------------
# text format


def _unpack(words: np.ndarray, params: np.ndarray) -> list:
    """Packed records (qkb200.h) + gate-id side channel -> instruction objects."""
    out, i, pi = [], 0, 0
    records = []
    while i < len(words) and words[i] != -1:
        kind, cnt = int(words[i]), int(words[i + 1])
        i += 2
        if kind == _lib.INS_BLOCK:
            gates = []
            for _ in range(cnt):
                code, nt = int(words[i]), int(words[i + 1])
                targets = tuple(int(t) for t in words[i + 2:i + 2 + nt])
                npar = int(words[i + 2 + nt])
                i += 3 + nt
                gates.append((code, targets, params[pi:pi + npar]))
                pi += npar
            records.append(("B", gates))
        else:
            a = tuple(int(t) for t in words[i:i + cnt])
            b = tuple(int(t) for t in words[i + cnt:i + 2 * cnt])
            i += 2 * cnt
            records.append(("S" if kind == _lib.INS_SQS else "X", a, b))
    ids = [int(x) for x in words[i + 2:]] if i < len(words) else []
    gi = 0
    for rec in records:
        if rec[0] == "B":
            gates = []
            for code, targets, par in rec[1]:
                name = _lib.CODE_KIND[code]
                if name == "D":
                    vals = tuple(complex(par[2 * j], par[2 * j + 1]) for j in range(len(par) // 2))
                else:
                    vals = tuple(float(x) for x in par)
                gates.append(Gate(GateKind(name), targets, ids[gi], vals))
                gi += 1
            out.append(GateBlock(tuple(gates)))
        elif rec[0] == "S":
            out.append(InMemSwap(rec[1], rec[2]))
        else:
            out.append(CrossRankSwap(rec[1], rec[2]))
    return out


def parse_optimized(text: str, layout: LayoutParams) -> OptimizedCircuit:
    """circuit.py:347-397 — count line + payload records; '#' comments ignored."""
    words, params = _lib.parse_text(text, layout.n, layout.local_qubits, layout.c)
    return OptimizedCircuit(layout.n, layout, tuple(_unpack(words, params)))


def _num(x: float) -> str:
    return repr(float(x))


def gate_line(g) -> str:                      # circuit.py:312-323
    name = _lib.kind_name(g.kind)
    if name == "D":
        toks = [f"D{len(g.targets)}", *map(str, g.targets)]
        for e in g.params:
            e = complex(e)
            toks += [_num(e.real), _num(e.imag)]
        return " ".join(toks)
    toks = [name, *map(str, g.targets), str(g.gid)]
    if tuple(g.params) != (DEFAULT_ANGLE,) * _ANGLES[name]:
        toks += [_num(p) for p in g.params]
    return " ".join(toks)


def serialize_optimized(circuit) -> str:      # circuit.py:400-414
    lines = []
    for ins in circuit.instructions:
        if hasattr(ins, "gates"):
            lines.append(str(len(ins.gates)))
            lines += [gate_line(g) for g in ins.gates]
        elif hasattr(ins, "out_set"):
            lines += ["1", " ".join(["SQS", str(len(ins.out_set)), *map(str, ins.out_set),
                                     *map(str, ins.in_set)])]
        else:
            lines += ["1", " ".join(["CSQS", str(len(ins.local_set)), *map(str, ins.local_set),
                                     *map(str, ins.rank_set)])]
    return "\n".join(lines)


# ---------------------------------------------------------------------------
# gate matrices (circuit.py:420-463); targets[0] is the MSB of the matrix index


def gate_matrix(gate) -> np.ndarray:
    name = _lib.kind_name(gate.kind)
    p = gate.params
    if name == "H":
        return np.array([[1, 1], [1, -1]], dtype=complex) * _SQRT1_2
    if name == "X":
        return np.array([[0, 1], [1, 0]], dtype=complex)
    if name == "U":
        th, ph, lam = p
        ct, st = math.cos(th / 2), math.sin(th / 2)
        return np.array([[ct, -cmath.exp(1j * lam) * st],
                         [cmath.exp(1j * ph) * st, cmath.exp(1j * (ph + lam)) * ct]])
    if name in ("CX", "SWAP"):
        m = np.eye(4, dtype=complex)
        rows = (2, 3) if name == "CX" else (1, 2)
        m[list(rows)] = m[list(rows[::-1])]
        return m
    if name == "CP":
        return np.diag([1, 1, 1, cmath.exp(1j * p[0])])
    if name in ("RX", "RY"):
        co, si = math.cos(p[0] / 2), math.sin(p[0] / 2)
        off = -1j * si if name == "RX" else si
        return np.array([[co, -si if name == "RY" else off], [off, co]], dtype=complex)
    if name == "RZ":
        return np.diag([cmath.exp(-1j * p[0] / 2), cmath.exp(1j * p[0] / 2)])
    if name == "RZZ":
        lo, hi = cmath.exp(-1j * p[0] / 2), cmath.exp(1j * p[0] / 2)
        return np.diag([lo, hi, hi, lo])
    if name == "D":
        d = np.asarray(p, dtype=complex)
        if np.max(np.abs(np.abs(d) - 1.0)) > 1e-9:
            raise ValueError("non-unitary fused gate")
        return np.diag(d)
    raise ValueError(f"no matrix for {gate.kind}")
