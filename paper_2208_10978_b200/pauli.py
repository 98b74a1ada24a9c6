"""Pauli strings and weighted sums -- the Hamiltonian input type of the engine.

Duck-compatible with the reference's pauli.PauliString / PauliTerm / PauliSum
(pauli.py:58-257): a string is a sorted tuple of ``(qubit, axis)`` factors,
a term carries a complex coefficient, and Hermiticity means real
coefficients (pauli.py:230-236).  Reference objects can be passed to the
engine directly; these classes exist so the engine, its tests and its
benchmarks run without the reference installed.  Text I/O follows the
reference's interchange format (pauli.py:260-314): one term per line,
``<real> [<imag>] <AXIS><index> ...``.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Iterator, TextIO

import numpy as np

from .errors import FormatError

AXES = ("X", "Y", "Z")

# (a, b) -> (phase, product axis or None)
_PRODUCT = {
    ("X", "Y"): (1j, "Z"), ("Y", "X"): (-1j, "Z"),
    ("Y", "Z"): (1j, "X"), ("Z", "Y"): (-1j, "X"),
    ("Z", "X"): (1j, "Y"), ("X", "Z"): (-1j, "Y"),
}


@dataclass(frozen=True)
class PauliString:
    factors: tuple[tuple[int, str], ...] = ()

    def __post_init__(self):
        seen = set()
        for q, axis in self.factors:
            if q < 0:
                raise ValueError(f"negative qubit index {q}")
            if axis not in AXES:
                raise ValueError(f"invalid Pauli axis {axis!r}")
            if q in seen:
                raise ValueError(f"duplicate qubit index {q}")
            seen.add(q)
        object.__setattr__(self, "factors", tuple(sorted(self.factors)))

    @classmethod
    def from_map(cls, support) -> "PauliString":
        return cls(tuple(support.items()))

    @classmethod
    def from_label(cls, label: str) -> "PauliString":
        out: dict[int, str] = {}
        for tok in label.split():
            axis, digits = tok[0].upper(), tok[1:]
            if axis not in AXES or not digits.isdigit():
                raise FormatError(f"bad Pauli factor {tok!r}")
            if int(digits) in out:
                raise FormatError(f"duplicate qubit index in {label!r}")
            out[int(digits)] = axis
        return cls.from_map(out)

    @property
    def support(self) -> tuple[int, ...]:
        return tuple(q for q, _ in self.factors)

    @property
    def weight(self) -> int:
        return len(self.factors)

    def is_identity(self) -> bool:
        return not self.factors

    def max_index(self) -> int:
        return self.factors[-1][0] if self.factors else -1

    def masks(self) -> tuple[int, int, int]:
        """(x, y, z) bit masks, as statevector._string_masks (statevector.py:77-88)."""
        x = y = z = 0
        for q, axis in self.factors:
            if axis == "X":
                x |= 1 << q
            elif axis == "Y":
                y |= 1 << q
            else:
                z |= 1 << q
        return x, y, z

    def __str__(self) -> str:
        return " ".join(f"{a}{q}" for q, a in self.factors) or "I"

    def __iter__(self) -> Iterator[tuple[int, str]]:
        return iter(self.factors)


def multiply(a: PauliString, b: PauliString) -> tuple[complex, PauliString]:
    """Operator product a @ b as (phase, string)."""
    phase: complex = 1
    acc = dict(a.factors)
    for q, axis in b.factors:
        prev = acc.pop(q, None)
        if prev is None:
            acc[q] = axis
        elif prev != axis:
            ph, prod = _PRODUCT[(prev, axis)]
            phase *= ph
            acc[q] = prod
    return phase, PauliString.from_map(acc)


@dataclass(frozen=True)
class PauliTerm:
    coefficient: complex
    string: PauliString


@dataclass(frozen=True)
class PauliSum:
    terms: tuple[PauliTerm, ...] = ()

    def __post_init__(self):
        object.__setattr__(self, "terms", tuple(self.terms))

    @classmethod
    def from_terms(cls, terms: Iterable[tuple[complex, PauliString]]) -> "PauliSum":
        return cls(tuple(PauliTerm(c, s) for c, s in terms))

    def __len__(self) -> int:
        return len(self.terms)

    def __iter__(self) -> Iterator[PauliTerm]:
        return iter(self.terms)

    def __add__(self, other: "PauliSum") -> "PauliSum":
        return PauliSum(self.terms + other.terms)

    def __mul__(self, scalar: complex) -> "PauliSum":
        return PauliSum(tuple(PauliTerm(t.coefficient * scalar, t.string) for t in self.terms))

    __rmul__ = __mul__

    def n_qubits(self) -> int:
        return max((t.string.max_index() for t in self.terms), default=-1) + 1

    def is_hermitian(self, tol: float = 1e-10) -> bool:
        return all(abs(complex(t.coefficient).imag) <= tol for t in self.terms)

    def simplify(self, drop_threshold: float = 1e-12) -> "PauliSum":
        """Combine like strings, drop small coefficients, sort canonically."""
        acc: dict[PauliString, complex] = {}
        for t in self.terms:
            acc[t.string] = acc.get(t.string, 0) + complex(t.coefficient)
        kept = [PauliTerm(c, s) for s, c in acc.items() if c != 0 and abs(c) >= drop_threshold]
        kept.sort(key=lambda t: t.string.factors)
        return PauliSum(tuple(kept))


def term_arrays(h, n_qubits: int):
    """Hamiltonian -> (x, y, z, coef_re, coef_im) numpy arrays for the C ABI.

    Accepts this module's PauliSum or the reference's (duck typed).  Raises
    ValueError on indices >= n_qubits, like statevector._string_masks
    (statevector.py:80-81)."""
    n = len(h.terms)
    x = np.zeros(n, dtype=np.uint64)
    y = np.zeros(n, dtype=np.uint64)
    z = np.zeros(n, dtype=np.uint64)
    cr = np.zeros(n, dtype=np.float64)
    ci = np.zeros(n, dtype=np.float64)
    for k, term in enumerate(h.terms):
        xm = ym = zm = 0
        for q, axis in term.string.factors:
            if q >= n_qubits:
                raise ValueError(f"string index {q} out of range for {n_qubits} qubits")
            if axis == "X":
                xm |= 1 << q
            elif axis == "Y":
                ym |= 1 << q
            else:
                zm |= 1 << q
        x[k], y[k], z[k] = xm, ym, zm
        c = complex(term.coefficient)
        cr[k], ci[k] = c.real, c.imag
    return x, y, z, cr, ci


def read_pauli_sum(stream: TextIO) -> PauliSum:
    terms = []
    for lineno, raw in enumerate(stream, start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        try:
            re_part = float(tok[0])
        except ValueError:
            raise FormatError(f"line {lineno}: expected a real coefficient, got {tok[0]!r}")
        im_part, rest = 0.0, tok[1:]
        if rest:
            try:
                im_part = float(rest[0])
                rest = rest[1:]
            except ValueError:
                pass
        try:
            s = PauliString.from_label(" ".join(rest))
        except FormatError as e:
            raise FormatError(f"line {lineno}: {e}")
        terms.append(PauliTerm(complex(re_part, im_part), s))
    return PauliSum(tuple(terms))


def write_pauli_sum(h, stream: TextIO) -> None:
    for t in h.terms:
        c = complex(t.coefficient)
        head = repr(c.real) if c.imag == 0.0 else f"{c.real!r} {c.imag!r}"
        ops = "" if not t.string.factors else str(t.string)
        stream.write(f"{head} {ops}".rstrip() + "\n")
