"""Variant parameter sets -- same names and fields as the reference's
``halftimehash.params`` (pkg/src/halftimehash/params.py:46-237).

These are immutable host-side descriptions.  The CUDA kernels carry the same
constants at compile time (csrc/variants.cuh); tests check the two agree
through ``hth_variant_geometry``.
"""

from __future__ import annotations

from dataclasses import dataclass

MASK64 = (1 << 64) - 1

# Combine-matrix coefficients and their shift/add forms (params.py:15-29):
# coefficient -> (shift, op) with op +1 / -1 adding / subtracting x once
# more, 0 for a bare shift; 0 itself maps to None (the product is 0).
_FORMS = {0: None, 1: (0, 0), 2: (1, 0), 3: (1, 1), 4: (2, 0), 5: (2, 1), 7: (3, -1), 8: (3, 0), 9: (3, 1)}

#: coefficients that have a shift/add form (params.py:31)
SUPPORTED_COEFFICIENTS = frozenset(_FORMS)


def coefficient_multiply(coeff: int, x, width: int = 64):
    """``coeff * x mod 2**width`` by at most two shifts and one add/sub
    (params.py:32-43).  ``x``: a Python int or a numpy uint64 array.  The
    GPU kernels fold the same products into IMAD/LEA forms (csrc/engine.cuh
    mac_const); this host form is kept for the reference's callers.
    ValueError for a coefficient without a shift/add form."""
    if coeff not in _FORMS:
        raise ValueError(f"coefficient {coeff} has no shift/add form")
    m = (1 << width) - 1 if width < 64 else MASK64
    form = _FORMS[coeff]
    if form is None:
        return x & 0
    if coeff == 1:  # identity, unmasked, as the reference returns it (params.py:20)
        return x
    sh, op = form
    y = (x << sh) if sh else x
    if op > 0:
        y = y + x
    elif op < 0:
        y = y - x
    return y & m


def _xt4(a: int) -> int:
    t = (a >> 3) & 1
    return ((a << 1) & 0xF) ^ t ^ (t << 1)


def _mul4(a: int, b: int) -> int:
    acc, t = 0, b
    for i in range(4):
        if (a >> i) & 1:
            acc ^= t
        t = _xt4(t)
    return acc


def _inv4(a: int) -> int:
    return next(b for b in range(1, 16) if _mul4(a, b) == 1)


@dataclass(frozen=True)
class TransformMatrix:
    """Combine matrix: ``rows`` output blocks from ``cols`` hashed blocks (params.py:46-69)."""

    entries: tuple

    def __post_init__(self):  # params.py:52-58
        if len({len(r) for r in self.entries}) != 1:
            raise ValueError("ragged matrix")
        unsupported = sorted({c for r in self.entries for c in r} - SUPPORTED_COEFFICIENTS)
        if unsupported:
            raise ValueError(f"entries without a shift/add form: {unsupported}")

    @property
    def rows(self) -> int:
        return len(self.entries)

    @property
    def cols(self) -> int:
        return len(self.entries[0])

    def column_subset(self, cols: tuple) -> list:
        """The matrix restricted to columns ``cols`` (params.py:68-69)."""
        return [[r[c] for c in cols] for r in self.entries]


@dataclass(frozen=True)
class ErasureCode:
    """Systematic GF(16) code (params.py:72-102)."""

    arity_in: int
    arity_out: int
    min_distance: int
    kind: str
    parity_rows: tuple

    def __post_init__(self):  # params.py:91-98
        if len(self.parity_rows) != self.arity_out - self.arity_in:
            raise ValueError("parity row count must equal arity_out - arity_in")
        for r in self.parity_rows:
            if len(r) != self.arity_in:
                raise ValueError("parity row width must equal arity_in")
            if any(not 0 <= c < 16 for c in r):
                raise ValueError("parity coefficients must be GF(16) elements")

    @property
    def bitwise_linear(self) -> bool:
        return True


@dataclass(frozen=True)
class HashParams:
    """One output-width variant (params.py:133-182)."""

    output_bytes: int
    output_words: int
    encoded_items: int
    instance_items: int
    item_blocks: int
    block_words: int
    fanout: int
    max_det_valuation: int
    matrix: TransformMatrix
    code: ErasureCode

    def __post_init__(self):  # params.py:158-169
        k, e, d = self.output_words, self.encoded_items, self.instance_items
        checks = (
            (self.output_bytes == 8 * k, "output_bytes must be 8 * output_words"),
            (d == e + 1 - k, "instance_items must equal encoded_items + 1 - output_words"),
            ((self.matrix.rows, self.matrix.cols) == (k, e), "combine matrix shape mismatch"),
            ((self.code.arity_in, self.code.arity_out) == (d, e), "erasure code arity mismatch"),
            (self.code.min_distance >= k, "erasure code distance below output_words"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)

    @property
    def instance_blocks(self) -> int:
        return self.instance_items * self.item_blocks

    @property
    def instance_words(self) -> int:
        return self.instance_blocks * self.block_words

    @property
    def entropy_words(self) -> int:
        return self.encoded_items * self.item_blocks


def _xor_code(d: int) -> ErasureCode:
    return ErasureCode(d, d + 1, 2, "xor-parity", ((1,) * d,))


def _cauchy_code(d: int, p: int) -> ErasureCode:
    rows = tuple(tuple(_inv4(j ^ (p + i)) for i in range(d)) for j in range(p))
    return ErasureCode(d, d + p, p + 1, "repo-defined-linear", rows)


_M16 = TransformMatrix(((1, 0, 1, 1, 2, 1, 4), (0, 1, 1, 2, 1, 4, 1)))
_M24 = TransformMatrix(((0, 0, 1, 4, 1, 1, 2, 2, 1), (1, 1, 0, 0, 1, 4, 1, 2, 2), (1, 4, 1, 1, 0, 0, 2, 1, 2)))
_M32 = TransformMatrix(((0, 0, 0, 1, 1, 4, 2, 4, 1, 1), (0, 1, 2, 0, 0, 1, 1, 2, 4, 1),
                        (2, 0, 1, 0, 4, 0, 1, 1, 1, 1), (1, 1, 0, 1, 0, 0, 4, 1, 2, 8)))
_M40 = TransformMatrix(((1, 0, 0, 0, 0, 1, 1, 2, 4), (0, 1, 0, 0, 0, 1, 2, 1, 7), (0, 0, 1, 0, 0, 1, 3, 8, 5),
                        (0, 0, 0, 1, 0, 1, 4, 9, 8), (0, 0, 0, 0, 1, 1, 5, 3, 9)))

#   bytes  k  e   d  w  b  f  p   (params.py:217-221)
VARIANTS = {
    16: HashParams(16, 2, 7, 6, 2, 8, 8, 2, _M16, _xor_code(6)),
    24: HashParams(24, 3, 9, 7, 3, 8, 8, 2, _M24, _cauchy_code(7, 2)),
    32: HashParams(32, 4, 10, 7, 3, 8, 8, 3, _M32, _cauchy_code(7, 3)),
    40: HashParams(40, 5, 9, 5, 3, 8, 8, 3, _M40, _cauchy_code(5, 4)),
}


def variant(output_bytes: int) -> HashParams:
    """Validated parameter set for a 16/24/32/40-byte digest (params.py:230-237)."""
    try:
        return VARIANTS[output_bytes]
    except (KeyError, TypeError):
        raise ValueError(
            f"unsupported output width {output_bytes!r}; choose one of 16, 24, 32, 40"
        ) from None
