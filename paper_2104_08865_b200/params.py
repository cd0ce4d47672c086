"""Variant parameter sets -- same names and fields as the reference's
``halftimehash.params`` (pkg/src/halftimehash/params.py:46-237).

These are immutable host-side descriptions.  The CUDA kernels carry the same
constants at compile time (csrc/variants.cuh); tests check the two agree
through ``hth_variant_geometry``.
"""

from __future__ import annotations

from dataclasses import dataclass


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

    @property
    def rows(self) -> int:
        return len(self.entries)

    @property
    def cols(self) -> int:
        return len(self.entries[0])


@dataclass(frozen=True)
class ErasureCode:
    """Systematic GF(16) code (params.py:72-102)."""

    arity_in: int
    arity_out: int
    min_distance: int
    kind: str
    parity_rows: tuple


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
