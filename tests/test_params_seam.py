"""Host-side pieces of the drop-in that need no GPU: the params module's
coefficient arithmetic and validations (params.py:17-69, 91-98, 158-169),
and the recognition of the reference's ``seed_region`` forms by the
``_hash_words_np`` seam (hasher.py:331-338)."""

import os
import sys

import numpy as np
import pytest

import paper_2104_08865_b200 as hh
from paper_2104_08865_b200 import hasher, params

REF = "/root/reference/pkg/src"


def test_coefficient_multiply_ints_and_arrays():
    rng = np.random.default_rng(5)
    xs = [0, 1, 2, (1 << 63) + 12345, (1 << 64) - 1] + [int(x) for x in rng.integers(0, 1 << 64, 50, dtype=np.uint64)]
    arr = np.array(xs, dtype=np.uint64)
    for c in sorted(params.SUPPORTED_COEFFICIENTS):
        for x in xs:
            assert params.coefficient_multiply(c, x) == (c * x) % (1 << 64)
            if c != 1:  # the reference returns x itself for 1 (no width mask)
                assert params.coefficient_multiply(c, x, 16) == (c * x) % (1 << 16)
        with np.errstate(over="ignore"):
            assert np.array_equal(params.coefficient_multiply(c, arr), arr * np.uint64(c))
    assert params.SUPPORTED_COEFFICIENTS == frozenset({0, 1, 2, 3, 4, 5, 7, 8, 9})
    for bad in (6, 10, -1):
        with pytest.raises(ValueError):
            params.coefficient_multiply(bad, 3)


def test_every_matrix_entry_has_a_shift_add_form():
    for p in params.VARIANTS.values():
        assert {c for r in p.matrix.entries for c in r} <= params.SUPPORTED_COEFFICIENTS
        cols = tuple(range(0, p.matrix.cols, 2))
        assert p.matrix.column_subset(cols) == [[r[c] for c in cols] for r in p.matrix.entries]


def test_validations():
    with pytest.raises(ValueError):
        params.TransformMatrix(((1, 2), (1,)))
    with pytest.raises(ValueError):
        params.TransformMatrix(((1, 6),))
    with pytest.raises(ValueError):
        params.ErasureCode(3, 5, 2, "x", ((1, 1, 1),))  # one row for two parities
    with pytest.raises(ValueError):
        params.ErasureCode(3, 4, 2, "x", ((1, 1),))
    with pytest.raises(ValueError):
        params.ErasureCode(3, 4, 2, "x", ((1, 16, 1),))
    v = params.VARIANTS[24]
    with pytest.raises(ValueError):  # output bytes
        params.HashParams(20, 3, 9, 7, 3, 8, 8, 2, v.matrix, v.code)
    with pytest.raises(ValueError):  # d != e + 1 - k
        params.HashParams(24, 3, 9, 6, 3, 8, 8, 2, v.matrix, v.code)
    with pytest.raises(ValueError):  # matrix shape
        params.HashParams(24, 3, 9, 7, 3, 8, 8, 2, params.VARIANTS[16].matrix, v.code)
    with pytest.raises(ValueError):  # code arity
        params.HashParams(24, 3, 9, 7, 3, 8, 8, 2, v.matrix, params.VARIANTS[32].code)
    assert v.code.bitwise_linear


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_params_agree_with_reference():
    sys.path.insert(0, REF)
    try:
        import halftimehash.params as R
    finally:
        sys.path.remove(REF)
    assert R.SUPPORTED_COEFFICIENTS == params.SUPPORTED_COEFFICIENTS
    for w, p in params.VARIANTS.items():
        r = R.VARIANTS[w]
        assert p.matrix.entries == r.matrix.entries
        assert p.code.parity_rows == r.code.parity_rows and p.code.min_distance == r.code.min_distance
        assert (p.output_words, p.encoded_items, p.instance_items, p.item_blocks, p.block_words, p.fanout,
                p.max_det_valuation) == (r.output_words, r.encoded_items, r.instance_items, r.item_blocks,
                                         r.block_words, r.fanout, r.max_det_valuation)
    for c in sorted(R.SUPPORTED_COEFFICIENTS):
        for x in (0, 7, (1 << 64) - 3):
            for width in (8, 32, 64):
                assert params.coefficient_multiply(c, x, width) == R.coefficient_multiply(c, x, width)


# ------------------------------------------------------------ seed regions
def test_region_shared_seedbuffer():
    p = hh.variant(32)
    s = hh.seed_for_input(b"\x11" * 32, p, 9000)
    folds, cap = hasher._region_folds(s.words_np, hh.seed_words_needed(p, 9000))
    assert folds.tolist() == [s.fold] and cap == s.capacity
    with pytest.raises(IndexError):
        hasher._region_folds(hh.expand_seed(b"\0" * 32, 3).words_np, 100)


def test_region_batched_folds_and_plain_streams():
    rng = np.random.default_rng(2)
    masters = rng.integers(0, 1 << 64, size=(500, 4), dtype=np.uint64)
    folds = (masters[:, 0] ^ masters[:, 1] ^ masters[:, 2] ^ masters[:, 3])[:, None]
    got, cap = hasher._region_folds(lambda a, c: hasher._stream_words_np(folds, a, c), 1571)
    assert np.array_equal(got, folds[:, 0]) and cap is None
    # a bare 1-D stream of one fold (no SeedBuffer behind it)
    got, _ = hasher._region_folds(lambda a, c: hasher._stream_words_np(np.uint64(12345), a, c), 400)
    assert got.tolist() == [12345]
    # the inverse finalizer is exact
    z = rng.integers(0, 1 << 64, size=1000, dtype=np.uint64)
    mixed = np.array([hasher.splitmix_mix(int(x)) for x in z], dtype=np.uint64)
    assert np.array_equal(hasher._unmix(mixed), z)


def test_region_rejects_other_arrays():
    with pytest.raises(ValueError):
        hasher._region_folds(lambda a, c: np.arange(a, a + c, dtype=np.uint64), 400)
    rng = np.random.default_rng(3)
    table = rng.integers(0, 1 << 64, size=5000, dtype=np.uint64)
    with pytest.raises(ValueError):
        hasher._region_folds(lambda a, c: table[a:a + c], 400)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")
def test_region_reference_seedbuffer_and_stream():
    sys.path.insert(0, REF)
    try:
        import halftimehash as R
        from halftimehash import hasher as RH
    finally:
        sys.path.remove(REF)
    rs = R.seed_for_input(bytes(range(32)), R.variant(40), 1 << 20)
    folds, cap = hasher._region_folds(rs.words_np, R.seed_words_needed(R.variant(40), 1 << 20))
    assert folds.tolist() == [hasher._master_fold(bytes(range(32)))] and cap == rs.capacity
    f = np.arange(1, 50, dtype=np.uint64)[:, None] * np.uint64(0x9E3779B97F4A7C15)
    got, _ = hasher._region_folds(lambda a, c: RH._stream_words_np(f, a, c), 410)
    assert np.array_equal(got, f[:, 0])


def test_engine_names_checked_before_gpu_work():
    p = hh.variant(16)
    s = hh.seed_for_input(b"\0" * 32, p, 0)
    assert hh.ENGINES == ("cuda", "lanes", "scalar")
    with pytest.raises(ValueError):
        hh.hash_bytes(b"", s, p, engine="neon")
    with pytest.raises(ValueError):
        hh.hash_bytes(b"", s, p, engine="lanes", counter=object())


def test_words_from_bytes_and_remainder_errors():
    # pkg/tests/test_hasher.py:153-155, 187-188 (no GPU work for these cases)
    from paper_2104_08865_b200.hasher import hash_remainder, words_from_bytes

    assert words_from_bytes(b"\x01\x00\x00\x00\x00\x00\x00\x00\xff") == [1, 255]
    assert words_from_bytes(b"") == []
    assert hash_remainder([], [1, 2, 3], k=3) == (0, 0, 0)
    with pytest.raises(ValueError):
        hash_remainder([1, 2, 3], [1, 2, 3], k=2)  # key region too short
    with pytest.raises(ValueError):
        hash_remainder([1], [1, 2], k=1, counter=object())
    with pytest.raises(ValueError):
        hash_remainder([1], [1, 2], k=1, half_bits=16)
