"""Host-side logic and the C-ABI boundary, CPU only (no kernel launches)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2104_08865_b200 as hh
from paper_2104_08865_b200 import _lib
from oracle import oracle_np as o

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "halftime_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hth_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    assert set(names) == set(_lib.EXPORTS)


def test_version_and_last_error():
    L = _lib.lib()
    assert L.hth_version() >= 100
    rc = L.hth_seed_words_needed(20, 0, ctypes.byref(ctypes.c_uint64()))
    assert rc == _lib.HTH_EINVAL
    assert b"unsupported output width" in L.hth_last_error()


@pytest.mark.parametrize("w", (16, 24, 32, 40))
def test_variant_geometry_matches_params(w):
    p = hh.variant(w)
    k, e, d, ww, m = (ctypes.c_int() for _ in range(5))
    _lib.check(_lib.lib().hth_variant_geometry(w, *(ctypes.byref(x) for x in (k, e, d, ww, m))))
    assert (k.value, e.value, d.value, ww.value, m.value) == (
        p.output_words, p.encoded_items, p.instance_items, p.item_blocks, p.instance_words)
    ov = o.variant(w)
    assert p.code.parity_rows == ov.parity
    assert p.matrix.entries == ov.matrix


def test_seed_layout_matches_oracle_and_budget():
    for w in (16, 24, 32, 40):
        p = hh.variant(w)
        for n in (0, 1, 1000, 167 * 8, 168 * 8, 10 ** 6, 1 << 20, 16 << 30):
            lay = hh.seed_layout(p, n)
            ol = o.layout(o.variant(w), n)
            assert lay.total_words == ol.total == hh.seed_words_needed(p, n)
            assert lay.levels == ol.levels
            assert lay.tree_start == ol.tree[0] and lay.finalize_start == ol.fin[0]
            assert lay.remainder_start == ol.rem
            k, b, f, h = p.output_words, 8, 8, lay.levels  # hasher.py:109-111 budget
            assert lay.total_words == p.entropy_words + (f - 1) * h * k + b * f * h * k + p.instance_words + k - 1


def test_seedbuffer_host_semantics():
    s = hh.expand_seed(bytes(range(32)), 100)
    assert s.words(0, 100) == [int(x) for x in o.splitmix_words(o.master_fold(bytes(range(32))), 0, 100)]
    assert s.words_np(5, 10).tolist() == s.words(5, 10)
    with pytest.raises(IndexError):
        s.word(100)
    with pytest.raises(IndexError):
        s.words(95, 10)
    with pytest.raises(ValueError):
        hh.expand_seed(b"\0" * 31, 4)
    with pytest.raises(ValueError):
        hh.SeedBuffer.from_master(b"\0" * 32, -1)
    empty = hh.expand_seed(b"\0" * 32, 0)
    assert empty.words(0, 0) == []
    fold = ctypes.c_uint64()
    _lib.check(_lib.lib().hth_master_fold(bytes(range(32)), ctypes.byref(fold)))
    assert fold.value == s.fold


def test_api_errors_before_any_gpu_work():
    p = hh.variant(24)
    with pytest.raises(ValueError):
        hh.variant(20)
    with pytest.raises(ValueError):
        hh.hash_bytes(b"", hh.seed_for_input(b"\0" * 32, p, 0), p, engine="avx2")
    with pytest.raises(ValueError):
        hh.hash_bytes(b"", hh.seed_for_input(b"\0" * 32, p, 0), p, engine="scalar", counter=object())
    with pytest.raises(hh.SeedSizeError):
        hh.hash_bytes(bytes(100000), hh.expand_seed(b"\0" * 32, 10), p)
    assert issubclass(hh.SeedSizeError, ValueError)


def test_cabi_seed_size_error_code():
    out = (ctypes.c_uint64 * 3)()
    rc = _lib.lib().hth_hash_fixed(24, None, 1, 4096, 4096, 0, None, 10, out, None, 0, None)
    assert rc == _lib.HTH_ESEEDSIZE
    with pytest.raises(hh.SeedSizeError):
        _lib.check(rc)


def test_digest_type():
    d = hh.Digest((1, 2, 3))
    assert d.bytes == (1).to_bytes(8, "little") + (2).to_bytes(8, "little") + (3).to_bytes(8, "little")
    assert d.hex() == d.bytes.hex()


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2104_08865_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("oracle_np", "x") or fn == "gen_encode.py", fn
