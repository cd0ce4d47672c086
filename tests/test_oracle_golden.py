"""Pin the CPU oracle (both restatements) to the reference's golden vectors.

CPU only.  The oracle is the checker for every GPU parity test, so it must
reproduce the reference bit for bit first."""

import os

import numpy as np
import pytest

from oracle import c as coracle
from oracle import oracle_np as o

from _golden import GOLDEN_EMPTY_24, ZERO_MASTER, classic_cases, gen_bytes, records


@pytest.mark.parametrize("case", classic_cases(), ids=lambda c: f"{c[0]}-{len(c[2])}")
def test_numpy_oracle_reference_goldens(case):
    w, master, data, hexd = case
    assert o.digest(data, master, w).hex() == hexd


@pytest.mark.parametrize("case", classic_cases(), ids=lambda c: f"{c[0]}-{len(c[2])}")
def test_c_oracle_reference_goldens(case):
    w, master, data, hexd = case
    v = o.variant(w)
    S = o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(v, len(data)))
    got = coracle.hash_one(w, data, S)
    assert b"".join(int(x).to_bytes(8, "little") for x in got).hex() == hexd


def test_cli_empty_golden():
    assert o.digest(b"", ZERO_MASTER, 24).hex() == GOLDEN_EMPTY_24


def _digest_hex(words):
    return b"".join(int(x).to_bytes(8, "little") for x in words).hex()


def test_fixture_records_numpy_and_c():
    recs = [r for r in records() if r["kind"] in ("lanes", "scalar", "cli_grid", "capacity")]
    assert len(recs) > 800
    for r in recs:
        w, n = r["variant"], r["length"]
        v = o.variant(w)
        data = gen_bytes(r["generator"], n)
        fold = o.master_fold(bytes.fromhex(r["master"]))
        cap = r.get("capacity", o.seed_words_needed(v, n))
        S = o.splitmix_words(fold, 0, cap)
        if n <= 300_000:
            assert _digest_hex(o.hash_bytes(v, data, S)) == r["digest"], r
        assert _digest_hex(coracle.hash_one(w, data, S)) == r["digest"], r


def test_fixture_many_seeds_fold_records():
    for r in records("fold"):
        v = o.variant(r["variant"])
        data = gen_bytes(r["generator"], r["length"])
        S = o.splitmix_words(r["fold"], 0, o.seed_words_needed(v, r["length"]))
        assert _digest_hex(o.hash_bytes(v, data, S)) == r["digest"]


def test_c_oracle_parallel_paths_agree():
    # hash_huge (parallel subtrees) and hash_fixed/varlen agree with hash_one
    rng = np.random.default_rng(5)
    for w in (16, 40):
        v = o.variant(w)
        n = 9 * 512 * v.m * 8 + 12345  # > 8^3 instances: exercises level >= 3 merges
        data = np.frombuffer(rng.bytes(n), dtype=np.uint8).copy()
        S = o.splitmix_words(7, 0, o.seed_words_needed(v, n))
        one = coracle.hash_one(w, data, S)
        assert np.array_equal(coracle.hash_huge(w, data, S, threads=4), one)
        buf = np.concatenate([data[:1000], data])
        offs = np.array([0, 1000, 1000, 1000 + n], dtype=np.uint64)
        vl = coracle.hash_varlen(w, buf, offs, S)
        assert np.array_equal(vl[2], one)
        assert np.array_equal(vl[0], coracle.hash_one(w, data[:1000], S))
        assert np.array_equal(vl[1], coracle.hash_one(w, b"", S))


def test_seed_stream_and_layout():
    # splitmix stream == reference formula (hasher.py:55-58), C == numpy
    for fold in (0, 1, 0xDEADBEEF, (1 << 64) - 1):
        a = o.splitmix_words(fold, 3, 50)
        assert np.array_equal(a, coracle.splitmix(fold, 3, 50))
    # appendix-B layout totals
    assert o.layout(o.variant(24), 4096).total == 410
    assert o.layout(o.variant(32), 1024).total == 485
    assert o.layout(o.variant(40), 1 << 20).total == 1571
    assert o.layout(o.variant(16), 16 << 30).total == 1389
    for w in (16, 24, 32, 40):
        for n in (0, 1, 1000, 10 ** 6, 16 << 30):
            assert coracle.seed_words_needed(w, n) == o.seed_words_needed(o.variant(w), n)


def test_oracle_matches_reference_deep_trees():
    # L = 6 and 7 records the reference computed (tests/golden/deep_vectors.jsonl)
    import json

    from oracle import c as coracle

    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "deep_vectors.jsonl")
    with open(path) as fh:
        recs = [r for r in map(json.loads, fh) if r["kind"] == "deep" and r["levels"] <= 7]
    assert len(recs) == 8
    for r in recs:
        n = r["length"]
        kind, seed, off = r["generator"].split(":")
        host = coracle.splitmix(int(seed, 16), int(off), (n + 7) // 8).view(np.uint8)[:n].copy()
        S = o.splitmix_words(o.master_fold(bytes.fromhex(r["master"])), 0, o.seed_words_needed(o.variant(r["variant"]), n))
        got = coracle.hash_huge(r["variant"], host, S)
        assert got.tobytes().hex() == r["digest"], (r["variant"], r["levels"])
