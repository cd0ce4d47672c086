"""Randomised parity: hypothesis draws variants, lengths, masters, batch
shapes and string alignments; every digest from the CUDA engine (through the
public Python API and the C-ABI underneath) must equal the C oracle's, which
is pinned to the reference's golden vectors (tests/test_oracle_golden.py).
Integer work: bit-exact, no tolerance."""

import os

import numpy as np
import pytest

from oracle import c as coracle
from oracle import oracle_np as o

hypothesis = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as stg  # noqa: E402

pytestmark = pytest.mark.gpu

VARIANTS = (16, 24, 32, 40)
# HTH_HYPOTHESIS_EXAMPLES=N: a longer, non-derandomised exploration run
_N = int(os.environ.get("HTH_HYPOTHESIS_EXAMPLES", "0"))
SETTINGS = dict(max_examples=_N or 150, deadline=None, derandomize=not _N,
                suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])


@pytest.fixture(scope="module")
def hh():
    import torch

    import paper_2104_08865_b200 as h

    assert torch.cuda.is_available()
    return h


def _master(seed):
    return np.random.default_rng(seed).integers(0, 256, 32, dtype=np.uint8).tobytes()


def _seeds(master, w, n):
    v = o.variant(w)
    return o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(v, n))


# lengths biased towards the boundaries that change the code path: tail-only,
# 1-7 instances (packed kernel), one partial level-1 group, job boundaries
def _length(draw, w):
    iw = o.variant(w).m * 8
    kind = draw(stg.integers(0, 4))
    if kind == 0:
        return draw(stg.integers(0, iw - 1))
    if kind == 1:
        return draw(stg.integers(iw, 8 * iw - 1))
    if kind == 2:
        return draw(stg.integers(8 * iw, 80 * iw))
    if kind == 3:
        k = draw(stg.sampled_from([1, 7, 8, 9, 63, 64, 65, 511, 512, 513]))
        return max(0, k * iw + draw(stg.integers(-9, 9)))
    return draw(stg.integers(0, 40000))


@stg.composite
def one_string(draw):
    w = draw(stg.sampled_from(VARIANTS))
    return w, _length(draw, w), draw(stg.integers(0, 2**31))


@settings(**SETTINGS)
@given(one_string())
def test_hash_bytes_random(hh, case):
    w, n, ms = case
    master = _master(ms)
    data = o.fill_bytes(n, ms & 0xFFFF)
    p = hh.variant(w)
    got = hh.hash_bytes(data, hh.seed_for_input(master, p, n), p)
    host = np.frombuffer(data, dtype=np.uint8).copy() if n else np.zeros(16, np.uint8)
    want = coracle.hash_fixed(w, host, 1, max(n, 1), n, _seeds(master, w, n))[0]
    assert tuple(int(x) for x in want) == tuple(got.words), (w, n)


@stg.composite
def fixed_batch(draw):
    w = draw(stg.sampled_from(VARIANTS))
    n = _length(draw, w) % 30000
    B = draw(stg.integers(1, 70))
    pad = draw(stg.sampled_from([0, 0, 8, 16, 24, 40, 264]))
    stride = ((n + 7) // 8) * 8 + pad if draw(stg.booleans()) else n + draw(stg.integers(0, 9))
    return w, n, B, max(stride, n, 1), draw(stg.integers(0, 2**31))


@settings(**SETTINGS)
@given(fixed_batch())
def test_hash_fixed_random(hh, case):
    w, n, B, stride, ms = case
    master = _master(ms)
    total = (B - 1) * stride + n
    p = hh.variant(w)
    buf = hh.fill_bytes(total, ms & 0xFFFF)
    got = hh.hash_fixed(buf, n, hh.seed_for_input(master, p, n), p, n_strings=B, stride=stride)
    got = got.cpu().numpy().view(np.uint64)
    host = np.frombuffer(o.fill_bytes(total, ms & 0xFFFF), dtype=np.uint8).copy() if total else np.zeros(16, np.uint8)
    want = coracle.hash_fixed(w, host, B, stride, n, _seeds(master, w, n))
    assert np.array_equal(got, want), (w, n, B, stride)


@stg.composite
def varlen_batch(draw):
    w = draw(stg.sampled_from(VARIANTS))
    count = draw(stg.integers(1, 60))
    lengths = [_length(draw, w) % 50000 for _ in range(count)]
    return w, lengths, draw(stg.integers(0, 2**31))


@settings(**SETTINGS)
@given(varlen_batch())
def test_hash_varlen_random(hh, case):
    w, lengths, ms = case
    master = _master(ms)
    off = np.zeros(len(lengths) + 1, dtype=np.uint64)
    off[1:] = np.cumsum(np.array(lengths, dtype=np.uint64))
    total = int(off[-1])
    p = hh.variant(w)
    mx = max(lengths)
    buf = hh.fill_bytes(max(total, 1), ms & 0xFFFF)
    got = hh.hash_varlen(buf, off, hh.seed_for_input(master, p, mx), p).cpu().numpy().view(np.uint64)
    host = np.frombuffer(o.fill_bytes(max(total, 1), ms & 0xFFFF), dtype=np.uint8).copy()
    want = coracle.hash_varlen(w, host, off, _seeds(master, w, mx))
    bad = np.nonzero(~np.all(got == want, axis=1))[0]
    assert bad.size == 0, (w, [lengths[i] for i in bad[:5]])


@stg.composite
def folds_batch(draw):
    w = draw(stg.sampled_from(VARIANTS))
    n = _length(draw, w) % 30000
    B = draw(stg.integers(1, 40))
    shared = draw(stg.booleans())  # one input under every fold (stride 0) or distinct inputs
    return w, n, B, shared, draw(stg.integers(0, 2**31))


@settings(**SETTINGS)
@given(folds_batch())
def test_many_seeds_random(hh, case):
    # hth_hash_fixed_folds: row s hashed under the seed stream of folds[s]
    # (the reference seam with a (B, 1) fold region, tests/test_hasher.py:254-310)
    w, n, B, shared, ms = case
    rng = np.random.default_rng(ms)
    folds = rng.integers(0, 1 << 64, size=B, dtype=np.uint64)
    stride = 0 if shared else (n + 15) // 16 * 16
    total = max(n if shared else B * stride, 16)
    p = hh.variant(w)
    buf = hh.fill_bytes(total, ms & 0xFFFF)
    got = hh.hash_fixed_folds(buf, n, folds, p, stride=max(stride, 0)).cpu().numpy().view(np.uint64)
    host = np.frombuffer(o.fill_bytes(total, ms & 0xFFFF), dtype=np.uint8).copy()
    v = o.variant(w)
    for b in range(B):
        s0 = 0 if shared else b * stride
        S = o.splitmix_words(int(folds[b]), 0, o.seed_words_needed(v, n))
        assert np.array_equal(got[b], coracle.hash_one(w, host[s0:s0 + n], S)), (w, n, b)


@stg.composite
def split_string(draw):
    w = draw(stg.sampled_from(VARIANTS))
    iw = o.variant(w).m * 8
    inst = draw(stg.sampled_from([0, 1, 63, 64, 65, 511, 512, 513, 600, 4096, 4097, 5000, 33000]))
    n = inst * iw + draw(stg.integers(0, iw - 1))
    return w, n, draw(stg.integers(1, 9)), draw(stg.integers(0, 2**31))


@settings(**dict(SETTINGS, max_examples=_N // 10 if _N else 150))
@given(split_string())
def test_split_string_and_stream_random(hh, case):
    # one string cut into ns slices (emulated ranks, one after another) and
    # merged, and the same bytes fed to StreamHasher in random pieces: both
    # equal the oracle's one-shot digest
    import torch

    from paper_2104_08865_b200 import multi_gpu

    w, n, ns, ms = case
    p = hh.variant(w)
    master = _master(ms)
    seed = hh.seed_for_input(master, p, n)
    buf = hh.fill_bytes(max(n, 16), ms & 0xFFFF)
    host = np.frombuffer(o.fill_bytes(max(n, 16), ms & 0xFFFF), dtype=np.uint8)[:n].copy()
    want = coracle.hash_one(w, host, _seeds(master, w, n))
    if n >= 512 * o.variant(w).m * 8:  # the split needs whole level-c subtrees (c >= the job level)
        plan = multi_gpu.slice_plan(p, n, ns)
        frs, parts = [], []
        for i in range(ns):
            b0, _ = plan.byte_range(i)
            fr, part = multi_gpu.hash_slice(buf[b0:], plan, i, seed)
            frs.append(fr.clone())
            parts.append(part.clone())
        got = multi_gpu.hash_merge(torch.cat(frs), torch.stack(parts), plan, seed)
        assert np.array_equal(got.cpu().numpy().view(np.uint64), want), (w, n, ns)
    h = hh.StreamHasher(p, seed, n, slice_bytes=1 << 20)
    rng = np.random.default_rng(ms)
    pos = 0
    while pos < n:
        step = int(rng.integers(1, max(2, n // 3 + 2)))
        h.update(host[pos:pos + step].tobytes())
        pos += step
    assert tuple(int(x) for x in want) == tuple(h.digest().words), (w, n, "stream")
