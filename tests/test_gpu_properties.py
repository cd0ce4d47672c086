"""The reference's statistical hash-path properties (pkg/tests/test_hasher.py:
100-117, 224-311) on the CUDA engine, at GPU scale where that is cheap.
Integer-exact digests are covered elsewhere; these check the behaviour a
caller relies on: avalanche, separation of variants, of lengths and of
near-identical inputs across many seeds, and seed-stream diffusion."""

import random

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ZERO_MASTER = b"\x00" * 32
RANGE_MASTER = bytes(range(32))


@pytest.fixture(scope="module")
def hh():
    import torch

    import paper_2104_08865_b200 as h

    assert torch.cuda.is_available()
    return h


def _fill(hh, n, seed=0x243F6A8885A308D3):
    return hh.fill_bytes(n, seed).cpu().numpy()[:n].tobytes()


def test_digest_bit_avalanche(hh):
    # one flipped input bit flips about half of the digest bits (test_hasher.py:224-240):
    # 2,000 flips in one batch (the reference: 200 one-shot calls)
    import torch

    p = hh.variant(24)
    n = 1344
    base = np.frombuffer(_fill(hh, n), dtype=np.uint8)
    rnd = random.Random(17)
    B = 2001
    batch = np.tile(base, (B, 1))
    for i in range(1, B):
        bit = rnd.randrange(n * 8)
        batch[i, bit // 8] ^= np.uint8(1 << (bit % 8))
    seed = hh.seed_for_input(ZERO_MASTER, p, n)
    out = hh.hash_fixed(torch.from_numpy(batch.reshape(-1).copy()).cuda(), n, seed, p, n_strings=B, stride=n)
    d = out.cpu().numpy().view(np.uint64)
    diff = np.unpackbits((d[1:] ^ d[0]).view(np.uint8), axis=1).sum(axis=1) / (d.shape[1] * 64)
    assert 0.45 <= diff.mean() <= 0.55
    assert (d[1:] != d[0]).any(axis=1).all()


def test_variants_unrelated_digests(hh):
    # test_hasher.py:243-251
    data = _fill(hh, 4096)
    digests = {w: hh.digest(data, RANGE_MASTER, w) for w in (16, 24, 32, 40)}
    hexes = [d.hex() for d in digests.values()]
    assert len(set(hexes)) == len(hexes)
    for a in digests:
        for b in digests:
            if a < b:
                assert not digests[b].hex().startswith(digests[a].hex())


def test_prefix_inputs_different_lengths_distinct(hh):
    # same content, lengths 1500 vs 1501, under 10^6 random seeds (the reference:
    # 10^4): no seed gives equal digests (test_hasher.py:290-311, bound 2^-20)
    import torch

    p = hh.variant(24)
    rng = np.random.default_rng(33)
    long_bytes = rng.integers(0, 256, 1501, dtype=np.uint8)
    folds = rng.integers(0, 1 << 64, size=10 ** 6, dtype=np.uint64)
    buf = torch.from_numpy(np.concatenate([long_bytes, np.zeros(15, np.uint8)])).cuda()
    da = hh.hash_fixed_folds(buf, 1500, folds, p, stride=0)
    db = hh.hash_fixed_folds(buf, 1501, folds, p, stride=0)
    assert int(torch.all(da == db, dim=1).sum()) == 0


def test_expand_seed_bit_flip_diffusion(hh):
    # test_hasher.py:100-111, on the device expansion
    base = hh.expand_seed(ZERO_MASTER, 64).device_words().cpu().numpy().view(np.uint64)
    rnd = random.Random(8)
    for _ in range(16):
        bit = rnd.randrange(256)
        master = bytearray(32)
        master[bit // 8] ^= 1 << (bit % 8)
        flipped = hh.expand_seed(bytes(master), 64).device_words().cpu().numpy().view(np.uint64)
        ham = np.unpackbits((base ^ flipped).view(np.uint8)).sum() / 64
        assert ham >= 20
    # mix(gamma) is the first word of the all-zero master's stream (test_hasher.py:114-117)
    from paper_2104_08865_b200.hasher import splitmix_mix

    assert int(base[0]) == splitmix_mix(0x9E3779B97F4A7C15)
