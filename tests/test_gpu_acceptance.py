"""GPU forms of the reference's acceptance checks on the hash path
(pkg/tests/test_acceptance.py):

* criterion 7 (:168-186): no digest collisions over 10^5 random 2 KB inputs
  per variant -- here all 10^5 inputs of a variant are one batch through the
  CUDA engine, and a sample is also checked against the C oracle;
* the engine-agreement sweep (:189-220): 2,500 random (length, master) pairs
  per variant through the public ``hash_bytes`` against the C oracle (the
  reference compares its scalar and lanes engines; the oracle is pinned to
  both through the golden digests, tests/test_oracle_golden.py).
Integer work: bit-exact, no tolerance.
"""

import numpy as np
import pytest

from oracle import c as coracle
from oracle import oracle_np as o

pytestmark = pytest.mark.gpu

VARIANTS = (16, 24, 32, 40)


@pytest.fixture(scope="module")
def hh():
    import torch

    import paper_2104_08865_b200 as h

    assert torch.cuda.is_available()
    return h


@pytest.mark.parametrize("w", VARIANTS)
def test_criterion7_no_collisions_1e5_random_2kb(hh, w):
    import torch

    n, B = 2048, 100_000
    rng = np.random.default_rng(700 + w)
    host = rng.integers(0, 256, size=B * n, dtype=np.uint8)
    master = rng.integers(0, 256, 32, dtype=np.uint8).tobytes()
    p = hh.variant(w)
    seed = hh.seed_for_input(master, p, n)
    got = hh.hash_fixed(torch.from_numpy(host).cuda(), n, seed, p, n_strings=B, stride=n).cpu().numpy()
    assert np.unique(got, axis=0).shape[0] == B, "digest collision"
    sample = rng.choice(B, 512, replace=False)
    S = seed.words_np(0, seed.capacity)
    want = coracle.hash_fixed(w, np.ascontiguousarray(host.reshape(B, n)[sample]).reshape(-1), 512, n, n, S)
    assert np.array_equal(got.view(np.uint64)[sample], want)


@pytest.mark.parametrize("w", VARIANTS)
def test_random_length_master_pairs_2500(hh, w):
    rng = np.random.default_rng(2500 + w)
    p = hh.variant(w)
    lengths = np.concatenate([rng.integers(0, 4096, 2000), rng.integers(4096, 200_000, 500)])
    for i, n in enumerate(lengths.tolist()):
        master = rng.integers(0, 256, 32, dtype=np.uint8).tobytes()
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        got = hh.hash_bytes(data, hh.seed_for_input(master, p, n), p)
        S = o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(o.variant(w), n))
        want = coracle.hash_one(w, np.frombuffer(data, dtype=np.uint8), S)
        assert got.words == tuple(int(x) for x in want), (w, i, n)
