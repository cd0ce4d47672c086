"""GPU forms of the reference's acceptance checks on the hash path
(pkg/tests/test_acceptance.py):

* criterion 7 (:168-186): no digest collisions over 10^5 random 2 KB inputs
  per variant -- here all 10^5 inputs of a variant are one batch through the
  CUDA engine, and a sample is also checked against the C oracle;
* the engine-agreement sweep (criterion 8, :189-220): 2,500 (length, master)
  pairs per variant with its boundary-heavy length mix (+250 longer strings)
  through the public ``hash_bytes`` against the C oracle (the
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
    # criterion 8's mix (test_acceptance.py:189-200): the instance/block
    # boundary lengths 40 times each, the rest uniform in [0, 2 instances),
    # plus 250 longer strings (multi-round and multi-job paths)
    rng = np.random.default_rng(2500 + w)
    p = hh.variant(w)
    iw = o.variant(w).m * 8
    boundary = [0, 1, 63, 64, 65, iw - 8, iw - 1, iw, iw + 1, iw + 8, 2 * iw - 1, 2 * iw, 2 * iw + 1]
    lengths = np.concatenate([np.array(boundary * 40), rng.integers(0, 2 * iw, 2500 - 40 * len(boundary)),
                              rng.integers(2 * iw, 200_000, 250)])
    for i, n in enumerate(lengths.tolist()):
        master = rng.integers(0, 256, 32, dtype=np.uint8).tobytes()
        data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
        got = hh.hash_bytes(data, hh.seed_for_input(master, p, n), p)
        S = o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(o.variant(w), n))
        want = coracle.hash_one(w, np.frombuffer(data, dtype=np.uint8), S)
        assert got.words == tuple(int(x) for x in want), (w, i, n)
