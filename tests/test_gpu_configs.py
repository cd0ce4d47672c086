"""Every BASELINE.json config at its stated size, checked digest by digest.

Inputs are the bench's (workloads.py): the reference's splitmix stream with
data seed 0 for the bytes and the fold-1 master for the seed array.  The CUDA
digests come through the C-ABI (hth_hash_fixed / hth_hash_varlen); the
expected ones from the threaded C restatement (oracle/halftime_oracle.c,
pinned to the reference's golden digests in test_oracle_golden.py) over bytes
regenerated on the host, not copied back from the GPU.  Integer work: no
tolerance.  Config 5 (one 16 GiB string) is test_gpu_parity.py's
test_config5_full_16gib.
"""

import numpy as np
import pytest

from oracle import c as coracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hh():
    import torch

    import paper_2104_08865_b200 as h

    assert torch.cuda.is_available()
    return h


def _u64(t):
    return t.cpu().numpy().view(np.uint64)


def _host_stream(n_bytes):
    """Bytes [0, n_bytes) of the data stream (seed 0), generated on the host."""
    from workloads import DATA_SEED

    words = coracle.splitmix(DATA_SEED, 0, (n_bytes + 7) // 8)
    return words.view(np.uint8)[:n_bytes]


def _fixed_config(hh, name):
    import torch

    from workloads import CONFIGS, DATA_SEED, MASTER

    cfg = CONFIGS[name]
    w, B, n = cfg["variant"], cfg["n_strings"], cfg["n_bytes"]
    p = hh.variant(w)
    buf = hh.fill_bytes(B * n, DATA_SEED)
    seed = hh.seed_for_input(MASTER, p, n)
    got = _u64(hh.hash_fixed(buf, n, seed, p, n_strings=B, stride=n))
    del buf
    torch.cuda.empty_cache()
    host = _host_stream(B * n)
    want = coracle.hash_fixed(w, host, B, n, n, seed.words_np(0, seed.capacity))
    return got, want


def _assert_same(got, want, what):
    assert got.shape == want.shape, what
    bad = np.nonzero(~np.all(got == want, axis=1))[0]
    assert bad.size == 0, f"{what}: {bad.size} of {len(want)} digests differ, first {bad[:8]}"


def test_config1_every_digest(hh):
    # 1024 strings x 4096 B, 24-byte variant: bit-exact on every digest
    got, want = _fixed_config(hh, "cfg1")
    _assert_same(got, want, "cfg1")


@pytest.mark.parametrize("w", (16, 24, 32, 40))
def test_config2_every_digest(hh, w):
    # 16384 strings, log-uniform 1 B - 64 KiB plus every length 0..127 once,
    # packed back to back (unaligned starts) with u64 offsets; all four variants
    import torch

    from workloads import DATA_SEED, MASTER, cfg2_lengths, offsets_of

    lengths = cfg2_lengths()
    assert len(lengths) == 16384 and set(range(128)) <= set(lengths.tolist())
    off = offsets_of(lengths)
    total = int(off[-1])
    buf = hh.fill_bytes(total, DATA_SEED)
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    p = hh.variant(w)
    seed = hh.seed_for_input(MASTER, p, int(lengths.max()))
    got = _u64(hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=int(lengths.max())))
    want = coracle.hash_varlen(w, _host_stream(total), off, seed.words_np(0, seed.capacity))
    _assert_same(got, want, f"cfg2 v{w}")


@pytest.mark.slow
def test_config3_every_digest(hh):
    # 4,194,304 strings x 1024 B (4 GiB), 32-byte variant (the config asks for
    # a 4096-string sample; every digest is checked here)
    got, want = _fixed_config(hh, "cfg3")
    _assert_same(got, want, "cfg3")
    rng = np.random.default_rng(3)
    sample = rng.choice(len(want), 4096, replace=False)
    assert np.array_equal(got[sample], want[sample])


@pytest.mark.slow
def test_config4_every_digest(hh):
    # 8192 strings x 1 MiB (8 GiB), 40-byte variant: the bench's headline batch
    got, want = _fixed_config(hh, "cfg4")
    _assert_same(got, want, "cfg4")
