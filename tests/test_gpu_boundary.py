"""Boundary behaviour of the CUDA engine against the oracle: error semantics
the reference raises, unaligned device bases, instance-boundary varlen
batches, the bounded host path for long strings, the reference's batched
seam signature and engine names.

Every digest must equal the oracle's bit for bit."""

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


def _u64(t):
    return t.cpu().numpy().view(np.uint64)


def _S(master, w, n):
    return o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(o.variant(w), n))


# ------------------------------------------------------------ varlen sizing
# A string of 8m-7 .. 8m-1 bytes already holds one instance (ceil(n/8)/m):
# homogeneous batches just below an instance boundary hold more instances
# than total_bytes / 8m.  Every one of them must come back hashed.
@pytest.mark.parametrize("w,lo", [(16, 761), (24, 1337), (32, 1337), (40, 953)])
@pytest.mark.parametrize("count", [200, 1000])
def test_varlen_just_below_instance_boundary(hh, w, lo, count):
    p = hh.variant(w)
    for n in range(lo, lo + 7):
        lengths = np.full(count, n, dtype=np.uint64)
        off = np.zeros(count + 1, dtype=np.uint64)
        off[1:] = np.cumsum(lengths)
        total = int(off[-1])
        buf = hh.fill_bytes(total, n)
        seed = hh.seed_for_input(bytes(range(32)), p, n)
        got = _u64(hh.hash_varlen(buf, off, seed, p))
        host = np.frombuffer(o.fill_bytes(total, n), dtype=np.uint8).copy()
        want = coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity))
        assert np.array_equal(got, want), (w, n, count)
        # the same through device offsets, checked by the device
        import torch

        d_off = torch.from_numpy(off.view(np.int64)).cuda()
        got = _u64(hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=n))
        assert np.array_equal(got, want), (w, n, count, "device offsets")


# ------------------------------------------------------------ error semantics
def test_varlen_device_offsets_errors_raise(hh):
    import torch

    p = hh.variant(16)
    off = np.array([0, 100, 7000], dtype=np.uint64)  # string 1 has 6900 bytes
    buf = hh.fill_bytes(7000, 2)
    seed = hh.seed_for_input(b"\0" * 32, p, 7000)
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    # a string longer than the declared max: the reference raises SeedSizeError
    with pytest.raises(hh.SeedSizeError):
        hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=200)
    # decreasing offsets
    bad = torch.from_numpy(np.array([0, 500, 100], dtype=np.int64)).cuda()
    with pytest.raises(ValueError):
        hh.hash_varlen(buf, bad, seed, p, max_n_bytes=7000)
    # offsets past the end of the buffer
    past = torch.from_numpy(np.array([0, 100, 9000], dtype=np.int64)).cuda()
    with pytest.raises(ValueError):
        hh.hash_varlen(buf, past, seed, p, max_n_bytes=9000)
    # and a correct call on the same stream afterwards is clean
    got = _u64(hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=7000))
    host = np.frombuffer(o.fill_bytes(7000, 2), dtype=np.uint8).copy()
    assert np.array_equal(got, coracle.hash_varlen(16, host, off, seed.words_np(0, seed.capacity)))
    # host offsets are validated on the host
    with pytest.raises(ValueError):
        hh.hash_varlen(buf, np.array([0, 500, 100], dtype=np.uint64), seed, p)


def test_host_entry_seed_capacity_is_checked(hh):
    p = hh.variant(24)
    host = np.frombuffer(o.fill_bytes(4096), dtype=np.uint8).copy()
    for cap in (0, 5, hh.seed_words_needed(p, 4096) - 1):
        with pytest.raises(hh.SeedSizeError):
            hh.hash_fixed_host(host, 1, 4096, bytes(32), p, seed_capacity=cap)
    ok = hh.hash_fixed_host(host, 1, 4096, bytes(32), p, seed_capacity=hh.seed_words_needed(p, 4096))
    assert np.array_equal(ok, hh.hash_fixed_host(host, 1, 4096, bytes(32), p))
    assert np.array_equal(ok[0], coracle.hash_one(24, host, _S(bytes(32), 24, 4096)))


def test_single_string_any_stride_through_cabi(hh):
    # one string: the stride argument is meaningless and must not matter
    # (stride 0 once aliased the tail kernel's ring with its mbarriers)
    import torch

    from paper_2104_08865_b200 import _lib, batch

    L = _lib.lib()
    for w in VARIANTS:
        p = hh.variant(w)
        for n in (1, 100, 700, 1000, 2000, 5000):
            buf = hh.fill_bytes(n, 9)
            seed = hh.seed_for_input(bytes(range(32)), p, n)
            want = coracle.hash_one(w, np.frombuffer(o.fill_bytes(n, 9), dtype=np.uint8).copy(),
                                    seed.words_np(0, seed.capacity))
            for stride in (0, 16, n // 2 & ~15, n):
                out = torch.empty((1, w // 8), dtype=torch.int64, device="cuda")
                ws = torch.zeros(batch.workspace_fixed(p, 1, n) + 256, dtype=torch.uint8, device="cuda")
                _lib.check(L.hth_hash_fixed(w, buf.data_ptr(), 1, stride, n, seed.fold,
                                            seed.device_words().data_ptr(), seed.capacity, out.data_ptr(),
                                            ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream))
                assert np.array_equal(_u64(out)[0], want), (w, n, stride)


# ------------------------------------------------------------ unaligned device bases
@pytest.mark.parametrize("w", VARIANTS)
def test_unaligned_device_bases(hh, w):
    p = hh.variant(w)
    m8 = o.variant(w).m * 8
    for shift in (1, 3, 8, 13):
        # tail-only, small (1-7 instances), and multi-job strings, and a batch
        for n, B in ((500, 5), (3 * m8 + 5, 7), (70 * m8 + 11, 2), (2 * m8, 33)):
            stride = n + (shift & 7)
            total = shift + B * stride
            buf = hh.fill_bytes(total, 77)
            host = np.frombuffer(o.fill_bytes(total, 77), dtype=np.uint8).copy()
            seed = hh.seed_for_input(bytes(range(32)), p, n)
            S = seed.words_np(0, seed.capacity)
            got = _u64(hh.hash_fixed(buf[shift:], n, seed, p, n_strings=B, stride=stride))
            want = coracle.hash_fixed(w, host[shift:].copy(), B, stride, n, S)
            assert np.array_equal(got, want), (w, shift, n, B)
        # hash_bytes on a view of a device tensor
        n = 5 * m8 + 3
        buf = hh.fill_bytes(n + shift, 5)
        host = np.frombuffer(o.fill_bytes(n + shift, 5), dtype=np.uint8)[shift:].copy()
        seed = hh.seed_for_input(b"\7" * 32, p, n)
        d = hh.hash_bytes(buf[shift:shift + n], seed, p)
        assert np.array_equal(np.array(d.words, dtype=np.uint64),
                              coracle.hash_one(w, host, seed.words_np(0, seed.capacity)))
        # varlen over a view
        lengths = np.array([0, 7, 127, m8 - 1, m8 + 9, 9 * m8 + 1, 65 * m8 + 3], dtype=np.uint64)
        off = np.zeros(lengths.size + 1, dtype=np.uint64)
        off[1:] = np.cumsum(lengths)
        total = int(off[-1])
        buf = hh.fill_bytes(total + shift, 6)
        host = np.frombuffer(o.fill_bytes(total + shift, 6), dtype=np.uint8)[shift:].copy()
        seed = hh.seed_for_input(b"\3" * 32, p, int(lengths.max()))
        got = _u64(hh.hash_varlen(buf[shift:], off, seed, p))
        assert np.array_equal(got, coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity)))


# ------------------------------------------------------------ bounded host path for long strings
@pytest.mark.parametrize("w,n", [(16, (200 << 20) + 7), (40, (130 << 20) + 961), (24, (64 << 20) + 1)])
def test_host_long_string_sliced(hh, w, n):
    import torch

    p = hh.variant(w)
    data = o.fill_bytes(n, 21)
    seed = hh.seed_for_input(bytes(range(32)), p, n)
    want = coracle.hash_one(w, np.frombuffer(data, dtype=np.uint8), seed.words_np(0, seed.capacity))
    hh.release_host()
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    d = hh.hash_bytes(data, seed, p)
    assert np.array_equal(np.array(d.words, dtype=np.uint64), want)
    used = free0 - torch.cuda.mem_get_info()[0]
    assert used < 512 << 20, f"host path held {used >> 20} MiB of device memory for a {n >> 20} MiB string"
    hh.release_host()
    assert torch.cuda.mem_get_info()[0] >= free0 - (64 << 20)


def test_host_batch_of_long_strings(hh):
    w, n, B = 32, (66 << 20) + 5, 2
    stride = n + 11
    p = hh.variant(w)
    host = np.frombuffer(o.fill_bytes(B * stride, 3), dtype=np.uint8).copy()
    got = hh.hash_fixed_host(host, B, n, bytes(range(32)), p, stride=stride)
    want = coracle.hash_fixed(w, host, B, stride, n, _S(bytes(range(32)), w, n))
    assert np.array_equal(got, want)


# ------------------------------------------------------------ the reference's seam and engine names
def _batched_region(masters):
    from paper_2104_08865_b200 import hasher

    folds = (masters[:, 0] ^ masters[:, 1] ^ masters[:, 2] ^ masters[:, 3])[:, None]
    return lambda start, count: hasher._stream_words_np(folds, start, count), folds[:, 0]


def test_hash_words_np_seam_many_seeds(hh):
    # the call shape of the reference's many-seeds tests: one input broadcast
    # over 10^4 seed rows, _stream_words_np of (B, 1) folds as the region
    from paper_2104_08865_b200 import hasher

    p = hh.variant(24)
    n = 2048
    rng = np.random.default_rng(31)
    a = rng.integers(0, 1 << 64, size=n // 8, dtype=np.uint64)
    b = a.copy()
    b[100] ^= np.uint64(0xFF00000000)
    masters = rng.integers(0, 1 << 64, size=(10 ** 4, 4), dtype=np.uint64)
    region, folds = _batched_region(masters)
    out_a = hasher._hash_words_np(np.broadcast_to(a, (len(folds), a.size)), n, region, p)
    out_b = hasher._hash_words_np(np.broadcast_to(b, (len(folds), b.size)), n, region, p)
    assert out_a.shape == (10 ** 4, 3) and out_a.dtype == np.uint64
    assert int(np.all(out_a == out_b, axis=1).sum()) == 0
    for row in (0, 1234, 9999):
        master = masters[row].astype("<u8").tobytes()
        S = _S(master, 24, n)
        assert np.array_equal(out_a[row], coracle.hash_one(24, a.view(np.uint8).copy(), S))
        # the reference spot-checks with engine="scalar": an alias here
        d = hh.hash_bytes(a.astype("<u8").tobytes(), hh.seed_for_input(master, p, n), p, engine="scalar")
        assert d.words == tuple(int(x) for x in out_a[row])


def test_hash_words_np_seam_shared_seed(hh):
    # tests/test_acceptance.py's form: distinct rows, region = seed.words_np
    from paper_2104_08865_b200 import hasher

    rng = np.random.default_rng(0xC0FFEE)
    for w in VARIANTS:
        p = hh.variant(w)
        n = 2048 - 3
        words = rng.integers(0, 1 << 64, size=(1000, (n + 7) // 8), dtype=np.uint64)
        words[:, -1] &= np.uint64((1 << 40) - 1)  # zero-padded final word
        master = rng.integers(0, 1 << 64, size=4, dtype=np.uint64).astype("<u8").tobytes()
        seed = hh.seed_for_input(master, p, n)
        out = hasher._hash_words_np(words, n, seed.words_np, p)
        want = coracle.hash_fixed(w, words.view(np.uint8).reshape(-1).copy(), 1000, words.shape[1] * 8, n,
                                  seed.words_np(0, seed.capacity))
        assert np.array_equal(out, want)
        assert len(np.unique(out, axis=0)) == 1000
    with pytest.raises(IndexError):  # a region too small for the layout
        hasher._hash_words_np(words, n, hh.expand_seed(b"\0" * 32, 10).words_np, p)
    with pytest.raises(ValueError):  # not a seed stream the engine can serve
        hasher._hash_words_np(words, n, lambda s, c: np.arange(s, s + c, dtype=np.uint64), p)


def test_engine_names(hh):
    p = hh.variant(40)
    data = o.fill_bytes(10000, 4)
    seed = hh.seed_for_input(bytes(range(32)), p, len(data))
    ds = {e: hh.hash_bytes(data, seed, p, engine=e) for e in ("cuda", "lanes", "scalar")}
    assert len(set(ds.values())) == 1
    assert np.array_equal(np.array(ds["lanes"].words, dtype=np.uint64),
                          coracle.hash_one(40, np.frombuffer(data, dtype=np.uint8), seed.words_np(0, seed.capacity)))
    with pytest.raises(ValueError):
        hh.hash_bytes(data, seed, p, engine="avx512")
    with pytest.raises(ValueError):
        hh.hash_bytes(data, seed, p, engine="scalar", counter=object())
