"""CUDA engine parity against the oracle and the reference's golden vectors.

Every digest produced by libhalftime_b200.so must equal the reference's bit
for bit (integer work: no tolerance)."""

import numpy as np
import pytest

from oracle import c as coracle
from oracle import oracle_np as o

from _golden import classic_cases, gen_bytes, records

pytestmark = pytest.mark.gpu

VARIANTS = (16, 24, 32, 40)


@pytest.fixture(scope="module")
def hh():
    import torch

    import paper_2104_08865_b200 as h

    assert torch.cuda.is_available()
    return h


def _hex(words):
    return b"".join(int(x).to_bytes(8, "little") for x in words).hex()


def _u64(t):
    return t.cpu().numpy().view(np.uint64)


# ------------------------------------------------------------------ goldens
@pytest.mark.parametrize("case", classic_cases(), ids=lambda c: f"{c[0]}-{len(c[2])}")
def test_reference_golden_digests(hh, case):
    w, master, data, hexd = case
    assert hh.digest(data, master, w).hex() == hexd


def test_fixture_records_public_api(hh):
    recs = [r for r in records() if r["kind"] in ("lanes", "scalar", "cli_grid", "capacity")]
    bad = []
    for r in recs:
        w, n = r["variant"], r["length"]
        p = hh.variant(w)
        data = gen_bytes(r["generator"], n)
        master = bytes.fromhex(r["master"])
        cap = r.get("capacity", hh.seed_words_needed(p, n))
        d = hh.hash_bytes(data, hh.expand_seed(master, cap), p)
        if d.hex() != r["digest"]:
            bad.append((w, n, r["kind"]))
    assert not bad, bad[:20]


def test_fixture_records_device_tensor(hh):
    import torch

    for r in records("lanes")[::7]:
        w, n = r["variant"], r["length"]
        p = hh.variant(w)
        data = torch.frombuffer(bytearray(gen_bytes(r["generator"], n)) or bytearray(1), dtype=torch.uint8)[:n]
        seed = hh.seed_for_input(bytes.fromhex(r["master"]), p, n)
        assert hh.hash_bytes(data.cuda(), seed, p).hex() == r["digest"], (w, n)


# ------------------------------------------------------------------ batches
def _check_fixed(hh, w, n_strings, n_bytes, stride=None, seed_fold=3, data_seed=11):
    import torch

    p = hh.variant(w)
    stride = n_bytes if stride is None else stride
    total = (n_strings - 1) * stride + n_bytes if n_strings else 0
    buf = hh.fill_bytes(total, data_seed)
    master = seed_fold.to_bytes(8, "little") + bytes(24)
    seed = hh.seed_for_input(master, p, n_bytes)
    got = _u64(hh.hash_fixed(buf, n_bytes, seed, p, n_strings=n_strings, stride=stride))
    host = np.frombuffer(o.fill_bytes(total, data_seed), dtype=np.uint8).copy() if total else np.zeros(16, np.uint8)
    S = o.splitmix_words(seed_fold, 0, o.seed_words_needed(o.variant(w), n_bytes))
    want = coracle.hash_fixed(w, host, n_strings, stride, n_bytes, S)
    bad = np.nonzero(~np.all(got == want, axis=1))[0]
    assert bad.size == 0, f"v{w} n={n_bytes} stride={stride}: {bad.size} mismatches, first {bad[:5]}"


@pytest.mark.parametrize("w", VARIANTS)
def test_every_short_length(hh, w):
    # n = 0..127 (all tail-only) plus instance/block boundaries, batch of 33
    v = o.variant(w)
    iw = v.m * 8
    lengths = list(range(0, 128)) + [iw - 9, iw - 8, iw - 1, iw, iw + 1, iw + 7, iw + 8, 2 * iw - 1, 2 * iw,
                                     2 * iw + 1, 4 * iw - 1, 4 * iw, 4 * iw + 3, 5 * iw + 100, 7 * iw + 5,
                                     8 * iw - 1, 8 * iw, 8 * iw + 1, 9 * iw - 3]
    for n in lengths:
        _check_fixed(hh, w, 33, n)


@pytest.mark.parametrize("w", VARIANTS)
def test_tail_only_kernel(hh, w):
    # strings shorter than one instance with 16-byte-aligned strides take the
    # dedicated tail kernel (hth_hash_fixed dispatch); odd batch sizes too
    v = o.variant(w)
    iw = v.m * 8
    for n in list(range(0, 130)) + [255, 256, 257, 1000, 1023, 1024, iw - 17, iw - 9, iw - 8, iw - 1]:
        stride = (n + 15) // 16 * 16
        _check_fixed(hh, w, 37, n, stride=max(stride, 16))


@pytest.mark.parametrize("w", VARIANTS)
def test_every_tail_only_length(hh, w):
    # every length below one instance (0 .. 8m-1 bytes): the tail-only batch
    # kernel's chunk-count instantiations (1/2/4/6 chunks per lane, masked or
    # not) must all match the oracle -- e.g. 768 and 1280 B, whose chunk counts
    # (48, 80) fall short of a whole instantiation
    iw = o.variant(w).m * 8
    master = bytes(range(32))
    p = hh.variant(w)
    B = 3
    for n in range(0, iw):
        host = np.frombuffer(o.fill_bytes(B * max(n, 1), 20 + n), dtype=np.uint8).copy()
        S = o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(o.variant(w), n))
        want = coracle.hash_fixed(w, host, B, max(n, 1), n, S)
        got = hh.hash_fixed_host(host, B, n, master, p, stride=max(n, 1))
        assert np.array_equal(got, want), (w, n)


@pytest.mark.parametrize("w", VARIANTS)
def test_every_length_up_to_ten_instances(hh, w):
    # every length from one instance to ten (the packed small-string kernel
    # for 1-7 instances with 8-byte-aligned strides, the unaligned job kernel
    # otherwise, then a partial or complete level-1 group), two strings per
    # batch: each must match the oracle
    iw = o.variant(w).m * 8
    master = bytes(range(32))
    p = hh.variant(w)
    for n in range(iw, 10 * iw):
        S = o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(o.variant(w), n))
        for stride in ((n + 7) // 8 * 8, n + 3):
            host = np.frombuffer(o.fill_bytes(2 * stride, n), dtype=np.uint8).copy()
            want = coracle.hash_fixed(w, host, 2, stride, n, S)
            got = hh.hash_fixed_host(host, 2, n, master, p, stride=stride)
            assert np.array_equal(got, want), (w, n, stride)


@pytest.mark.parametrize("w", VARIANTS)
def test_small_string_kernel(hh, w):
    # 1..7 instances with 8-byte-aligned strides take the packed small-string
    # kernel (G = 4/2/1 strings per stage by stride); partial final words in
    # the tail, batch sizes not a multiple of G, and the strides just inside
    # and outside its packing limit (stride <= n + 256)
    v = o.variant(w)
    iw = v.m * 8
    for inst in range(1, 8):
        for tail in (0, 8, 13, iw - 1):
            n = inst * iw + tail
            a8 = (n + 7) // 8 * 8
            for stride, count in ((a8, 33), (a8 + 8, 5), ((n + 15) // 16 * 16, 3), (a8 + 256, 7), (a8 + 264, 2)):
                if stride >= n:
                    _check_fixed(hh, w, count, n, stride=stride)
    # batches large enough for 4 and 2 strings per stage (odd counts)
    _check_fixed(hh, w, 12001, iw + 13)
    _check_fixed(hh, w, 6001, 3 * iw + 8)
    _check_fixed(hh, w, 12003, 2 * iw, stride=2 * iw + 24)
    # the partial final word inside the last instance (job-kernel path)
    _check_fixed(hh, w, 9, 3 * iw - 3, stride=3 * iw)
    _check_fixed(hh, w, 1001, 2 * iw + 40)
    _check_fixed(hh, w, 1, 5 * iw + 77)


@pytest.mark.parametrize("w", VARIANTS)
def test_multi_job_and_tree_levels(hh, w):
    # job boundaries (64 instances), level-2 / level-3 merges, powers of 8 +- 1
    v = o.variant(w)
    iw = v.m * 8
    for inst in (63, 64, 65, 127, 128, 129, 511, 512, 513, 575, 1092, 4095, 4096, 4097):
        for extra in (0, 13):
            _check_fixed(hh, w, 5, inst * iw + extra)


@pytest.mark.parametrize("w", VARIANTS)
def test_unaligned_stride(hh, w):
    for stride_extra in (1, 3, 8, 9):
        n = 3000 + 17 * stride_extra
        _check_fixed(hh, w, 40, n, stride=n + stride_extra)


@pytest.mark.parametrize("w", VARIANTS)
def test_varlen_packed(hh, w):
    import torch

    from workloads import cfg2_lengths, offsets_of

    lengths = cfg2_lengths(2048, seed=w)
    lengths[::97] = np.arange(0, len(lengths[::97])) * 41 % 3000 + 70000  # a few multi-job strings
    off = offsets_of(lengths)
    total = int(off[-1])
    buf = hh.fill_bytes(total, 5)
    p = hh.variant(w)
    seed = hh.seed_for_input(bytes(range(32)), p, int(lengths.max()))
    got = _u64(hh.hash_varlen(buf, off, seed, p))
    host = np.frombuffer(o.fill_bytes(total, 5), dtype=np.uint8).copy()
    S = seed.words_np(0, seed.capacity)
    want = coracle.hash_varlen(w, host, off, S)
    bad = np.nonzero(~np.all(got == want, axis=1))[0]
    assert bad.size == 0, f"{bad.size} mismatches; lengths {lengths[bad[:8]]} offsets {off[bad[:8]] % 16}"


@pytest.mark.parametrize("w", VARIANTS)
def test_varlen_every_length_up_to_ten_instances(hh, w):
    # one packed batch holding every length 0 .. 10 instances once, shuffled
    # (unaligned starts): tail-only strings (planning kernel), 1-7 instances
    # and partial/complete level-1 groups (varlen job kernel)
    from workloads import offsets_of

    iw = o.variant(w).m * 8
    lengths = np.random.default_rng(w).permutation(np.arange(10 * iw + 1, dtype=np.int64))
    off = offsets_of(lengths)
    total = int(off[-1])
    buf = hh.fill_bytes(total, 33)
    p = hh.variant(w)
    seed = hh.seed_for_input(bytes(range(32)), p, int(lengths.max()))
    got = _u64(hh.hash_varlen(buf, off, seed, p))
    host = np.frombuffer(o.fill_bytes(total, 33), dtype=np.uint8).copy()
    want = coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity))
    bad = np.nonzero(~np.all(got == want, axis=1))[0]
    assert bad.size == 0, f"{bad.size} mismatches; lengths {lengths[bad[:8]]}"


@pytest.mark.parametrize("w", VARIANTS)
@pytest.mark.parametrize("odd", (0, 1))
def test_varlen_pairs_and_small_last_jobs(hh, w, odd):
    # one-level strings of 1..4 instances are hashed two per round (pair
    # jobs, any tail length, an odd count per class leaves one unpaired);
    # multi-job strings whose last job holds 1..4 instances (64 k + 1..4, and
    # 512 + 1..4 / 4096 + 1..4 with 512-instance jobs) must not be paired
    from workloads import offsets_of

    iw = o.variant(w).m * 8
    rng = np.random.default_rng(100 * w + odd)
    small = [c * iw + int(rng.integers(0, iw)) for c in range(1, 5) for _ in range(7 + 2 * c + odd)]
    multi = [(64 * k + c) * iw + int(rng.integers(0, iw)) for k in (1, 2) for c in range(1, 5)]
    if odd:
        multi += [(4096 + c) * iw + 5 for c in (1, 4)]  # 512-instance jobs
    lengths = rng.permutation(np.array(small + multi + [0, 1, iw - 1], dtype=np.int64))
    off = offsets_of(lengths)
    total = int(off[-1])
    buf = hh.fill_bytes(total, 44 + odd)
    p = hh.variant(w)
    seed = hh.seed_for_input(bytes(range(32)), p, int(lengths.max()))
    got = _u64(hh.hash_varlen(buf, off, seed, p))
    host = np.frombuffer(o.fill_bytes(total, 44 + odd), dtype=np.uint8).copy()
    want = coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity))
    bad = np.nonzero(~np.all(got == want, axis=1))[0]
    assert bad.size == 0, f"{bad.size} mismatches; lengths {lengths[bad[:8]]}"


def test_varlen_workspace_reused_across_layouts(hh):
    # one workspace, alternating batch shapes: the engine clears its counter
    # region only when the layout changes and otherwise relies on the
    # kernels leaving it zeroed -- every call must still match the oracle
    import torch

    from paper_2104_08865_b200 import batch
    from workloads import offsets_of

    w = 32
    p = hh.variant(w)
    rng = np.random.default_rng(77)
    shapes = [rng.integers(0, 9000, 300), rng.integers(0, 3000, 1100), rng.integers(0, 80000, 40)]
    bufs = []
    for i, ln in enumerate(shapes):
        ln = ln.astype(np.int64)
        off = offsets_of(ln)
        total = int(off[-1])
        bufs.append((hh.fill_bytes(total, 60 + i), off, total, int(ln.max())))
    wsz = max(batch.workspace_varlen(p, len(o_) - 1, t) for _, o_, t, _ in bufs)
    ws = torch.zeros(wsz, dtype=torch.uint8, device="cuda")
    for k in (0, 1, 0, 2, 2, 1, 0):
        buf, off, total, mx = bufs[k]
        seed = hh.seed_for_input(bytes(range(32)), p, mx)
        got = _u64(hh.hash_varlen(buf, off, seed, p, workspace=ws))
        host = np.frombuffer(o.fill_bytes(total, 60 + k), dtype=np.uint8).copy()
        want = coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity))
        assert np.array_equal(got, want), k


@pytest.mark.parametrize("n_strings", (16384, 16385, 70001))
def test_varlen_plan_paths(hh, n_strings):
    # batch sizes around and far beyond one planning pass, with a few
    # multi-job strings among them: every string must come back hashed
    from workloads import offsets_of

    rng = np.random.default_rng(n_strings)
    lengths = rng.integers(0, 2500, n_strings).astype(np.uint64)
    lengths[::1009] = 70000 + rng.integers(0, 9000, len(lengths[::1009]))
    off = offsets_of(lengths)
    total = int(off[-1])
    buf = hh.fill_bytes(total, 9)
    host = np.frombuffer(o.fill_bytes(total, 9), dtype=np.uint8).copy()
    for w in (24, 40):
        p = hh.variant(w)
        seed = hh.seed_for_input(bytes(range(32)), p, int(lengths.max()))
        got = _u64(hh.hash_varlen(buf, off, seed, p))
        want = coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity))
        bad = np.nonzero(~np.all(got == want, axis=1))[0]
        assert bad.size == 0, f"v{w}: {bad.size} mismatches, first {bad[:8]}"


@pytest.mark.parametrize("w", (16, 40))
def test_long_single_string(hh, w):
    # multi-level last-arriver merges within one string (n_inst >> 8^3)
    import torch

    v = o.variant(w)
    n = 64 * 4096 * v.m * 8 + 777  # 262,144 instances -> 6 levels
    buf = hh.fill_bytes(n, 9)
    p = hh.variant(w)
    seed = hh.seed_for_input(bytes(range(32)), p, n)
    got = _u64(hh.hash_fixed(buf, n, seed, p))[0]
    host = np.frombuffer(o.fill_bytes(n, 9), dtype=np.uint8).copy()
    want = coracle.hash_huge(w, host, seed.words_np(0, seed.capacity))
    assert np.array_equal(got, want)


# ------------------------------------------------------------------ API/errors
def test_seed_size_error_and_capacity(hh):
    p = hh.variant(24)
    data = bytes(100000)
    small = hh.expand_seed(b"\0" * 32, hh.seed_words_needed(p, 64))
    with pytest.raises(hh.SeedSizeError):
        hh.hash_bytes(data, small, p)
    d = o.fill_bytes(5000)
    exact = hh.hash_bytes(d, hh.seed_for_input(b"\0" * 32, p, len(d)), p)
    big = hh.hash_bytes(d, hh.expand_seed(b"\0" * 32, 10 ** 5), p)
    assert exact == big


def test_engine_and_counter_errors(hh):
    p = hh.variant(24)
    s = hh.seed_for_input(b"\0" * 32, p, 0)
    # the reference's engine names are aliases (identical digests)
    assert hh.hash_bytes(b"", s, p, engine="lanes") == hh.hash_bytes(b"", s, p)
    with pytest.raises(ValueError):
        hh.hash_bytes(b"", s, p, engine="numpy")
    with pytest.raises(ValueError):
        hh.hash_bytes(b"", s, p, counter=object())
    with pytest.raises(ValueError):
        hh.digest(b"", b"\0" * 32, 20)


def test_device_seed_expansion_matches_host(hh):
    s = hh.expand_seed(bytes(range(32)), 3000)
    dev = s.device_words().cpu().numpy().view(np.uint64)
    assert np.array_equal(dev, s.words_np(0, 3000))


def test_host_batch_entry(hh):
    p = hh.variant(40)
    n, B = 70000, 37
    host = np.frombuffer(o.fill_bytes(B * n, 4), dtype=np.uint8).copy()
    got = hh.hash_fixed_host(host, B, n, bytes(range(32)), p)
    S = o.splitmix_words(o.master_fold(bytes(range(32))), 0, o.seed_words_needed(o.variant(40), n))
    want = coracle.hash_fixed(40, host, B, n, n, S)
    assert np.array_equal(got, want)


def test_hash_words_seam(hh):
    # the _hash_words_np seam (hasher.py:331-413) on a (B, n_words) batch
    p = hh.variant(32)
    n_bytes = 2048
    rng = np.random.default_rng(0)
    words = rng.integers(0, 1 << 64, size=(100, n_bytes // 8), dtype=np.uint64)
    seed = hh.seed_for_input(bytes(range(32)), p, n_bytes)
    got = hh.hash_words(words, n_bytes, seed, p)
    want = o.hash_batch(o.variant(32), words, n_bytes, seed.words_np(0, seed.capacity))
    assert np.array_equal(got, want)


# ------------------------------------------------------------------ slices (config 5)
@pytest.mark.parametrize("w", VARIANTS)
def test_slices_and_merge_match_full(hh, w):
    # emulate N ranks one after another on one GPU (no kernel waits on another)
    import torch

    from paper_2104_08865_b200 import multi_gpu

    v = o.variant(w)
    for inst in (600, 8 ** 4 + 8 ** 3 * 3 + 11, 8 ** 5 * 2 + 8 ** 4 + 5):
        n = inst * v.m * 8 + 45
        buf = hh.fill_bytes(n, 12)
        p = hh.variant(w)
        seed = hh.seed_for_input(bytes(range(32)), p, n)
        full = _u64(hh.hash_fixed(buf, n, seed, p))[0]
        host = np.frombuffer(o.fill_bytes(n, 12), dtype=np.uint8).copy()
        want = coracle.hash_one(w, host, seed.words_np(0, seed.capacity))
        assert np.array_equal(full, want)
        for ns in (1, 2, 3, 8):
            plan = multi_gpu.slice_plan(p, n, ns)
            frs, parts = [], []
            for i in range(ns):
                b0, b1 = plan.byte_range(i)
                fr, part = multi_gpu.hash_slice(buf[b0:], plan, i, seed)
                frs.append(fr.clone())
                parts.append(part.clone())
            got = multi_gpu.hash_merge(torch.cat(frs), torch.stack(parts), plan, seed)
            assert np.array_equal(_u64(got), want), (w, inst, ns)


@pytest.mark.slow
def test_config5_full_16gib(hh):
    # config 5: one 16 GiB string, 16-byte variant; GPU single-device digest,
    # 8-slice decomposition and the threaded C oracle must all agree
    import torch

    from paper_2104_08865_b200 import multi_gpu
    from workloads import DATA_SEED, MASTER

    n = 16 << 30
    p = hh.variant(16)
    buf = hh.fill_bytes(n, DATA_SEED)
    seed = hh.seed_for_input(MASTER, p, n)
    full = _u64(hh.hash_fixed(buf, n, seed, p))[0]
    plan = multi_gpu.slice_plan(p, n, 8)
    frs, parts = [], []
    for i in range(8):
        b0, _ = plan.byte_range(i)
        fr, part = multi_gpu.hash_slice(buf[b0:], plan, i, seed)
        frs.append(fr.clone())
        parts.append(part.clone())
    sliced = _u64(multi_gpu.hash_merge(torch.cat(frs), torch.stack(parts), plan, seed))
    del buf
    torch.cuda.empty_cache()
    host = coracle.splitmix(DATA_SEED, 0, n // 8).view(np.uint8)
    want = coracle.hash_huge(16, host, seed.words_np(0, seed.capacity))
    assert np.array_equal(full, want)
    assert np.array_equal(sliced, want)
    # and the digest the reference itself produced for this string
    # (tests/golden/deep_vectors.jsonl, chunked harness over its internals)
    import json
    import os

    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "deep_vectors.jsonl")) as fh:
        ref = [r for r in map(json.loads, fh) if r["kind"] == "huge"][0]
    assert ref["length"] == n and bytes.fromhex(ref["master"]) == MASTER
    assert full.tobytes().hex() == ref["digest"]


# ------------------------------------------------------------------ many seeds
def test_many_seeds_reference_records(hh):
    # the reference's batched seam with per-row folds (tests/test_hasher.py:254-287 style),
    # records generated by running the reference (tests/golden/make_golden.py)
    recs = records("fold")
    assert len(recs) == 16
    r0 = recs[0]
    data = gen_bytes(r0["generator"], r0["length"])
    words = np.frombuffer(data, dtype="<u8").astype(np.uint64)
    folds = [r["fold"] for r in recs]
    got = hh.hash_words_many_seeds(words, r0["length"], folds, hh.variant(r0["variant"]))
    for r, row in zip(recs, got):
        assert _hex(row) == r["digest"]


@pytest.mark.parametrize("w", VARIANTS)
def test_many_seeds_vs_oracle(hh, w):
    import torch

    v = o.variant(w)
    rng = np.random.default_rng(w + 100)
    for n in (0, 5, 100, v.m * 8 - 1, v.m * 8 + 3, 9 * v.m * 8 + 17, 70 * v.m * 8 + 5, 600 * v.m * 8 + 1):
        B = 9
        folds = rng.integers(0, 1 << 64, size=B, dtype=np.uint64)
        data = np.frombuffer(o.fill_bytes(max(n, 1), 21), dtype=np.uint8).copy()
        t = torch.from_numpy(data).cuda()
        got = _u64(hh.hash_fixed_folds(t, n, folds, hh.variant(w), stride=0))
        for b in range(B):
            S = o.splitmix_words(int(folds[b]), 0, o.seed_words_needed(v, n))
            want = coracle.hash_one(w, data[:n], S)
            assert np.array_equal(got[b], want), (w, n, b)
        # distinct inputs too (stride = n rounded to 16)
        stride = (n + 15) // 16 * 16
        buf = hh.fill_bytes(B * max(stride, 16), 22)
        got2 = _u64(hh.hash_fixed_folds(buf, n, folds, hh.variant(w), stride=max(stride, 16)))
        host = np.frombuffer(o.fill_bytes(B * max(stride, 16), 22), dtype=np.uint8).copy()
        for b in range(B):
            S = o.splitmix_words(int(folds[b]), 0, o.seed_words_needed(v, n))
            s0 = b * max(stride, 16)
            assert np.array_equal(got2[b], coracle.hash_one(w, host[s0:s0 + n], S)), (w, n, b, "strided")


@pytest.mark.parametrize("w", VARIANTS)
def test_many_seeds_every_length_up_to_three_instances(hh, w):
    # the per-seed job kernel (every length goes through hash_kernel with
    # seeds recomputed from each row's fold), lengths 0 .. 3 instances
    import torch

    v = o.variant(w)
    folds = np.array([7, 0xFFFFFFFFFFFFFFFF], dtype=np.uint64)
    data = np.frombuffer(o.fill_bytes(3 * v.m * 8, 23), dtype=np.uint8).copy()
    t = torch.from_numpy(data).cuda()
    p = hh.variant(w)
    for n in range(0, 3 * v.m * 8):
        got = _u64(hh.hash_fixed_folds(t, n, folds, p, stride=0))
        for b in range(2):
            S = o.splitmix_words(int(folds[b]), 0, o.seed_words_needed(v, n))
            assert np.array_equal(got[b], coracle.hash_one(w, data[:n], S)), (w, n, b)


def test_many_seeds_collision_smoke(hh):
    # GPU-scale version of the reference's seam test (tests/test_hasher.py:263-281):
    # two 2 KB inputs one byte apart under 10^6 seeds -> no colliding digest
    import torch

    p = hh.variant(24)
    n = 2048
    rng = np.random.default_rng(31)
    a = rng.integers(0, 1 << 64, size=n // 8, dtype=np.uint64)
    b = a.copy()
    b[100] ^= np.uint64(0xFF00000000)
    folds = rng.integers(0, 1 << 64, size=10 ** 6, dtype=np.uint64)
    da = hh.hash_fixed_folds(torch.from_numpy(a.view(np.uint8)).cuda(), n, folds, p, stride=0)
    db = hh.hash_fixed_folds(torch.from_numpy(b.view(np.uint8)).cuda(), n, folds, p, stride=0)
    assert int(torch.all(da == db, dim=1).sum()) == 0


# ------------------------------------------------------------------ CLI / vector wire format
def test_cli_vectors_match_reference_grid(hh, tmp_path):
    from paper_2104_08865_b200.__main__ import main

    path = tmp_path / "vectors.txt"
    assert main(["vectors", "--emit", str(path)]) == 0
    ours = [line.strip() for line in open(path) if line.strip()]
    ref = [r["line"] for r in records("cli_grid")]  # the reference's own vector file (cli.py:189-201)
    assert ours == ref
    assert main(["vectors", "--check", str(path)]) == 0
    path.write_text("\n".join(ours[:-1] + [ours[-1][:-2] + "00"]) + "\n")
    assert main(["vectors", "--check", str(path)]) == 1


def test_cli_hash_empty_stdin(hh, monkeypatch, capsys):
    # reference CLI golden (pkg/tests/test_cli.py:8, 26-30): 24-byte digest of empty stdin
    import io

    from paper_2104_08865_b200.__main__ import main

    monkeypatch.setattr("sys.stdin", io.TextIOWrapper(io.BytesIO(b"")))
    assert main(["hash"]) == 0
    assert capsys.readouterr().out.strip() == "f76f757856e9c252a8a1ce42dc0e2a5df09d621286a62a2d"
    assert main(["hash", "--seed-hex", "00"]) == 2


def test_cli_bench_csv_contract(hh, capsys):
    # the reference's bench CSV contract (pkg/tests/test_cli.py:117-129)
    from paper_2104_08865_b200.__main__ import main

    assert main(["bench", "--sizes", "1K,4K", "--reps", "2"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0] == "size_bytes,variant,bytes_per_second,bytes_per_cycle"
    rows = [line.split(",") for line in lines[1:]]
    assert len(rows) == 2 * 4
    for size, width, bps, bpc in rows:
        assert int(size) in (1024, 4096)
        assert int(width) in (16, 24, 32, 40)
        assert float(bps) > 0
        assert bpc == ""


# ------------------------------------------------------------------ edge cases
def test_empty_batches_and_zero_length(hh):
    import torch

    p = hh.variant(32)
    seed = hh.seed_for_input(b"\0" * 32, p, 0)
    buf = torch.zeros(16, dtype=torch.uint8, device="cuda")
    out = hh.hash_fixed(buf, 0, seed, p, n_strings=0, stride=16)
    assert out.shape == (0, 4)
    out = hh.hash_fixed(buf, 0, seed, p, n_strings=5, stride=0)  # five empty strings
    want = o.hash_batch(o.variant(32), np.zeros((1, 0), np.uint64), 0, seed.words_np(0, seed.capacity))[0]
    assert all(np.array_equal(row, want) for row in _u64(out))
    got = hh.hash_varlen(buf, np.array([0, 0, 0], dtype=np.uint64), seed, p)
    assert all(np.array_equal(row, want) for row in _u64(got))


def test_varlen_mixed_huge_and_tiny(hh):
    # multi-level merges (level >= 3 scratch) next to tail-only strings in one varlen call
    w = 24
    v = o.variant(w)
    lengths = np.array([0, 3, 5000, 600 * v.m * 8 + 7, 1, 70 * v.m * 8, 4097 * v.m * 8 + 13, 100, 64 * v.m * 8],
                       dtype=np.int64)
    from workloads import offsets_of

    off = offsets_of(lengths) + np.uint64(5)  # unaligned base offset for every string
    total = int(off[-1])
    buf = hh.fill_bytes(total, 31)
    p = hh.variant(w)
    seed = hh.seed_for_input(bytes(range(32)), p, int(lengths.max()))
    got = _u64(hh.hash_varlen(buf, off, seed, p))
    host = np.frombuffer(o.fill_bytes(total, 31), dtype=np.uint8).copy()
    want = coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity))
    assert np.array_equal(got, want)


def test_varlen_bound_violation_is_flagged(hh):
    import ctypes

    import torch

    from paper_2104_08865_b200 import _lib, batch

    p = hh.variant(16)
    off = np.array([0, 100, 7000], dtype=np.uint64)  # string 1: 9 instances -> 2 levels
    buf = hh.fill_bytes(7000, 2)
    seed = hh.seed_for_input(b"\0" * 32, p, 7000)
    with pytest.raises(hh.SeedSizeError):  # host-side bound check against capacity
        hh.hash_varlen(buf, off, hh.seed_for_input(b"\0" * 32, p, 10), p)
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    out = torch.empty((2, 2), dtype=torch.int64, device="cuda")
    ws = torch.zeros(batch.workspace_varlen(p, 2, 7000), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    L = _lib.lib()
    rc = L.hth_hash_varlen(16, buf.data_ptr(), d_off.data_ptr(), 2, 200, 7000, seed.fold,
                           seed.device_words().data_ptr(), seed.capacity, out.data_ptr(), ws.data_ptr(),
                           ws.numel(), st)
    assert rc == 0
    assert L.hth_varlen_status(ws.data_ptr(), st) == _lib.HTH_ESEEDSIZE  # string 1 exceeds max_n_bytes
    rc = L.hth_hash_varlen(16, buf.data_ptr(), d_off.data_ptr(), 2, 7000, 7000, seed.fold,
                           seed.device_words().data_ptr(), seed.capacity, out.data_ptr(), ws.data_ptr(),
                           ws.numel(), st)
    assert rc == 0 and L.hth_varlen_status(ws.data_ptr(), st) == 0


def test_varlen_undeclared_bytes_are_flagged(hh):
    # total_bytes sizes the job queues; a batch holding more instances than it
    # declares must be reported (HTH_EINVAL), never written out of bounds
    import torch

    from paper_2104_08865_b200 import _lib, batch

    p = hh.variant(40)
    lengths = np.full(300, 960 * 3, dtype=np.uint64)  # 300 strings of 3 instances
    off = np.zeros(301, dtype=np.uint64)
    off[1:] = np.cumsum(lengths)
    total = int(off[-1])
    buf = hh.fill_bytes(total, 4)
    seed = hh.seed_for_input(b"\1" * 32, p, 960 * 3)
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    out = torch.empty((300, 5), dtype=torch.int64, device="cuda")
    small = 960 * 3 * 10  # declares 10 strings' worth
    ws = torch.zeros(batch.workspace_varlen(p, 300, small) + 4096, dtype=torch.uint8, device="cuda")
    guard = ws[-4096:].clone()
    st = torch.cuda.current_stream().cuda_stream
    L = _lib.lib()
    rc = L.hth_hash_varlen(40, buf.data_ptr(), d_off.data_ptr(), 300, 960 * 3, small, seed.fold,
                           seed.device_words().data_ptr(), seed.capacity, out.data_ptr(), ws.data_ptr(),
                           ws.numel() - 4096, st)
    assert rc == 0
    assert L.hth_varlen_status(ws.data_ptr(), st) == _lib.HTH_EINVAL
    assert torch.equal(ws[-4096:], guard)  # nothing written past the declared workspace
    # declared correctly, the same batch hashes cleanly and matches the oracle
    got = _u64(hh.hash_varlen(buf, off, seed, p))
    host = np.frombuffer(o.fill_bytes(total, 4), dtype=np.uint8).copy()
    assert np.array_equal(got, coracle.hash_varlen(40, host, off, seed.words_np(0, seed.capacity)))


def test_concurrent_streams(hh):
    # independent calls on two streams with their own workspaces give the same digests
    import torch

    from paper_2104_08865_b200 import batch

    w = 40
    v = o.variant(w)
    n = 1100 * v.m * 8 + 9
    p = hh.variant(w)
    seed = hh.seed_for_input(bytes(range(32)), p, n)
    bufs = [hh.fill_bytes(4 * n, 40 + i) for i in range(2)]
    seed.device_words()
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for i, stv in enumerate(streams):
        with torch.cuda.stream(stv):
            ws = torch.zeros(batch.workspace_fixed(p, 4, n), dtype=torch.uint8, device="cuda")
            outs.append(hh.hash_fixed(bufs[i], n, seed, p, n_strings=4, stride=n, workspace=ws))
    torch.cuda.synchronize()
    for i in range(2):
        host = np.frombuffer(o.fill_bytes(4 * n, 40 + i), dtype=np.uint8).copy()
        want = coracle.hash_fixed(w, host, 4, n, n, seed.words_np(0, seed.capacity))
        assert np.array_equal(_u64(outs[i]), want)


def test_host_api_strides_and_capacity(hh):
    p = hh.variant(16)
    n, B, stride = 3001, 21, 3013  # unaligned stride on the host
    host = np.frombuffer(o.fill_bytes(B * stride, 8), dtype=np.uint8).copy()
    got = hh.hash_fixed_host(host, B, n, bytes(range(32)), p, stride=stride)
    S = o.splitmix_words(o.master_fold(bytes(range(32))), 0, o.seed_words_needed(o.variant(16), n))
    want = coracle.hash_fixed(16, host, B, stride, n, S)
    assert np.array_equal(got, want)
    with pytest.raises(hh.SeedSizeError):
        hh.hash_fixed_host(host, B, n, bytes(range(32)), p, stride=stride, seed_capacity=5)


def test_host_paths_pageable_staging_and_small_calls(hh):
    # the host-copy routes of hth_hash_fixed_host: <= 64 KiB calls read
    # mapped pinned memory, <= 256 KiB go through pinned staging on one
    # stream, larger pageable inputs through the parallel memcpy into pinned
    # slots (quarter-size slices from 256 KiB, 16 MiB slots for large ones, a
    # partial last slice), pinned sources straight to the DMA engine -- all
    # equal to the oracle
    import torch

    master = bytes(range(32))
    for w, n in ((24, 100), (40, 200_000), (32, 300_001), (24, (1 << 20) + 3), (40, (5 << 20) + 77),
                 (16, (40 << 20) + 13), (40, (33 << 20) + 5)):
        p = hh.variant(w)
        data = o.fill_bytes(n, 11)
        S = o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(o.variant(w), n))
        want = coracle.hash_one(w, np.frombuffer(data, dtype=np.uint8), S)
        got = hh.hash_bytes(data, hh.seed_for_input(master, p, n), p)
        assert tuple(int(x) for x in want) == got.words, (w, n)
    # a pageable batch whose chunk copies take the staging path, and the same
    # bytes from pinned memory
    p = hh.variant(32)
    n, B = 1 << 20, 24
    host = np.frombuffer(o.fill_bytes(B * n, 12), dtype=np.uint8).copy()
    S = o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(o.variant(32), n))
    want = coracle.hash_fixed(32, host, B, n, n, S)
    assert np.array_equal(hh.hash_fixed_host(host, B, n, master, p), want)
    pinned = torch.from_numpy(host).pin_memory()
    assert np.array_equal(hh.hash_fixed_host(pinned, B, n, master, p), want)


def test_host_batch_many_chunks(hh):
    # hth_hash_fixed_host cuts a large batch into ~64 MiB chunks over three
    # streams and three device buffers (reused from the fourth chunk on), and
    # copies the digests back once: 260 x 1 MiB (5 chunks, a short last one)
    # from pageable and from pinned memory, against the oracle
    import torch

    master = bytes(range(32))
    p = hh.variant(40)
    n, B = (1 << 20) + 40, 260
    stride = n + 24
    host = np.frombuffer(o.fill_bytes(B * stride, 31), dtype=np.uint8).copy()
    S = o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(o.variant(40), n))
    want = coracle.hash_fixed(40, host, B, stride, n, S)
    got = hh.hash_fixed_host(host, B, n, master, p, stride=stride)
    bad = np.nonzero(~np.all(got == want, axis=1))[0]
    assert bad.size == 0, f"pageable: {bad.size} mismatches, first {bad[:8]}"
    pinned = torch.from_numpy(host).pin_memory()
    got = hh.hash_fixed_host(pinned, B, n, master, p, stride=stride)
    bad = np.nonzero(~np.all(got == want, axis=1))[0]
    assert bad.size == 0, f"pinned: {bad.size} mismatches, first {bad[:8]}"


def test_host_api_from_many_threads(hh):
    # hash_bytes / hash_fixed_host from 8 Python threads at once (ctypes drops
    # the GIL; each thread gets its own host context, streams and staging):
    # every digest equals the oracle's
    import threading

    master = bytes(range(32))
    errors = []

    def worker(t):
        try:
            rng = np.random.default_rng(900 + t)
            for _ in range(40):
                w = int(rng.choice([16, 24, 32, 40]))
                n = int(rng.choice([0, 7, 999, 5000, 70_000, 300_000, 9 << 20]))
                data = rng.integers(0, 256, n, dtype=np.uint8).tobytes()
                p = hh.variant(w)
                got = hh.hash_bytes(data, hh.seed_for_input(master, p, n), p)
                S = o.splitmix_words(o.master_fold(master), 0, o.seed_words_needed(o.variant(w), n))
                want = coracle.hash_one(w, np.frombuffer(data, dtype=np.uint8), S)
                if tuple(int(x) for x in want) != got.words:
                    errors.append((t, w, n))
        except Exception as ex:  # pragma: no cover - surfaced below
            errors.append((t, repr(ex)))

    threads = [threading.Thread(target=worker, args=(t,)) for t in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors[:5]


# ------------------------------------------------------------------ streaming
@pytest.mark.parametrize("w", (16, 40))
def test_stream_hasher_matches_one_shot(hh, w):
    import torch

    from paper_2104_08865_b200.stream import StreamHasher

    v = o.variant(w)
    ib = v.m * 8
    rng = np.random.default_rng(w)
    p = hh.variant(w)
    for inst, extra in ((0, 0), (0, 77), (100, 5), (511, 0), (512, 0), (512, 9), (1024, 0), (1024, 3),
                        (3 * 512 + 17, 41), (5000, 1)):
        n = inst * ib + extra
        data = o.fill_bytes(n, 55)
        seed = hh.seed_for_input(bytes(range(32)), p, n)
        want = hh.hash_bytes(data, seed, p)
        for trial in range(2):
            h = StreamHasher(p, seed, n, slice_bytes=512 * ib)  # c = 3: slices of 512 instances
            pos = 0
            while pos < n:
                step = int(rng.integers(1, max(2, n // 3)))
                chunk = data[pos:pos + step]
                h.update(torch.frombuffer(bytearray(chunk), dtype=torch.uint8).cuda() if trial else chunk)
                pos += len(chunk)
            assert h.digest() == want, (w, inst, extra, trial)
    h = StreamHasher(p, hh.seed_for_input(b"\0" * 32, p, 10), 10)
    h.update(b"12345")
    with pytest.raises(ValueError):
        h.digest()
    with pytest.raises(ValueError):
        h.update(b"123456")


def test_cuda_graph_replays(hh):
    # one captured sequence (a multi-job fixed batch whose counters and
    # accumulators self-reset, then a varlen batch: planner + job kernel as a
    # programmatic dependent), replayed several times on the same workspaces:
    # every replay must reproduce the oracle digests
    import torch

    from paper_2104_08865_b200 import batch
    from workloads import offsets_of

    w = 40
    p = hh.variant(w)
    n, B = 1100 * o.variant(w).m * 8 + 13, 5  # 1,100 instances: level-2 jobs with merges
    fbuf = hh.fill_bytes(B * n, 70)
    fseed = hh.seed_for_input(bytes(range(32)), p, n)
    fws = torch.zeros(batch.workspace_fixed(p, B, n), dtype=torch.uint8, device="cuda")
    fout = torch.empty((B, p.output_words), dtype=torch.int64, device="cuda")
    lengths = np.random.default_rng(71).integers(0, 70000, 500).astype(np.int64)
    off = offsets_of(lengths)
    total = int(off[-1])
    vbuf = hh.fill_bytes(total, 72)
    d_off = torch.from_numpy(off.view(np.int64)).cuda()
    vseed = hh.seed_for_input(bytes(range(32)), p, int(lengths.max()))
    vws = torch.zeros(batch.workspace_varlen(p, len(lengths), total), dtype=torch.uint8, device="cuda")
    vout = torch.empty((len(lengths), p.output_words), dtype=torch.int64, device="cuda")

    def step():
        hh.hash_fixed(fbuf, n, fseed, p, n_strings=B, stride=n, out=fout, workspace=fws)
        hh.hash_varlen(vbuf, d_off, vseed, p, max_n_bytes=int(lengths.max()), out=vout, workspace=vws, check=False)

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        step()  # warm-up outside capture (first-layout workspace clear)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    fwant = coracle.hash_fixed(w, np.frombuffer(o.fill_bytes(B * n, 70), dtype=np.uint8).copy(), B, n, n,
                               fseed.words_np(0, fseed.capacity))
    vwant = coracle.hash_varlen(w, np.frombuffer(o.fill_bytes(total, 72), dtype=np.uint8).copy(), off,
                                vseed.words_np(0, vseed.capacity))
    for _ in range(3):
        fout.zero_()
        vout.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(_u64(fout), fwant)
        assert np.array_equal(_u64(vout), vwant)
    batch.varlen_status(vws)


@pytest.mark.parametrize("n_strings", (2047, 2048))
def test_job_level_threshold(hh, n_strings):
    # 600-instance strings: 2047 of them make 4094 level-3 jobs (the batch
    # runs level-2 jobs), 2048 make 4096 (level-3 jobs); digests must agree
    # with the oracle either way
    w = 16
    v = o.variant(w)
    n = 600 * v.m * 8 + 5
    stride = n + 11
    buf = hh.fill_bytes(n_strings * stride, 80)
    p = hh.variant(w)
    seed = hh.seed_for_input(bytes(range(32)), p, n)
    got = _u64(hh.hash_fixed(buf, n, seed, p, n_strings=n_strings, stride=stride))
    host = np.frombuffer(o.fill_bytes(n_strings * stride, 80), dtype=np.uint8).copy()
    want = coracle.hash_fixed(w, host, n_strings, stride, n, seed.words_np(0, seed.capacity))
    assert np.array_equal(got, want)


def test_varlen_many_pair_jobs_dynamic_claims(hh):
    # thousands of one-level strings of 1-4 instances (pair jobs, claimed
    # dynamically), odd counts per class, random tails and alignments, mixed
    # with multi-job strings whose last job is small (class 5)
    from workloads import offsets_of

    w = 24
    iw = o.variant(w).m * 8
    rng = np.random.default_rng(90)
    c = rng.integers(1, 5, 6001)
    lengths = c * iw + rng.integers(0, iw, c.size)
    multi = (64 * rng.integers(1, 3, 41) + rng.integers(1, 5, 41)) * iw + rng.integers(0, iw, 41)
    lengths = rng.permutation(np.concatenate([lengths, multi, rng.integers(0, iw, 300)]).astype(np.int64))
    off = offsets_of(lengths)
    total = int(off[-1])
    buf = hh.fill_bytes(total, 91)
    p = hh.variant(w)
    seed = hh.seed_for_input(bytes(range(32)), p, int(lengths.max()))
    got = _u64(hh.hash_varlen(buf, off, seed, p))
    host = np.frombuffer(o.fill_bytes(total, 91), dtype=np.uint8).copy()
    want = coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity))
    bad = np.nonzero(~np.all(got == want, axis=1))[0]
    assert bad.size == 0, f"{bad.size} mismatches; lengths {lengths[bad[:8]]}"


def test_hash_remainder_on_the_gpu(hh):
    # hash_remainder (hasher.py:186-206): component i is NH of the tail under
    # the key window starting at i (pkg/tests/test_hasher.py:187-211)
    from paper_2104_08865_b200.hasher import hash_remainder

    M64 = (1 << 64) - 1

    def nh(x, s):
        return (((x + s) & 0xFFFFFFFF) * (((x >> 32) + (s >> 32)) & 0xFFFFFFFF)) & M64

    rng = np.random.default_rng(5)
    for n, k in ((1, 1), (7, 3), (300, 5), (1001, 2)):
        tail = [int(x) for x in rng.integers(0, 1 << 63, n, dtype=np.uint64) * 2 + 1]
        keys = [int(x) for x in rng.integers(0, 1 << 63, n + k + 3, dtype=np.uint64) * 3]
        want = tuple(sum(nh(tail[j], keys[i + j]) for j in range(n)) & M64 for i in range(k))
        assert hash_remainder(tail, keys, k) == want, (n, k)
    # the windows overlap: component i+1 of keys == component i of keys[1:]
    tail, keys = [5, 6, 7], [11, 12, 13, 14, 15]
    a, b = hash_remainder(tail, keys, 3), hash_remainder(tail, keys[1:], 2)
    assert a[1:] == b
