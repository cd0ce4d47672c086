"""Config 5's in-stream exchange protocol (FlagExchange) on one GPU.

The ranks' slices run one after another on one stream in one process
(multi_gpu.hash_string_emulated), so every flag a kernel waits on was raised
by an earlier launch: no kernel ever waits on a concurrently running one.
What is checked is the protocol's data path: slice kernels that accumulate
into pre-zeroed partials and raise arrival flags (also for empty slices),
the merge kernel that waits on the flags, merges, re-zeroes the partials and
releases the slot, and double-buffered slot reuse over several strings --
every digest equal to the C oracle."""

import numpy as np
import pytest

from oracle import c as coracle
from oracle import oracle_np as o

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hh():
    import torch

    import paper_2104_08865_b200 as h

    assert torch.cuda.is_available()
    return h


@pytest.mark.parametrize("w", (16, 24, 32, 40))
def test_flag_protocol_matches_oracle_over_many_strings(hh, w):
    from paper_2104_08865_b200 import multi_gpu

    v = o.variant(w)
    for inst in (70, 600, 8 ** 4 + 8 ** 3 * 3 + 11, 8 ** 5 * 2 + 8 ** 4 + 5):
        n = inst * v.m * 8 + 45
        p = hh.variant(w)
        seed = hh.seed_for_input(bytes(range(32)), p, n)
        for ns in (1, 2, 3, 8):
            plan = multi_gpu.slice_plan(p, n, ns)
            state = None
            # five strings through the two slots: a slot whose partials were
            # not re-zeroed would corrupt the third string on
            for epoch in range(1, 6):
                fill = 100 + epoch
                buf = hh.fill_bytes(n, fill)
                d, state = multi_gpu.hash_string_emulated(buf, plan, seed, epoch, state)
                got = d.cpu().numpy().view(np.uint64)
                host = np.frombuffer(o.fill_bytes(n, fill), dtype=np.uint8).copy()
                want = coracle.hash_one(w, host, seed.words_np(0, seed.capacity))
                assert np.array_equal(got, want), (w, inst, ns, epoch)
            assert int(state["status"].item()) == 0
            lay = multi_gpu._SlotLayout(plan)
            words = state["buf"].cpu().numpy().view(np.uint64)
            flags = words[2 * lay.slot_words:2 * lay.slot_words + 2 * ns].reshape(2, ns)
            consumed = words[2 * lay.slot_words + 2 * ns:]
            assert flags[0].tolist() == [5] * ns and flags[1].tolist() == [4] * ns  # incl. empty slices
            assert consumed.tolist() == [5, 4]
            for slot in (0, 1):  # partials handed back zeroed
                a = slot * lay.slot_words + lay.nfw
                assert not words[a:a + ns * lay.k].any()


def test_wait_times_out_instead_of_hanging(hh):
    # a flag nobody raises: the bounded wait reports status 1 and returns
    import time

    import torch

    from paper_2104_08865_b200 import _lib

    flag = torch.zeros(1, dtype=torch.int64, device="cuda")
    status = torch.zeros(1, dtype=torch.int32, device="cuda")
    t0 = time.perf_counter()
    _lib.check(_lib.lib().hth_wait_flag(flag.data_ptr(), 1, 50_000_000, status.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert int(status.item()) == 1
    assert time.perf_counter() - t0 < 5
    _lib.check(_lib.lib().hth_signal(flag.data_ptr(), 7, torch.cuda.current_stream().cuda_stream))
    status.zero_()
    _lib.check(_lib.lib().hth_wait_flag(flag.data_ptr(), 7, 50_000_000, status.data_ptr(),
                                        torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert int(status.item()) == 0 and int(flag.item()) == 7


def test_fill_strings_matches_host_stream(hh):
    # one-launch shard fill: local string i = global string first + i * step
    for n, B, first, step in ((1024, 37, 3, 8), (4096, 5, 0, 1), (1 << 20, 3, 1, 2)):
        t = hh.fill_strings(B, n, first, step, fill_seed=0)
        got = t[:B * n].cpu().numpy()
        want = np.concatenate([np.frombuffer(o.fill_bytes(n, 0, (first + i * step) * n // 8), dtype=np.uint8)
                               for i in range(B)])
        assert np.array_equal(got, want)
