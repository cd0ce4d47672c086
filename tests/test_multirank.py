"""Multi-rank host logic on CPU: world_size 2 and 3 over gloo.

The slice/merge arithmetic is supplied by the C oracle (test infrastructure);
what is exercised is the product's orchestration -- hth_slice_plan's bounds
and frontier counts, the padded all_gather of frontier roots and partials,
their rank-order concatenation, and the hand-off to merge."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import paper_2104_08865_b200 as hh
from paper_2104_08865_b200 import multi_gpu
from oracle import c as coracle
from oracle import oracle_np as o


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_slice(data, seeds):
    def fn(local, plan, i, seed):
        b0, b1 = plan.byte_range(i)
        assert local.shape[0] == b1 - b0
        fr, part = coracle.slice(plan.params.output_bytes, data, plan.n_bytes, plan.bounds[i], plan.bounds[i + 1],
                                 plan.level, plan.counts[i], seeds)
        return torch.from_numpy(fr.view(np.int64).copy()), torch.from_numpy(part.view(np.int64).copy())
    return fn


def _oracle_merge(seeds):
    def fn(frontier, partials, plan, seed):
        out = coracle.merge(plan.params.output_bytes, plan.n_bytes, plan.level,
                            frontier.numpy().view(np.uint64), partials.numpy().view(np.uint64), seeds)
        return torch.from_numpy(out.view(np.int64).copy())
    return fn


def _worker(rank, world, port, w, inst, result_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = hh.variant(w)
    v = o.variant(w)
    n = inst * v.m * 8 + 77
    data = np.frombuffer(o.fill_bytes(n, 6), dtype=np.uint8).copy()
    seed = hh.seed_for_input(bytes(range(32)), p, n)
    S = seed.words_np(0, seed.capacity)
    plan = multi_gpu.slice_plan(p, n, world)
    b0, b1 = plan.byte_range(rank)
    local = data[b0:b1]
    got = multi_gpu.hash_string_distributed(local, plan, seed, slice_fn=_oracle_slice(data, S),
                                            merge_fn=_oracle_merge(S))
    if rank == 0:
        result_q.put((got.tolist(), coracle.hash_one(w, data, S).tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,w,inst", [(2, 16, 8 ** 4 * 2 + 8 ** 3 * 3 + 5), (3, 40, 8 ** 4 + 123),
                                          (2, 24, 700)])
def test_distributed_string_gloo(world, w, inst):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, w, inst, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got, want = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert got == want


def test_slice_plan_shapes():
    for w in (16, 40):
        p = hh.variant(w)
        for n in (16 << 30, 1 << 30, 5 * 10 ** 6):
            for world in (1, 2, 4, 8):
                plan = multi_gpu.slice_plan(p, n, world)
                sub = 8 ** plan.level
                n_inst = ((n + 7) // 8) // p.instance_words
                assert plan.bounds[0] == 0 and plan.bounds[-1] == n_inst
                assert all(b % sub == 0 for b in plan.bounds[:-1])
                assert plan.n_frontier == (n_inst >> (3 * plan.level)) & ~7
                spans = np.diff(plan.bounds)
                if n_inst > 64 * sub * world:
                    assert spans.max() / spans.mean() < 1.05  # balanced to within a few percent
    plan = multi_gpu.slice_plan(hh.variant(16), 16 << 30, 8)
    assert plan.level == 5 and plan.n_frontier == 680  # SURVEY.md 8(e) example: 682 subtrees at c = 5


def test_round_robin_shards_partition():
    n, world = 8192 * 8, 8
    seen = np.concatenate([multi_gpu.shard_round_robin(n, r, world) for r in range(world)])
    assert np.array_equal(np.sort(seen), np.arange(n))
    blocks = [list(multi_gpu.shard_blocks(4194304, r, 8)) for r in range(8)]
    assert sum(len(b) for b in blocks) == 4194304


def test_flag_exchange_slot_layout():
    # rank 0's exchange buffer: two slots of [frontier | partials], then the
    # arrival flags and consumed words, no overlaps, every rank's frontier
    # range where the plan puts it
    from paper_2104_08865_b200 import multi_gpu

    for w, n, world in ((16, 16 << 30, 8), (40, 8 << 30, 3), (24, 5 << 20, 2)):
        plan = multi_gpu.slice_plan(hh.variant(w), n, world)
        lay = multi_gpu._SlotLayout(plan)
        k = w // 8
        spans = []
        for slot in (0, 1):
            for r in range(world):
                a = lay.frontier(0, slot, r) // 8
                spans.append((a, a + plan.counts[r] * 8 * k))
                b = lay.partials(0, slot, r) // 8
                spans.append((b, b + k))
                f = lay.flag(0, slot, r) // 8
                spans.append((f, f + 1))
            c = lay.consumed(0, slot) // 8
            spans.append((c, c + 1))
        spans = sorted(s for s in spans if s[1] > s[0])
        assert all(a[1] <= b[0] for a, b in zip(spans, spans[1:]))
        assert spans[-1][1] <= lay.words
        assert sum(b - a for a, b in spans) == lay.words
