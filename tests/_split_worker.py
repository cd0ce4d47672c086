"""Worker for test_gpu_multiproc.py (run under torch.distributed.run, gloo):
each rank hashes its slice of one string, the roots are exchanged through
rank 0's memory (CUDA-IPC peer mapping) or with all_gather, and rank 0 checks
the digest against the threaded C oracle.  Several ranks may share one GPU:
no kernel waits on another rank (the only cross-rank wait is a host barrier).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    import paper_2104_08865_b200 as hh
    from oracle import c as coracle
    from paper_2104_08865_b200 import multi_gpu

    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    cases = [(16, (64 << 20) + 12345), (40, (48 << 20) + 77), (24, 3 * 1344 * 4096 + 5)]
    for w, n in cases:
        p = hh.variant(w)
        plan = multi_gpu.slice_plan(p, n, world)
        b0, b1 = plan.byte_range(rank)
        local = hh.fill_bytes(b1 - b0, 7, b0 // 8) if b1 > b0 else torch.zeros(16, dtype=torch.uint8, device="cuda")
        seed = hh.seed_for_input(bytes(range(32)), p, n)
        got = [multi_gpu.hash_string_p2p(local, plan, seed) for _ in range(3)]  # both buffers, reused
        got.append(multi_gpu.hash_string_distributed(local, plan, seed))
        if rank == 0:
            host = coracle.splitmix(7, 0, (n + 7) // 8).view(np.uint8)[:n]
            want = coracle.hash_huge(w, host, seed.words_np(0, seed.capacity))
            for i, g in enumerate(got):
                assert np.array_equal(g, want), (w, n, i, g, want)
            print(f"split v{w} n={n} slices={plan.n_slices} level={plan.level} ok", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
