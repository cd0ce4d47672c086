"""Where a small hash_bytes call's time goes (median of 2000 calls each):
Python wrapper, the C-ABI call alone, and a bare torch launch + synchronize."""
import ctypes
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_08865_b200 as hh  # noqa: E402
from paper_2104_08865_b200 import _lib  # noqa: E402


def med(f, n=2000):
    for _ in range(200):
        f()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return round(statistics.median(ts) * 1e6, 2)


p = hh.variant(24)
out = {}
for n in (64, 4096):
    data = bytes(range(256)) * (n // 256) if n >= 256 else bytes(range(n))
    seed = hh.seed_for_input(bytes(range(32)), p, n)
    res = (ctypes.c_uint64 * 3)()
    L = _lib.lib()
    out[f"hash_bytes_{n}"] = med(lambda: hh.hash_bytes(data, seed, p))
    out[f"c_abi_{n}"] = med(lambda: L.hth_hash_host(24, data, n, seed.master, seed.capacity, res, 0))
x = torch.zeros(1, device="cuda")
out["torch_add_sync"] = med(lambda: (x.add_(1), torch.cuda.synchronize()))
out["torch_sync_only"] = med(lambda: torch.cuda.synchronize())
print(out)
