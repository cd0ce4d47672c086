"""hash_bytes wall time (median of 200) for pageable inputs of 256 KiB - 16 MiB."""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_08865_b200 as hh  # noqa: E402

p = hh.variant(24)
out = {}
for n in (300 << 10, 1 << 20, 4 << 20, 8 << 20, 16 << 20, 64 << 20):
    data = os.urandom(n)
    seed = hh.seed_for_input(bytes(range(32)), p, n)
    for _ in range(10):
        hh.hash_bytes(data, seed, p)
    ts = []
    for _ in range(100 if n <= (4 << 20) else 30):
        t0 = time.perf_counter()
        hh.hash_bytes(data, seed, p)
        ts.append(time.perf_counter() - t0)
    out[n >> 10] = round(statistics.median(ts) * 1e6, 1)
print(os.environ.get("HTH_PAGEABLE_DIRECT", "default"), out)
