"""Config 5 full-size parity with explicit timings (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_08865_b200 as hh  # noqa: E402
from oracle import c as coracle  # noqa: E402
from workloads import DATA_SEED, MASTER  # noqa: E402

n = 16 << 30
p = hh.variant(16)
t = time.time()
buf = hh.fill_bytes(n, DATA_SEED)
seed = hh.seed_for_input(MASTER, p, n)
gpu = hh.hash_fixed(buf, n, seed, p).cpu().numpy().view(np.uint64)[0]
print("gpu", [hex(x) for x in gpu], f"{time.time() - t:.2f}s", flush=True)
t = time.time()
host = coracle.splitmix(DATA_SEED, 0, n // 8).view(np.uint8)
print("host gen", host.nbytes, f"{time.time() - t:.2f}s", "cores", os.cpu_count(), flush=True)
sample = buf[:64].cpu().numpy()
print("first bytes equal:", bool(np.array_equal(sample, host[:64])), "last:",
      bool(np.array_equal(buf[n - 64:n].cpu().numpy(), host[n - 64:])), flush=True)
t = time.time()
want = coracle.hash_huge(16, host, seed.words_np(0, seed.capacity))
print("oracle", [hex(x) for x in want], f"{time.time() - t:.2f}s", flush=True)
print("MATCH" if np.array_equal(gpu, want) else "MISMATCH")
