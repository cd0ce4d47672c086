"""One warm config-2 step (all four variants) for launch-list profiling."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_08865_b200 as hh  # noqa: E402
import workloads as wl  # noqa: E402

lengths = wl.cfg2_lengths()
off = wl.offsets_of(lengths)
total = int(off[-1])
buf = torch.empty(total + 64, dtype=torch.uint8, device="cuda")
hh.fill_bytes(total, wl.DATA_SEED, 0, out=buf)
d_off = torch.from_numpy(off.view(np.int64)).cuda()
mx = int(lengths.max())
seeds = {w: hh.seed_for_input(wl.MASTER, hh.variant(w), mx) for w in (16, 24, 32, 40)}
for it in range(3):
    for w in (16, 24, 32, 40):
        hh.hash_varlen(buf, d_off, seeds[w], hh.variant(w), max_n_bytes=mx)
torch.cuda.synchronize()
print("bytes", total, "strings", len(lengths), "tail-only per variant:",
      {w: int(np.sum(lengths < 8 * hh.variant(w).instance_words * 8 // 8 * 8)) for w in (16, 24, 32, 40)})
