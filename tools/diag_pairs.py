"""Pair-job debug: homogeneous varlen batches of c-instance strings."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2104_08865_b200 as hh  # noqa: E402
import workloads as wl  # noqa: E402
from oracle import c as coracle  # noqa: E402
from oracle import oracle_np as o  # noqa: E402

for w in (16, 40):
    iw = o.variant(w).m * 8
    p = hh.variant(w)
    for c in (1, 4, 5):
        for count in (100, 3000):
            for tail in ("none", "rand"):
                rng = np.random.default_rng(c * 7 + count)
                t = rng.integers(0, iw, count) if tail == "rand" else np.zeros(count, dtype=np.int64)
                lengths = (c * iw + t).astype(np.int64)
                off = wl.offsets_of(lengths)
                total = int(off[-1])
                buf = hh.fill_bytes(total, 3)
                host = buf[:total].cpu().numpy()
                seed = hh.seed_for_input(wl.MASTER, p, int(lengths.max()))
                got = hh.hash_varlen(buf, off, seed, p).cpu().numpy().view(np.uint64)
                want = coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity))
                bad = np.nonzero(~np.all(got == want, axis=1))[0]
                print(f"v{w} c={c} count={count} tail={tail}: {bad.size} bad; idx {bad[:10]} parity {np.bincount(bad % 2, minlength=2) if bad.size else ''}")
