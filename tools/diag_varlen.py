"""Which config-2 strings mismatch the oracle, by instance count (debug aid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2104_08865_b200 as hh  # noqa: E402
import workloads as wl  # noqa: E402
from oracle import c as coracle  # noqa: E402
from oracle import oracle_np as o  # noqa: E402

w = int(sys.argv[1]) if len(sys.argv) > 1 else 16
lengths = wl.cfg2_lengths()
off = wl.offsets_of(lengths)
total = int(off[-1])
buf = hh.fill_bytes(total, wl.DATA_SEED)
host = buf[:total].cpu().numpy()
p = hh.variant(w)
seed = hh.seed_for_input(wl.MASTER, p, int(lengths.max()))
got = hh.hash_varlen(buf, off, seed, p).cpu().numpy().view(np.uint64)
want = coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity))
m = o.variant(w).m
ni = ((lengths + 7) // 8) // m
bad = ~np.all(got == want, axis=1)
print("mismatches", int(bad.sum()), "of", len(lengths))
for c in sorted(set(ni[bad].tolist()))[:20]:
    sel = ni == c
    print(f"  ni={c}: {int((bad & sel).sum())} / {int(sel.sum())}; e.g. lengths {lengths[bad & sel][:5]}")
