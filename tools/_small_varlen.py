import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, paper_2104_08865_b200 as hh, workloads as wl
from oracle import c as coracle
lengths = wl.cfg2_lengths(2000, seed=3)
off = wl.offsets_of(lengths); total = int(off[-1])
buf = hh.fill_bytes(total, 3)
for w in (40,):
    p = hh.variant(w); seed = hh.seed_for_input(wl.MASTER, p, int(lengths.max()))
    got = hh.hash_varlen(buf, off, seed, p).cpu().numpy().view(np.uint64)
    want = coracle.hash_varlen(w, buf[:total].cpu().numpy(), off, seed.words_np(0, seed.capacity))
    print("ok", np.array_equal(got, want))
