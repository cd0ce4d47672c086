"""Time hash_varlen on config 2's strings per variant with the library named by
$HTH_LIB (experiments); checks the digests against the C oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_08865_b200 as hh  # noqa: E402
from paper_2104_08865_b200 import batch  # noqa: E402
import workloads as wl  # noqa: E402
from oracle import c as coracle  # noqa: E402

lengths = wl.cfg2_lengths()
off = wl.offsets_of(lengths)
total = int(off[-1])
buf = torch.empty(total + 64, dtype=torch.uint8, device="cuda")
hh.fill_bytes(total, wl.DATA_SEED, 0, out=buf)
d_off = torch.from_numpy(off.view(np.int64)).cuda()
mx = int(lengths.max())
host = buf[:total].cpu().numpy()
only = [int(x) for x in sys.argv[1:]] or [16, 24, 32, 40]
for w in only:
    p = hh.variant(w)
    seed = hh.seed_for_input(wl.MASTER, p, mx)
    out = hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=mx)
    torch.cuda.synchronize()
    want = coracle.hash_varlen(w, host, off, seed.words_np(0, seed.capacity))
    ok = np.array_equal(out.cpu().numpy().view(np.uint64), want)
    ws = torch.zeros(batch.workspace_varlen(p, len(lengths), total), dtype=torch.uint8, device="cuda")
    for _ in range(5):
        hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=mx, workspace=ws, check=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record()
    for _ in range(n):
        hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=mx, workspace=ws, check=False)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    hh.varlen_status(ws)
    again = hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=mx, workspace=ws)
    ok = ok and np.array_equal(again.cpu().numpy().view(np.uint64), want)
    print(f"{os.path.basename(os.environ.get('HTH_LIB', 'default'))} v{w}: {us:.1f} us/call  "
          f"{total / us / 1e3:.0f} GB/s  ok={ok}")
