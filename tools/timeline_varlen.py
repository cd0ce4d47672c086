"""Per-kernel GPU times of one hash_varlen call per variant (torch.profiler /
CUPTI, no replay): shows how the call splits into planning, tail and hash."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2104_08865_b200 as hh  # noqa: E402
import workloads as wl  # noqa: E402

lengths = wl.cfg2_lengths()
off = wl.offsets_of(lengths)
total = int(off[-1])
buf = torch.empty(total + 64, dtype=torch.uint8, device="cuda")
hh.fill_bytes(total, wl.DATA_SEED, 0, out=buf)
d_off = torch.from_numpy(off.view(np.int64)).cuda()
mx = int(lengths.max())
for w in [int(x) for x in sys.argv[1:]] or [16, 24, 32, 40]:
    p = hh.variant(w)
    seed = hh.seed_for_input(wl.MASTER, p, mx)
    for _ in range(5):
        hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=mx)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=mx)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    ev = ev[len(ev) * 2 // 3:]  # last call
    t0 = ev[0].time_range.start
    print(f"v{w}: call span {ev[-1].time_range.end - t0:.1f} us")
    for e in ev:
        print(f"   +{e.time_range.start - t0:7.1f} us  {e.time_range.end - e.time_range.start:7.1f} us  {e.name[:90]}")
