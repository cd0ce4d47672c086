"""CUPTI timeline of one hth_hash_fixed_host call (config 4 strings): copy
engine busy fraction and the gaps between host->device copies."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2104_08865_b200 as hh  # noqa: E402
import workloads as wl  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
n = 1 << 20
p = hh.variant(40)
host = torch.empty(B * n, dtype=torch.uint8, pin_memory=True)
dev = torch.empty(B * n + 16, dtype=torch.uint8, device="cuda")
hh.fill_bytes(B * n, wl.DATA_SEED, 0, out=dev)
host.copy_(dev[:B * n])
del dev
torch.cuda.empty_cache()
hh.hash_fixed_host(host, B, n, wl.MASTER, p)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    hh.hash_fixed_host(host, B, n, wl.MASTER, p)
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
h2d = [e for e in ev if "HtoD" in e.name or "Memcpy HtoD" in e.name]
t0, t1 = ev[0].time_range.start, ev[-1].time_range.end
busy = sum(e.time_range.end - e.time_range.start for e in h2d)
print(f"span {t1 - t0:.0f} us, H2D busy {busy:.0f} us ({100 * busy / (t1 - t0):.1f} %), {len(h2d)} copies, "
      f"{B * n / (t1 - t0) / 1e3:.1f} GB/s over the span")
gaps = [b.time_range.start - a.time_range.end for a, b in zip(h2d, h2d[1:])]
print("first copy starts at +%.0f us; largest gaps between copies (us):" % (h2d[0].time_range.start - t0),
      sorted(gaps)[-8:])
print("after last copy: %.0f us" % (t1 - h2d[-1].time_range.end))
names = {}
for e in ev:
    k = e.name[:50]
    names[k] = names.get(k, 0) + (e.time_range.end - e.time_range.start)
for k, v in sorted(names.items(), key=lambda kv: -kv[1])[:8]:
    print(f"  {v:9.0f} us  {k}")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
