"""Launch the hash kernel of one BASELINE config a few times (for ncu).

  python tools/profile_kernel.py cfg4 [launches]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_08865_b200 as hh  # noqa: E402

wk = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if wk == "cfg2":
    bench.measure_workload(hh, torch, "cfg2", steps=n, warmup=1, peak=6545.0)
else:
    ctx = bench.setup_fixed(hh, torch, wk)
    for _ in range(n):
        hh.hash_fixed(ctx["buf"], ctx["n"], ctx["seed"], ctx["p"], n_strings=ctx["B"], stride=ctx["n"], out=ctx["out"])
    torch.cuda.synchronize()
print("done", wk)
