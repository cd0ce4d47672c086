"""cfg4 throughput vs run length, with nvidia-smi clocks/power sampled during each run (diagnostic)."""
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_08865_b200 as hh  # noqa: E402

ctx = bench.setup_fixed(hh, torch, sys.argv[1] if len(sys.argv) > 1 else "cfg4")
for steps in (10, 30, 100, 300, 1000):
    s = bench.ClockSampler(0)
    s.start()
    time.sleep(0.2)
    total_ms, per, (w0, w1) = bench.run_fixed(hh, torch, ctx, steps, 5)
    time.sleep(0.1)
    s.stop()
    ms = total_ms / steps
    pw = [float(l.split(",")[2]) for (_, l) in s.lines if len(l.split(",")) > 3]
    print(f"steps={steps:5d} {ms:.3f} ms/step {ctx['B'] * ctx['n'] / ms / 1e6:.0f} GB/s clocks={s.summary(w0, w1)} "
          f"max_power={max(pw) if pw else None}", flush=True)
    time.sleep(2)
