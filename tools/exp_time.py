"""Time one config's hash kernel with the library named by $HTH_LIB (experiments)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_08865_b200 as hh  # noqa: E402

wk = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
if wk.startswith("fixed:"):  # fixed:<variant>:<n_strings>:<n_bytes>
    _, w_, b_, n_ = wk.split(":")
    bench.wl.CONFIGS[wk] = dict(desc=wk, variant=int(w_), n_strings=int(b_), n_bytes=int(n_))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ctx = bench.setup_fixed(hh, torch, wk)
flush = bench.make_flush(torch) if wk == "cfg1" else None  # as bench.py: L2 flushed per step
total_ms, per, _ = bench.run_fixed(hh, torch, ctx, steps, 5, flush)
ms = total_ms / steps
gbs = ctx["B"] * ctx["n"] / ms / 1e6
from oracle import c as coracle  # noqa: E402
import workloads as wl  # noqa: E402
nchk = min(2, ctx["B"]) if ctx["n"] <= (1 << 24) else 0
got = ctx["out"][:nchk].cpu().numpy().view(np.uint64)
host = np.frombuffer(b"".join(wl.host_bytes(i * ctx["n"], ctx["n"]) for i in range(nchk)), np.uint8).copy()
want = coracle.hash_fixed(ctx["w"], host, nchk, ctx["n"], ctx["n"], ctx["seed"].words_np(0, ctx["seed"].capacity))
print(f"{os.path.basename(os.environ.get('HTH_LIB', 'default'))} {wk} x{steps}: {ms:.3f} ms  {gbs:.0f} GB/s  ok={np.array_equal(got, want)}")
