"""Per-warp time structure of one hash_varlen call (config 2) or one
hash_fixed call (config 4) with an HTH_DEBUG_TIMING build:
  HTH_LIB=exp/dbg.so python tools/warp_timeline.py [cfg2 40 | cfg4]
Prints the kernel span, the spread of warp start/end times, jobs and rounds
per warp, and the share of warp time spent waiting for stage data."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_08865_b200 as hh  # noqa: E402
import workloads as wl  # noqa: E402
from paper_2104_08865_b200 import _lib  # noqa: E402

wk = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
lib = _lib.lib()
lib.hth_debug_timing.argtypes = [ctypes.c_void_p, ctypes.c_int]
NW = 8192
rec = np.zeros((NW, 12), dtype=np.uint64)


def run():
    if wk == "cfg2":
        w = int(sys.argv[2]) if len(sys.argv) > 2 else 40
        lengths = wl.cfg2_lengths()
        off = wl.offsets_of(lengths)
        total = int(off[-1])
        buf = torch.empty(total + 64, dtype=torch.uint8, device="cuda")
        hh.fill_bytes(total, wl.DATA_SEED, 0, out=buf)
        d_off = torch.from_numpy(off.view(np.int64)).cuda()
        p = hh.variant(w)
        seed = hh.seed_for_input(wl.MASTER, p, int(lengths.max()))
        return lambda: hh.hash_varlen(buf, d_off, seed, p, max_n_bytes=int(lengths.max()))
    import bench
    ctx = bench.setup_fixed(hh, torch, wk)
    return lambda: hh.hash_fixed(ctx["buf"], ctx["n"], ctx["seed"], ctx["p"], n_strings=ctx["B"], stride=ctx["n"],
                                 out=ctx["out"])


f = run()
for _ in range(3):
    f()
lib.hth_debug_timing(rec.ctypes.data, NW)
f()
lib.hth_debug_timing(rec.ctypes.data, NW)
r = rec[rec[:, 5] != 0].astype(np.float64)
t0 = r[:, 0].min()
st, en = (r[:, 0] - t0) / 1e3, (r[:, 1] - t0) / 1e3
busy = en - st
print(f"{wk}: {len(r)} warps; span {en.max():.1f} us; warp start spread {st.min():.1f}-{st.max():.1f} us; "
      f"end p10/p50/p90/max {np.percentile(en, 10):.1f}/{np.percentile(en, 50):.1f}/{np.percentile(en, 90):.1f}/"
      f"{en.max():.1f} us")
print(f"jobs/warp mean {r[:, 2].mean():.2f} max {r[:, 2].max():.0f}; rounds/warp mean {r[:, 3].mean():.1f} "
      f"max {r[:, 3].max():.0f}; data-wait share of warp time {r[:, 4].sum() / 1e3 / busy.sum():.1%}; "
      f"warp-time utilisation (sum busy / (warps x span)) {busy.sum() / (len(r) * en.max()):.1%}")
je = (r[:, 5] - t0) / 1e3
print(f"job phase end p10/p50/p90/max {np.percentile(je, 10):.1f}/{np.percentile(je, 50):.1f}/{np.percentile(je, 90):.1f}/"
      f"{je.max():.1f} us (then exit)")
print(f"mean us per round (busy / rounds) {busy.sum() / r[:, 3].sum():.2f}")
J = r[:, 2].sum()
idle = busy.sum() - (r[:, 7].sum() + r[:, 8].sum() + r[:, 9].sum()) / 1e3
print(f"per job (us): consumer decode+seeds {r[:, 7].sum() / 1e3 / J:.2f}, round loop {r[:, 8].sum() / 1e3 / J:.2f} "
      f"(of which data wait {r[:, 4].sum() / 1e3 / J:.2f}), finalize+publish {r[:, 9].sum() / 1e3 / J:.2f}, "
      f"other {idle / J:.2f}; producer claims (inside the above) {r[:, 6].sum() / 1e3 / J:.2f}; round-loop us per round "
      f"{(r[:, 8].sum() - r[:, 4].sum()) / 1e3 / r[:, 3].sum():.2f}")
