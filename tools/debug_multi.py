"""Debug helper: multi-job strings, repeated calls on one workspace."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2104_08865_b200 as hh  # noqa: E402
from paper_2104_08865_b200 import batch  # noqa: E402
from oracle import c as coracle  # noqa: E402
from oracle import oracle_np as o  # noqa: E402

for w, inst, B in [(16, 65, 1), (16, 65, 3), (40, 1092, 2), (16, 64 * 17 + 4, 1), (16, 129, 1)]:
    v = o.variant(w)
    n = inst * v.m * 8
    p = hh.variant(w)
    buf = hh.fill_bytes(B * n, 11)
    seed = hh.seed_for_input(bytes(range(32)), p, n)
    ws = torch.zeros(batch.workspace_fixed(p, B, n), dtype=torch.uint8, device="cuda")
    outs = []
    for rep in range(3):
        out = torch.full((B, p.output_words), 7, dtype=torch.int64, device="cuda")
        hh.hash_fixed(buf, n, seed, p, n_strings=B, stride=n, out=out, workspace=ws)
        torch.cuda.synchronize()
        outs.append(out.cpu().numpy().view(np.uint64).copy())
    host = np.frombuffer(o.fill_bytes(B * n, 11), dtype=np.uint8).copy()
    want = coracle.hash_fixed(w, host, B, n, n, seed.words_np(0, seed.capacity))
    wsn = ws.cpu().numpy()
    print(f"v{w} inst={inst} B={B} ws={ws.numel()} nonzero_ws={np.count_nonzero(wsn)}")
    for rep in range(3):
        print("  rep", rep, "ok" if np.array_equal(outs[rep], want) else f"BAD got {outs[rep][0]} want {want[0]}")
