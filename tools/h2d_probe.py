"""Host->device copy ceiling on this box (pinned memory): one big copy, and
chunked copies on 1-3 streams -- the bound of the e2e (host buffer) path."""
import time

import torch

N = 4 << 30
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(N, dtype=torch.uint8, device="cuda")


def run(chunk, nst):
    sts = [torch.cuda.Stream() for _ in range(nst)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, off in enumerate(range(0, N, chunk)):
        with torch.cuda.stream(sts[i % nst]):
            d[off:off + chunk].copy_(h[off:off + chunk], non_blocking=True)
    torch.cuda.synchronize()
    return N / (time.perf_counter() - t0) / 1e9


for chunk in (N, 256 << 20, 64 << 20, 16 << 20):
    for nst in (1, 2, 3):
        if chunk == N and nst > 1:
            continue
        run(chunk, nst)
        print(f"chunk {chunk >> 20:5d} MiB streams {nst}: {max(run(chunk, nst) for _ in range(3)):.1f} GB/s")
