"""hash_bytes latency per size, in a fresh process per host-path setting:
  python tools/lat_ab.py            # runs both HTH_HOST_MAPPED=1 and =0
Each run checks its digests against the C oracle and prints one JSON line."""
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIZES = (64, 1024, 4096, 16384, 65536, 1 << 20)


def child():
    import numpy as np

    import paper_2104_08865_b200 as hh
    from oracle import c as coracle
    from oracle import oracle_np as o

    out = {"mapped": os.environ.get("HTH_HOST_MAPPED", "1"), "us": {}}
    for w in (24,):
        p = hh.variant(w)
        for n in SIZES:
            data = o.fill_bytes(n, 5)
            seed = hh.seed_for_input(bytes(range(32)), p, n)
            d = hh.hash_bytes(data, seed, p)
            want = coracle.hash_one(w, np.frombuffer(data, dtype=np.uint8), seed.words_np(0, seed.capacity))
            assert np.array_equal(np.array(d.words, dtype=np.uint64), want), n
            ts = []
            for _ in range(200):
                t0 = time.perf_counter()
                hh.hash_bytes(data, seed, p)
                ts.append(time.perf_counter() - t0)
            out["us"][n] = round(statistics.median(ts) * 1e6, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "child":
        child()
    else:
        for m in ("1", "0", "1", "0"):
            subprocess.run([sys.executable, __file__, "child"], env=dict(os.environ, HTH_HOST_MAPPED=m), check=True)
