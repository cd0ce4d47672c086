"""Config 5's 8-GPU exchange emulated on one GPU (bench.measure_exchange_emulated)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2104_08865_b200 as hh  # noqa: E402

for ns in (2, 4, 8):
    print(json.dumps(dict(bench.measure_exchange_emulated(hh, torch, n_slices=ns), n_slices=ns)), flush=True)
