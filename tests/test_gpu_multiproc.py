"""Multi-process paths on the GPU: two ranks (sharing the box's one GPU when
that is all there is) run the split-string exchange through rank 0's memory
(CUDA-IPC peer pointers written by the slice kernels) and through all_gather,
and rank 0 checks the digests against the C oracle (tests/_split_worker.py)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", (2, 3, 8))
def test_split_string_exchange_two_processes(world):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(HERE, "_split_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count(" ok") == 3, r.stdout
