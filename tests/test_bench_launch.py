"""bench.py's launcher contract, on the CPU: --gpus N outside torchrun
spawns N ranks itself, and a WORLD_SIZE that disagrees with --gpus fails
loudly.  The reference arm is used (it needs no GPU: rank 0 times the CPU
path, the other ranks exit 0)."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None, timeout=600):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.pop("RANK", None)
    e.pop("LOCAL_RANK", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=e, timeout=timeout, cwd=ROOT)


def _line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out
    return json.loads(lines[0])


def test_bench_spawns_its_ranks():
    r = _run(["--gpus", "2", "--impl", "reference", "--workload", "cfg1", "--steps", "1", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    line = _line(r.stdout)
    assert line["n_gpus"] == 2 and line["impl"] == "reference"
    assert "launching 2 ranks" in r.stderr


def test_bench_rejects_world_size_mismatch():
    r = _run(["--gpus", "2", "--impl", "reference"], env={"WORLD_SIZE": "3", "RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=3" in r.stderr


def test_bench_roofline_helpers():
    # the bench line's secondary rooflines come from committed measurements
    sys.path.insert(0, ROOT)
    import bench

    imad = bench._imad_bound("cfg4", 6100.0)
    assert imad and imad["bound_gbs"] > 10 * 6100.0  # the multiply pipe never binds here
    rp = bench._read_peak(6100.0)
    assert rp and 0 < rp["frac"] < 1.2
    floor = bench._cfg1_floor()
    assert floor and 0 < floor["empty_launch_us"] < floor["us"]
    assert set(bench.MULT_PER_BYTE) >= {"cfg1", "cfg2", "cfg3", "cfg4", "cfg5"}
