"""``python -m paper_2104_08865_b200`` -- the hash-path commands, on the GPU.

  hash     [--variant W] [--seed-hex HEX | --seed-file F] [PATH|- ...]
  bench    [--sizes 1K,256K,1M] [--reps N]
  vectors  (--emit PATH | --check PATH)

What is kept from the reference front end is its observable contract only
(halftimehash/cli.py, pkg/tests/test_cli.py): exit status 0 = ok, 1 = a
check failed, 2 = usage or I/O error; ``hash`` prints the lowercase hex
digest; ``bench`` prints the CSV ``size_bytes,variant,bytes_per_second,
bytes_per_cycle`` (cycle column empty); the vector file holds the lines
``variant,master_hex,length,splitmix:<fill seed>,digest_hex`` over the
reference's grid; sizes take binary K/M/G/T/P/E suffixes.  ``analyze`` and
``verify`` are off the hash path and not provided.

The implementation is organised around the device: the vector grid is one
splitmix fill in HBM whose prefixes are hashed in place (every grid input is
a prefix of the same stream), ``bench`` times the public host-bytes API
(``hash_bytes``: copy in, hash, digest out), and ``hash`` accepts several
inputs (one ``digest  path`` line each, like ``sha256sum``; a single input
prints the bare digest as the reference does).
"""

from __future__ import annotations

import argparse
import re
import statistics
import sys
import time
from dataclasses import dataclass
from typing import Callable

from . import hasher
from .params import VARIANTS, variant

FILL_SEED = 0x243F6A8885A308D3  # the reference's fill key
GRID_LENGTHS = (0, 1, 1336, 1344, 1024, (1 << 20) - 1, (1 << 20) + 1, 4 << 20)
GRID_MASTERS = (bytes(32), bytes(range(32)))
ZERO_MASTER = bytes(32)


class Mismatch(Exception):
    """A check found records that disagree (exit status 1)."""


# ------------------------------------------------------------ small parsers
_SIZE = re.compile(r"^\s*(\d+)\s*([kmgtpe]?)\s*$", re.IGNORECASE)
_POW = {"": 0, "k": 1, "m": 2, "g": 3, "t": 4, "p": 5, "e": 6}


def parse_size(text: str) -> int:
    """Byte count with an optional binary suffix: '1K' = 1024, '2m' = 2 MiB."""
    hit = _SIZE.match(text or "")
    if not hit:
        raise argparse.ArgumentTypeError(f"not a size: {text!r}")
    return int(hit.group(1)) << (10 * _POW[hit.group(2).lower()])


def read_master(seed_hex, seed_file) -> bytes:
    """The 32-byte master from --seed-hex or --seed-file (zeros if neither)."""
    if seed_hex is None and seed_file is None:
        return ZERO_MASTER
    if seed_hex is not None:
        raw, what = bytes.fromhex(seed_hex), "seed"
    else:
        with open(seed_file, "rb") as fh:
            raw, what = fh.read(33), "seed file"
    if len(raw) != 32:
        raise ValueError(f"{what} must hold exactly 32 bytes, got {len(raw)}")
    return raw


def read_input(path) -> bytes:
    if path in (None, "-"):
        return sys.stdin.buffer.read()
    with open(path, "rb") as fh:
        return fh.read()


# ------------------------------------------------------------ commands
@dataclass(frozen=True)
class Command:
    name: str
    help: str
    options: Callable[[argparse.ArgumentParser], None]
    run: Callable[[argparse.Namespace], int]


def _hash_options(p):
    p.add_argument("--variant", type=int, choices=sorted(VARIANTS), default=24)
    who = p.add_mutually_exclusive_group()
    who.add_argument("--seed-hex", help="master seed as 64 hex characters")
    who.add_argument("--seed-file", help="file holding the 32-byte master seed")
    p.add_argument("inputs", nargs="*", metavar="PATH", help="files to hash ('-' or none: stdin)")


def _hash_run(a) -> int:
    params = variant(a.variant)
    master = read_master(a.seed_hex, a.seed_file)
    paths = a.inputs or ["-"]
    for path in paths:
        data = read_input(path)
        d = hasher.hash_bytes(data, hasher.seed_for_input(master, params, len(data)), params)
        print(d.hex() if len(paths) == 1 else f"{d.hex()}  {path}")
    return 0


def _device_fill(n: int):
    """The reference's fill stream (cli.fill_bytes algorithm) generated in HBM."""
    from .batch import fill_bytes

    return fill_bytes(max(n, 1), FILL_SEED)


def grid_lines() -> list:
    """The vector grid, hashed on the device: all inputs are prefixes of one
    fill stream, so one fill serves every record (no host copies)."""
    from .batch import hash_fixed

    stream = _device_fill(max(GRID_LENGTHS))
    table = {}
    for width in sorted(VARIANTS):
        params = variant(width)
        for master in GRID_MASTERS:
            for n in GRID_LENGTHS:
                seed = hasher.seed_for_input(master, params, n)
                table[(width, master, n)] = hash_fixed(stream[:max(n, 1)], n, seed, params, n_strings=1)
    lines = []
    for (width, master, n), out in table.items():  # read back after all launches
        words = out.cpu().numpy().view("<u8")[0]
        lines.append(f"{width},{master.hex()},{n},splitmix:{FILL_SEED:016x},{words.tobytes().hex()}")
    return lines


def _vectors_options(p):
    mode = p.add_mutually_exclusive_group(required=True)
    mode.add_argument("--emit", metavar="PATH", help="write the grid")
    mode.add_argument("--check", metavar="PATH", help="compare a file with the grid")


def _vectors_run(a) -> int:
    lines = grid_lines()
    if a.emit:
        with open(a.emit, "w") as fh:
            fh.write("".join(x + "\n" for x in lines))
        return 0
    with open(a.check) as fh:
        got = [x.strip() for x in fh if x.strip()]
    want = set(lines)
    have = set(got)
    extra = [x for x in got if x not in want]
    absent = [x for x in lines if x not in have]
    for x in extra:
        print(f"mismatch: {x}")
    for x in absent:
        print(f"missing: {x}")
    if extra or absent:
        raise Mismatch(f"{len(extra) + len(absent)} vector records disagree with the grid")
    print(f"{len(got)} vector records verified")
    return 0


def _bench_options(p):
    p.add_argument("--sizes", default="1K,256K,1M", help="comma-separated sizes (K/M/G suffixes)")
    p.add_argument("--reps", type=int, default=5, help="timed calls per size and variant (median reported)")


def _rate(fn, size: int, reps: int) -> float:
    fn()  # the first call sets up streams, buffers and seeds
    samples = []
    for _ in range(max(reps, 1)):
        t0 = time.perf_counter()
        fn()
        dt = time.perf_counter() - t0
        samples.append(size / dt if dt > 0 else float("inf"))
    return statistics.median(samples)


def _bench_run(a) -> int:
    """Report-only: wall-clock throughput of the public one-shot API on host
    bytes (copy in, hash, digest out), per size and variant."""
    sizes = [parse_size(x) for x in a.sizes.split(",") if x.strip()]
    print("size_bytes,variant,bytes_per_second,bytes_per_cycle")
    for size in sizes:
        data = _device_fill(size)[:size].cpu().numpy().tobytes()
        for width in sorted(VARIANTS):
            params = variant(width)
            seed = hasher.seed_for_input(ZERO_MASTER, params, size)
            r = _rate(lambda: hasher.hash_bytes(data, seed, params), size, a.reps)
            print(f"{size},{width},{r:.0f},")
    return 0


COMMANDS = (
    Command("hash", "hash files or stdin", _hash_options, _hash_run),
    Command("bench", "report-only throughput of hash_bytes", _bench_options, _bench_run),
    Command("vectors", "emit or check the golden vector grid", _vectors_options, _vectors_run),
)


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2104_08865_b200",
                                 description="HalftimeHash on B200: the hash path of halftimehash 0.1.0.")
    sub = ap.add_subparsers(dest="command", required=True)
    for c in COMMANDS:
        c.options(sub.add_parser(c.name, help=c.help))
    return ap


def main(argv=None) -> int:
    a = build_parser().parse_args(argv)
    run = next(c.run for c in COMMANDS if c.name == a.command)
    try:
        return run(a)
    except Mismatch as e:
        print(str(e), file=sys.stderr)
        return 1
    except (ValueError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
