"""Command line served by the CUDA engine: ``hash``, ``bench`` and ``vectors``.

Mirrors the reference's front end for its hash-path commands
(halftimehash/cli.py:78-84 ``hash``, 169-186 ``bench``, 189-222 ``vectors``);
analyze/verify are out of scope.  Exit codes follow cli.py:263-273: 0 ok,
1 check failure, 2 usage/IO.

  python -m paper_2104_08865_b200 hash [--variant 24] [--seed-hex HEX | --seed-file F] [FILE|-]
  python -m paper_2104_08865_b200 bench [--sizes 1K,256K,1M] [--reps 5]
  python -m paper_2104_08865_b200 vectors (--emit PATH | --check PATH)
"""

from __future__ import annotations

import argparse
import statistics
import sys
import time

import numpy as np

from . import hasher
from .params import VARIANTS, variant

#: the reference's fill key and vector grid (cli.py:22-26)
FILL_SEED = 0x243F6A8885A308D3
VECTOR_LENGTHS = (0, 1, 167 * 8, 168 * 8, 1024, 2 ** 20 - 1, 2 ** 20 + 1, 4 * 2 ** 20)
VECTOR_MASTERS = (b"\x00" * 32, bytes(range(32)))


class CheckFailure(Exception):
    pass


def _master(args) -> bytes:
    if args.seed_hex is not None:
        raw = bytes.fromhex(args.seed_hex)
        if len(raw) != 32:
            raise ValueError("seed must be 32 bytes (64 hex chars)")
        return raw
    if args.seed_file is not None:
        with open(args.seed_file, "rb") as fh:
            raw = fh.read()
        if len(raw) != 32:
            raise ValueError("seed file must hold exactly 32 bytes")
        return raw
    return b"\x00" * 32


def cmd_hash(args) -> int:
    params = variant(args.variant)
    master = _master(args)
    if args.input is None or args.input == "-":
        data = sys.stdin.buffer.read()
    else:
        with open(args.input, "rb") as fh:
            data = fh.read()
    seed = hasher.seed_for_input(master, params, len(data))
    print(hasher.hash_bytes(data, seed, params).hex())
    return 0


def _fill(n: int) -> bytes:
    """cli.fill_bytes on the GPU (hth_fill_splitmix), copied back."""
    if n == 0:
        return b""
    from .batch import fill_bytes

    return fill_bytes(n, FILL_SEED).cpu().numpy()[:n].tobytes()


_SIZE_SUFFIXES = {"K": 1, "M": 2, "G": 3, "T": 4, "P": 5, "E": 6}  # cli.py:20


def parse_size(text: str) -> int:
    """'1K' -> 1024 (cli.py:33-45)."""
    text = text.strip()
    if not text:
        raise argparse.ArgumentTypeError("empty size")
    mult = 1
    if text[-1].upper() in _SIZE_SUFFIXES:
        mult = 1024 ** _SIZE_SUFFIXES[text[-1].upper()]
        text = text[:-1]
    try:
        value = int(text)
    except ValueError:
        raise argparse.ArgumentTypeError(f"bad size {text!r}") from None
    return value * mult


def cmd_bench(args) -> int:
    """Report-only throughput of ``hash_bytes`` per size and variant, in the
    reference's CSV (cli.py:169-186): median of ``reps`` timed calls after one
    warm-up call, wall clock around the public one-shot API (host bytes in,
    Digest out).  The cycle column stays empty, as in the reference."""
    sizes = [parse_size(s) for s in args.sizes.split(",")]
    print("size_bytes,variant,bytes_per_second,bytes_per_cycle")
    for size in sizes:
        data = _fill(size)
        for width in sorted(VARIANTS):
            params = variant(width)
            seed = hasher.seed_for_input(b"\x00" * 32, params, size)
            hasher.hash_bytes(data, seed, params)  # warm-up
            rates = []
            for _ in range(args.reps):
                t0 = time.perf_counter()
                hasher.hash_bytes(data, seed, params)
                dt = time.perf_counter() - t0
                rates.append(size / dt if dt > 0 else float("inf"))
            print(f"{size},{width},{statistics.median(rates):.0f},")
    return 0


def vector_records():
    datas = {n: _fill(n) for n in VECTOR_LENGTHS}
    for width in sorted(VARIANTS):
        params = variant(width)
        for master in VECTOR_MASTERS:
            for n in VECTOR_LENGTHS:
                d = hasher.hash_bytes(datas[n], hasher.seed_for_input(master, params, n), params)
                yield f"{width},{master.hex()},{n},splitmix:{FILL_SEED:016x},{d.hex()}"


def cmd_vectors(args) -> int:
    if args.emit:
        with open(args.emit, "w") as fh:
            for line in vector_records():
                fh.write(line + "\n")
        return 0
    with open(args.check) as fh:
        recorded = [line.strip() for line in fh if line.strip()]
    expected = list(vector_records())
    bad = [line for line in recorded if line not in set(expected)]
    missing = [line for line in expected if line not in set(recorded)]
    if bad or missing:
        for line in bad:
            print(f"mismatch: {line}")
        for line in missing:
            print(f"missing:  {line}")
        raise CheckFailure(f"{len(bad) + len(missing)} vector records disagree")
    print(f"{len(recorded)} vector records verified")
    return 0


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="python -m paper_2104_08865_b200",
                                 description="HalftimeHash on B200 (hash path of halftimehash 0.1.0).")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("hash", help="hash a file or stdin")
    p.add_argument("--variant", type=int, choices=sorted(VARIANTS), default=24)
    p.add_argument("--seed-hex")
    p.add_argument("--seed-file")
    p.add_argument("input", nargs="?")
    p.set_defaults(func=cmd_hash)
    p = sub.add_parser("bench", help="report-only throughput benchmark")
    p.add_argument("--sizes", default="1K,256K,1M")
    p.add_argument("--reps", type=int, default=5)
    p.set_defaults(func=cmd_bench)
    p = sub.add_parser("vectors", help="emit or check the golden vector file")
    g = p.add_mutually_exclusive_group(required=True)
    g.add_argument("--emit", metavar="PATH")
    g.add_argument("--check", metavar="PATH")
    p.set_defaults(func=cmd_vectors)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except CheckFailure as exc:
        print(str(exc), file=sys.stderr)
        return 1
    except (ValueError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
