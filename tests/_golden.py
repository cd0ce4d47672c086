"""Load tests/golden/vectors.jsonl (made by tests/golden/make_golden.py from
the reference itself) and regenerate each record's input bytes without the
reference: ``fill`` = splitmix stream (oracle.oracle_np.splitmix_words, the
algorithm of halftimehash/hasher.py:61-67), ``rng`` = numpy default_rng."""

import json
import os

import numpy as np

from oracle import oracle_np

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "vectors.jsonl")

# The reference's own frozen golden digests (pkg/tests/test_hasher.py:30-53).
GOLDEN_EMPTY = {
    16: "b2ad1af365fccb72a0fa4d4600620c32",
    24: "f76f757856e9c252a8a1ce42dc0e2a5df09d621286a62a2d",
    32: "e8012c5533c9bec29c82cf1a7d771a4cc785d467494ed31c565c80f59ea86106",
    40: "4546303a3bed160a8640a6e8d48def023082a183442027049c8d66f38ca7bb00984146daa6cfb40c",
}
GOLDEN_ABC = {
    16: "d5493fea616e9bede05a920090c10e58",
    24: "cb9cfe00b1b1efbee41c5f999fe187bb47660fa1a13b8e60",
    32: "9c043287f44c9b7e98f8481632d319d89abe9155f01c0048dc616e58bf51dc06",
    40: "84ff722ce77a18502b1bdc5c71d23b63a7b660e0db41458b545b26dab5fb3e25ac1488cbc433f678",
}
GOLDEN_FILL_1344 = {
    16: "570153ce3db39cb2aa839e9818a00c3f",
    24: "31f937b85598a3a218c5f8ce6dba25517893116de61c37b1",
    32: "c366c94207afed3320f2afa8ceebb3eb29fd2b58be7f763edb834aeda52d2b54",
    40: "0c247b89ddf25b1f364088b20d4d80cb0c113c926db4e9d77bbd43137cfe5c2aabf077980f8c2875",
}
GOLDEN_FILL_100000 = {
    16: "4d19ef44b82f64cd071c9b93dafe7e3d",
    24: "005665bd13f50134a248676baed78e5951e0d8eef7d77dab",
    32: "5059cb578236e4ad9ffd69dd74e21e9f513ceaf5a1de14badc9cf29e33815736",
    40: "4ecc10841f5feccde5658fa5ce348a8c8d478d2f98e66a493ba330fac48de76d68ae034d010883ec",
}
# CLI golden (pkg/tests/test_cli.py:8): 24-byte digest of empty stdin, zero master
GOLDEN_EMPTY_24 = GOLDEN_EMPTY[24]
ZERO_MASTER = b"\0" * 32
RANGE_MASTER = bytes(range(32))


def records(kind=None):
    with open(PATH) as fh:
        recs = [json.loads(line) for line in fh if line.strip()]
    return [r for r in recs if kind is None or r["kind"] == kind]


def gen_bytes(gen: str, n: int) -> bytes:
    kind, *rest = gen.split(":")
    if kind == "fill":
        return oracle_np.fill_bytes(n, int(rest[0], 16), int(rest[1]))
    if kind == "rng":
        return np.random.default_rng(int(rest[0])).bytes(n)
    raise ValueError(gen)


def classic_cases():
    """(width, master, data, hex) for the reference's four golden tables."""
    out = []
    for w in (16, 24, 32, 40):
        out.append((w, ZERO_MASTER, b"", GOLDEN_EMPTY[w]))
        out.append((w, ZERO_MASTER, b"abc", GOLDEN_ABC[w]))
        out.append((w, RANGE_MASTER, oracle_np.fill_bytes(1344), GOLDEN_FILL_1344[w]))
        out.append((w, RANGE_MASTER, oracle_np.fill_bytes(100000), GOLDEN_FILL_100000[w]))
    return out
