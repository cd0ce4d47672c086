"""BASELINE.json configs as seeded synthetic workloads (bench + tests tooling).

The reference measures on no dataset; every config is synthetic.  Choices
(SURVEY.md Appendix C):
  * data bytes: the reference's own splitmix stream (halftimehash/cli.py:48-53
    algorithm) keyed by the config's "PRNG seed 0": byte b of the packed
    input buffer is byte b of the stream mix(0 + (t+1) * gamma), t = b // 8.
    Generated in place on the GPU (hth_fill_splitmix) and regenerable on the
    CPU for any sampled string (oracle.oracle_np.fill_bytes with word_offset).
  * seed/entropy array "PRNG seed 1": master = (1).to_bytes(8) + 24 zero
    bytes, whose fold is 1, so S = SeedBuffer(master).words_np(0, cap).
  * config 2 lengths: numpy default_rng(2) log-uniform in [1, 65536], 16384 -
    128 of them, plus every length 0..127 once (16384 strings in total),
    shuffled; packed back to back (unaligned starts), u64 offsets.
"""

from __future__ import annotations

import numpy as np

DATA_SEED = 0
MASTER = (1).to_bytes(8, "little") + bytes(24)  # fold == 1

CONFIGS = {
    "cfg1": dict(desc="1024 x 4096 B, v24", variant=24, n_strings=1024, n_bytes=4096),
    "cfg2": dict(desc="16384 varlen log-uniform 1 B-64 KiB + 0..127 B, all variants", variant=None,
                 n_strings=16384),
    "cfg3": dict(desc="4,194,304 x 1024 B (4 GiB), v32", variant=32, n_strings=4 * 1024 * 1024, n_bytes=1024),
    "cfg4": dict(desc="8192 x 1 MiB (8 GiB), v40", variant=40, n_strings=8192, n_bytes=1 << 20),
    "cfg5": dict(desc="1 x 16 GiB, v16", variant=16, n_strings=1, n_bytes=16 << 30),
    # not a BASELINE config: a probe of the masked six-chunks-per-lane tail
    # kernel (strings of 81 16-byte chunks), the path whose register spills
    # were removed in round 2
    "probe_tail1296": dict(desc="probe: 3,000,000 x 1296 B (3.9 GB), v32, masked 6-chunk tail kernel", variant=32,
                           n_strings=3_000_000, n_bytes=1296),
}


def cfg2_lengths(n_strings: int = 16384, seed: int = 2) -> np.ndarray:
    rng = np.random.default_rng(seed)
    k = n_strings - 128
    ln = np.floor(np.exp(rng.uniform(0.0, np.log(65536.0), size=k))).astype(np.int64)
    ln = np.clip(ln, 1, 65536)
    lengths = np.concatenate([ln, np.arange(128, dtype=np.int64)])
    rng.shuffle(lengths)
    return lengths


def offsets_of(lengths: np.ndarray) -> np.ndarray:
    off = np.zeros(len(lengths) + 1, dtype=np.uint64)
    off[1:] = np.cumsum(lengths.astype(np.uint64))
    return off


def host_bytes(byte_offset: int, n: int, data_seed: int = DATA_SEED) -> bytes:
    """CPU regeneration of bytes [byte_offset, byte_offset+n) of a config buffer."""
    from oracle import oracle_np

    w0 = byte_offset // 8
    lead = byte_offset - 8 * w0
    raw = oracle_np.fill_bytes(lead + n, data_seed, w0)
    return raw[lead:lead + n]
