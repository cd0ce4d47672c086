"""Golden digests of deep trees and of config 5, computed by the REFERENCE.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_deep_golden.py [--workers N]

Writes ``tests/golden/deep_vectors.jsonl``.  The GPU box never runs this
script; tests read only the committed JSONL.

Two kinds of record:

* ``deep``: ``hash_bytes`` of the reference itself (hasher.py:434-453, lanes
  engine) on strings whose trees have L = 6, 7 and 8 levels, all four
  variants (up to 2.8 GB per string: the reference's numpy intermediates
  need ~6x that in RAM, which this container has).
* ``huge``: config 5 -- one 16 GiB string, 16-byte variant -- which the
  reference cannot hash in one call here (~90 GB of intermediates).  It is
  computed by a chunked harness over the reference's OWN internals
  (SURVEY.md 8(c)): ``_encode_np``, ``_nh_words_np``, ``_combine_np`` and
  ``_nh_node_np`` (hasher.py:279-328) reduce each run of 8^c instances to
  its level-c subtree roots (the stack construction is front-aligned,
  tree.py:63-100), and the leftover / finalize / tail logic of
  ``_hash_words_np`` (hasher.py:366-412) is replayed over the ragged end and
  the roots.  The harness is first checked bit-exact against the reference's
  ``hash_bytes`` on strings up to 1 GiB (several chunk levels, ragged and
  exact ends, every variant); the script aborts if any check fails.

Inputs are ``fill:<seed_hex>:<word_offset>`` = the reference's splitmix fill
(cli.py:48-53); config 5 uses BASELINE's "PRNG seed 0" data stream and the
"seed 1" master (workloads.py: fold 1).
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import halftimehash as R  # noqa: E402
from halftimehash import hasher as RH  # noqa: E402
from halftimehash.cli import FILL_SEED  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "deep_vectors.jsonl")
CFG5_BYTES = 16 << 30
CFG5_MASTER = (1).to_bytes(8, "little") + bytes(24)  # workloads.MASTER (fold 1)
CFG5_DATA_SEED = 0  # workloads.DATA_SEED


def fill_bytes(n: int, seed: int, word_offset: int = 0) -> bytes:
    if n == 0:
        return b""
    return RH._stream_words_np(seed, word_offset, (n + 7) // 8).astype("<u8").tobytes()[:n]


def data_words(seed: int, n_bytes: int, start: int, count: int) -> np.ndarray:
    """Words [start, start+count) of the LE word view of fill_bytes(n_bytes,
    seed), the final partial word zero-padded (hasher.py:416-419)."""
    w = RH._stream_words_np(seed, start, count)
    n_words = (n_bytes + 7) // 8
    if count and n_bytes % 8 and start + count == n_words:
        w[-1] &= np.uint64((1 << (8 * (n_bytes % 8))) - 1)
    return w


# ------------------------------------------------------------ chunked harness
_G = {}


def _leaf_blocks(p, words, ent):
    """(n_inst*m,) words -> combined leaf blocks (n_inst, k, b): the first
    half of _hash_words_np (hasher.py:355-364) on one batch row."""
    d, w, b = p.instance_items, p.item_blocks, p.block_words
    n = words.size // p.instance_words
    inst = words.reshape(1, n, d, w, b)
    enc = RH._encode_np(inst, p)
    hashed = RH._nh_words_np(enc.swapaxes(-2, -1), ent.reshape(p.encoded_items, 1, w))
    return RH._combine_np(hashed, p)[0]


def _roots_task(rng):
    """Level-c roots (k, b) of chunks j0..j1 (each 8^c whole instances)."""
    j0, j1 = rng
    p, n_bytes, c, seed_words, data_seed, layout = (_G[x] for x in ("p", "n", "c", "S", "data", "layout"))
    m, k, f = p.instance_words, p.output_words, p.fanout
    per = f ** c
    ent = seed_words[layout.ehc_start:layout.ehc_start + layout.ehc_words]
    out = np.empty((j1 - j0, k, p.block_words), dtype=np.uint64)
    for j in range(j0, j1):
        comb = _leaf_blocks(p, data_words(data_seed, n_bytes, j * per * m, per * m), ent)
        for r in range(k):
            t0 = layout.tree_start + r * layout.tree_words_per_tree
            cur = comb[None, :, r, :]
            for lvl in range(c):  # complete groups only: no leftovers below the root
                groups = cur.reshape(1, cur.shape[1] // f, f, p.block_words)
                cur = RH._nh_node_np(groups, seed_words[t0 + lvl * (f - 1):t0 + (lvl + 1) * (f - 1)])
            out[j - j0, r] = cur[0, 0]
    return out


def chunked_hash(p, n_bytes: int, master: bytes, data_seed: int, c: int, workers: int) -> bytes:
    """The digest of fill_bytes(n_bytes, data_seed) under seed_for_input(master)."""
    layout = RH.seed_layout(p, n_bytes)
    seed = R.seed_for_input(master, p, n_bytes)
    S = seed.words_np(0, seed.capacity)
    m, k, f, b = p.instance_words, p.output_words, p.fanout, p.block_words
    n_words = (n_bytes + 7) // 8
    n_inst = n_words // m
    per = f ** c
    nfull = n_inst // per
    assert nfull >= 1, "string shorter than one chunk: use hash_bytes"
    _G.update(p=p, n=n_bytes, c=c, S=S, data=data_seed, layout=layout)
    step = max(1, min(64, nfull // (4 * workers) or 1))
    ranges = [(j, min(nfull, j + step)) for j in range(0, nfull, step)]
    if workers > 1:
        with mp.get_context("fork").Pool(workers) as pool:
            roots = np.concatenate(pool.map(_roots_task, ranges, chunksize=1))
    else:
        roots = np.concatenate([_roots_task(r) for r in ranges])
    rag = n_inst - nfull * per
    ent = S[layout.ehc_start:layout.ehc_start + layout.ehc_words]
    comb_rag = _leaf_blocks(p, data_words(data_seed, n_bytes, nfull * per * m, rag * m), ent) if rag else None
    tag = np.full((1, 1), n_bytes & ((1 << 64) - 1), dtype=np.uint64)
    out = np.zeros(k, dtype=np.uint64)
    for r in range(k):
        t0 = layout.tree_start + r * layout.tree_words_per_tree
        lvl_seeds = S[t0:t0 + layout.tree_words_per_tree]
        leftover_levels = []
        # levels < c: the leftovers all lie in the ragged end, whose groups are
        # aligned with the string's (nfull * 8^c is a multiple of every 8^l)
        cur = comb_rag[None, :, r, :] if rag else np.zeros((1, 0, b), dtype=np.uint64)
        for lvl in range(c):
            cut = cur.shape[1] - cur.shape[1] % f
            leftover_levels.append(cur[:, cut:, :])
            groups = cur[:, :cut, :].reshape(1, cut // f, f, b)
            cur = RH._nh_node_np(groups, lvl_seeds[lvl * (f - 1):(lvl + 1) * (f - 1)]) if cut else \
                np.zeros((1, 0, b), dtype=np.uint64)
        # levels >= c: the stack construction continued over the roots
        cur = roots[None, :, r, :]
        lvl = c
        while True:  # hasher.py:374-386
            cut = cur.shape[1] - cur.shape[1] % f
            leftover_levels.append(cur[:, cut:, :])
            if cut == 0:
                break
            groups = cur[:, :cut, :].reshape(1, cut // f, f, b)
            cur = RH._nh_node_np(groups, lvl_seeds[lvl * (f - 1):(lvl + 1) * (f - 1)])
            lvl += 1
        assert len(leftover_levels) == layout.levels
        parts = []
        for lo in leftover_levels:  # hasher.py:387-405
            if lo.shape[1] < f - 1:
                lo = np.concatenate([lo, np.zeros((1, f - 1 - lo.shape[1], b), dtype=np.uint64)], axis=1)
            parts.append(lo.reshape(1, (f - 1) * b))
        flat = np.concatenate(parts + [tag], axis=1)
        fs = layout.finalize_start + r * layout.finalize_words_per_tree
        out[r] = RH._nh_words_np(flat, S[fs:fs + layout.levels * (f - 1) * b + 1])[0]
    tail = data_words(data_seed, n_bytes, n_inst * m, n_words - n_inst * m)
    if tail.size:  # hasher.py:407-412
        rem = S[layout.remainder_start:layout.remainder_start + layout.remainder_words]
        with np.errstate(over="ignore"):
            for r in range(k):
                out[r] += RH._nh_words_np(tail[None, :], rem[r:r + tail.size])[0]
    return b"".join(int(x).to_bytes(8, "little") for x in out)


def reference_digest(p, n_bytes, master, data_seed) -> bytes:
    return R.hash_bytes(fill_bytes(n_bytes, data_seed), R.seed_for_input(master, p, n_bytes), p).bytes


def validate(workers: int) -> list:
    """The harness against hash_bytes (<= 1 GiB), several chunk levels."""
    checks = []
    cases = []
    for w in (16, 24, 32, 40):
        m8 = R.variant(w).instance_words * 8
        cases += [(w, (8 ** 3 * 5 + 8 ** 2 * 3 + 7) * m8 + 45, 2), (w, (8 ** 3 * 5 + 8 ** 2 * 3 + 7) * m8 + 45, 3),
                  (w, 8 ** 4 * 3 * m8, 3), (w, (8 ** 4 * 9 + 8 ** 3 * 7 + 1) * m8 + m8 - 3, 4),
                  (w, (8 ** 5 * 2 + 8 ** 4 + 5) * m8 + 1, 5)]
    cases.append((16, (8 ** 6 * 4 + 8 ** 5 * 7 + 8 ** 3 + 2) * 768 + 700, 5))  # ~1.0 GB, L = 7
    master = bytes(range(7, 39))
    for w, n, c in cases:
        p = R.variant(w)
        t0 = time.time()
        want = reference_digest(p, n, master, FILL_SEED)
        got = chunked_hash(p, n, master, FILL_SEED, c, workers)
        ok = got == want
        checks.append(dict(variant=w, length=n, chunk_level=c, ok=ok))
        print(f"harness v{w} n={n} c={c}: {'ok' if ok else 'MISMATCH'} ({time.time() - t0:.1f} s)", flush=True)
        if not ok:
            raise SystemExit(f"chunked harness disagrees with hash_bytes: v{w} n={n} c={c}")
    return checks


def deep_lengths(w: int):
    """One length per L = 6, 7, 8 (ragged digits on every level, a tail)."""
    m8 = R.variant(w).instance_words * 8
    return [(6, (8 ** 5 + 8 ** 4 * 3 + 8 ** 2 * 5 + 7) * m8 + 61),
            (7, (8 ** 6 + 8 ** 5 * 2 + 8 ** 3 + 3) * m8 + m8 - 1),
            (8, (8 ** 7 + 8 ** 4 + 1) * m8 + 13)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--skip-deep", action="store_true")
    args = ap.parse_args()
    t_all = time.time()
    checks = validate(args.workers)
    recs = []
    masters = [bytes(range(32)), b"\x5a" * 32]
    if not args.skip_deep:
        for i, w in enumerate((16, 24, 32, 40)):
            p = R.variant(w)
            for L, n in deep_lengths(w):
                master = masters[(i + L) % 2]
                t0 = time.time()
                d = reference_digest(p, n, master, FILL_SEED)
                assert RH.seed_layout(p, n).levels == L
                recs.append(dict(kind="deep", variant=w, levels=L, master=master.hex(), length=n,
                                 generator=f"fill:{FILL_SEED:016x}:0", digest=d.hex(), method="hash_bytes"))
                print(f"deep v{w} L={L} n={n}: {d.hex()} ({time.time() - t0:.1f} s)", flush=True)
    t0 = time.time()
    p16 = R.variant(16)
    d = chunked_hash(p16, CFG5_BYTES, CFG5_MASTER, CFG5_DATA_SEED, 5, args.workers)
    recs.append(dict(kind="huge", config="cfg5", variant=16, levels=RH.seed_layout(p16, CFG5_BYTES).levels,
                     master=CFG5_MASTER.hex(), length=CFG5_BYTES, generator=f"fill:{CFG5_DATA_SEED:016x}:0",
                     digest=d.hex(), method="chunked harness over the reference's internals (chunk level 5)",
                     harness_checks=checks))
    print(f"cfg5 16 GiB v16: {d.hex()} ({time.time() - t0:.1f} s)", flush=True)
    with open(OUT, "w") as fh:
        for r in recs:
            fh.write(json.dumps(r, sort_keys=True) + "\n")
    print(f"wrote {len(recs)} records to {OUT} in {time.time() - t_all:.0f} s")


if __name__ == "__main__":
    main()
