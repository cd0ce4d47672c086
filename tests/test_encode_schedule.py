"""The generated bit-plane parity schedules (csrc/gen_encode.py ->
encode_gen.cuh) must equal the reference's GF(16) encode (ehc.py:23-46,
gf16.py:17-32) on two packed instances.  CPU only: evaluates the schedule."""

import importlib.util
import os

import numpy as np
import pytest

from oracle import oracle_np as o

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
spec = importlib.util.spec_from_file_location(
    "gen_encode", os.path.join(ROOT, "paper_2104_08865_b200", "csrc", "gen_encode.py"))
gen = importlib.util.module_from_spec(spec)
spec.loader.exec_module(gen)


def planes(wa, wb):
    """u32 planes: plane b of word A in the low 16 bits, of word B in the high 16."""
    return [((int(wa) >> (16 * b)) & 0xFFFF) | (((int(wb) >> (16 * b)) & 0xFFFF) << 16) for b in range(4)]


@pytest.mark.parametrize("w", (24, 32, 40))
def test_schedule_matches_reference_encode(w):
    v = o.variant(w)
    d, P = gen.VARIANTS[w]
    assert [list(r) for r in v.parity] == P
    prog = gen.lop3_program(d, P)  # exactly what encode_gen.cuh computes
    rng = np.random.default_rng(w)
    for _ in range(200):
        xa = rng.integers(0, 1 << 64, size=d, dtype=np.uint64)
        xb = rng.integers(0, 1 << 64, size=d, dtype=np.uint64)
        vals = {}
        for i in range(d):
            for b, pl in enumerate(planes(xa[i], xb[i])):
                vals[4 * i + b] = pl
        y = [0] * (4 * len(P))
        for dest, terms in prog:
            acc = 0
            for t in terms:
                acc ^= vals[int(t[1:]) if isinstance(t, str) else t]
            if dest.startswith("t"):
                vals[int(dest[1:])] = acc
            else:
                y[int(dest[2:-1])] = acc
        for p, row in enumerate(v.parity):
            want_a = np.uint64(0)
            want_b = np.uint64(0)
            for i, c in enumerate(row):
                want_a ^= o.scale64(c, xa[i:i + 1])[0]
                want_b ^= o.scale64(c, xb[i:i + 1])[0]
            got_a = sum((y[4 * p + a] & 0xFFFF) << (16 * a) for a in range(4))
            got_b = sum((y[4 * p + a] >> 16) << (16 * a) for a in range(4))
            assert got_a == int(want_a) and got_b == int(want_b)


def test_generated_header_is_current():
    import io
    import contextlib

    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        gen.main()
    with open(os.path.join(ROOT, "paper_2104_08865_b200", "csrc", "encode_gen.cuh")) as fh:
        assert fh.read() == buf.getvalue()
