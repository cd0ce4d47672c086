"""Deep trees and config 5 against digests the REFERENCE computed
(tests/golden/deep_vectors.jsonl, made by tests/golden/make_deep_golden.py:
the reference's hash_bytes for L = 6, 7, 8 levels in every variant, and config
5's 16 GiB string through a chunked harness over the reference's own
internals).  Device-resident inputs through hash_fixed, and host inputs
through the host entry point (strings over 64 MiB take its sliced path)."""

import json
import os

import numpy as np
import pytest

from oracle import c as coracle

pytestmark = pytest.mark.gpu

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "deep_vectors.jsonl")


def _records(kind):
    with open(PATH) as fh:
        return [r for r in map(json.loads, fh) if r["kind"] == kind]


@pytest.fixture(scope="module")
def hh():
    import torch

    import paper_2104_08865_b200 as h

    assert torch.cuda.is_available()
    return h


def _fill(gen):
    kind, seed, off = gen.split(":")
    assert kind == "fill" and off == "0"
    return int(seed, 16)


def test_deep_records_present():
    deep = _records("deep")
    assert sorted({(r["variant"], r["levels"]) for r in deep}) == [(w, L) for w in (16, 24, 32, 40) for L in (6, 7, 8)]
    huge = _records("huge")
    assert len(huge) == 1 and huge[0]["length"] == 16 << 30 and huge[0]["variant"] == 16
    assert all(c["ok"] for c in huge[0]["harness_checks"])


@pytest.mark.parametrize("rec", _records("deep"), ids=lambda r: f"v{r['variant']}-L{r['levels']}")
def test_deep_device(hh, rec):
    import torch

    w, n = rec["variant"], rec["length"]
    p = hh.variant(w)
    buf = hh.fill_bytes(n, _fill(rec["generator"]))
    seed = hh.seed_for_input(bytes.fromhex(rec["master"]), p, n)
    got = hh.hash_fixed(buf, n, seed, p)[0].cpu().numpy().view(np.uint64)
    assert got.tobytes().hex() == rec["digest"]
    del buf
    torch.cuda.empty_cache()


@pytest.mark.parametrize("rec", [r for r in _records("deep") if r["levels"] == 7 or (r["levels"] == 8 and r["variant"] == 16)],
                         ids=lambda r: f"v{r['variant']}-L{r['levels']}")
def test_deep_host_sliced(hh, rec):
    w, n = rec["variant"], rec["length"]
    host = coracle.splitmix(_fill(rec["generator"]), 0, (n + 7) // 8).view(np.uint8)[:n]
    got = hh.hash_fixed_host(host, 1, n, bytes.fromhex(rec["master"]), hh.variant(w))[0]
    assert got.tobytes().hex() == rec["digest"]


@pytest.mark.slow
def test_config5_reference_digest(hh):
    # the 16 GiB string of config 5 on one GPU, against the reference's digest
    import torch

    rec = _records("huge")[0]
    n = rec["length"]
    p = hh.variant(16)
    buf = hh.fill_bytes(n, _fill(rec["generator"]))
    seed = hh.seed_for_input(bytes.fromhex(rec["master"]), p, n)
    got = hh.hash_fixed(buf, n, seed, p)[0].cpu().numpy().view(np.uint64)
    del buf
    torch.cuda.empty_cache()
    assert got.tobytes().hex() == rec["digest"]
