"""Drop-in mirror of the reference's public hash API
(halftimehash/hasher.py:36-176, 434-461), served by the CUDA engine.

``hash_bytes(data, seed, params, engine="cuda")`` and ``digest`` keep the
reference's names, argument meaning and errors:

* ``ValueError``    unsupported width (params.py:230-237), bad master
                    (hasher.py:48-50), unknown engine / counter with a
                    non-scalar engine (hasher.py:447-453)
* ``SeedSizeError`` capacity below ``seed_words_needed`` (hasher.py:209-214)
* ``IndexError``    seed word out of range (hasher.py:84-97)

Engines: ``"cuda"`` (default).  The reference's engine names ``"lanes"``
(its default) and ``"scalar"`` are accepted as aliases so unmodified
callers keep working: all three produce the reference's bit-identical
digests (hasher.py:217-269 vs :331-413), computed here by the GPU.  No CPU
engine exists; ``counter=`` (the scalar engine's multiplication accounting)
raises ``ValueError``.

``_hash_words_np(words, n_bytes, seed_region, params)`` keeps the
reference's batched seam signature (hasher.py:331-413) on the GPU engine.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._errors import SeedSizeError
from .params import HashParams, variant

GOLDEN_GAMMA = 0x9E3779B97F4A7C15
_MIX_1 = 0xBF58476D1CE4E5B9
_MIX_2 = 0x94D049BB133111EB
MASK64 = (1 << 64) - 1

__all__ = [
    "Digest", "SeedBuffer", "SeedLayout", "SeedSizeError", "digest", "expand_seed", "hash_bytes",
    "seed_for_input", "seed_layout", "seed_words_needed", "instance_count", "splitmix_mix", "ENGINES",
    "words_from_bytes", "hash_remainder",
]


def splitmix_mix(z: int) -> int:
    """splitmix64 finalizer (hasher.py:40-45)."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * _MIX_1) & MASK64
    z = ((z ^ (z >> 27)) * _MIX_2) & MASK64
    return z ^ (z >> 31)


def _master_fold(master: bytes) -> int:
    if not isinstance(master, (bytes, bytearray)) or len(master) != 32:
        raise ValueError("master seed must be exactly 32 bytes")
    a, b, c, d = struct.unpack("<4Q", bytes(master))
    return a ^ b ^ c ^ d


def _stream_words_np(fold, start: int, count: int) -> np.ndarray:
    idx = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.asarray(fold, dtype=np.uint64) + idx * np.uint64(GOLDEN_GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX_1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX_2)
    return z ^ (z >> np.uint64(31))


@dataclass(frozen=True)
class SeedBuffer:
    """Deterministic expansion of a 32-byte master seed (hasher.py:70-97).

    Host accessors (``word``, ``words``, ``words_np``) keep the reference's
    semantics; ``device_words`` materialises S[0..capacity) on a GPU with the
    ``hth_expand_seed`` kernel and caches it per device.
    """

    master: bytes
    capacity: int
    fold: int
    _dev: dict = field(default_factory=dict, compare=False, repr=False, hash=False)

    @classmethod
    def from_master(cls, master: bytes, capacity: int) -> "SeedBuffer":
        if capacity < 0:
            raise ValueError("capacity must be nonnegative")
        return cls(bytes(master), capacity, _master_fold(master))

    def word(self, index: int) -> int:
        if not 0 <= index < self.capacity:
            raise IndexError("seed word index out of range")
        return splitmix_mix((self.fold + (index + 1) * GOLDEN_GAMMA) & MASK64)

    def words(self, start: int, count: int) -> list:
        if start < 0 or start + count > self.capacity:
            raise IndexError("seed word range out of range")
        return [int(x) for x in _stream_words_np(self.fold, start, count)]

    def words_np(self, start: int, count: int) -> np.ndarray:
        if start < 0 or start + count > self.capacity:
            raise IndexError("seed word range out of range")
        return _stream_words_np(self.fold, start, count)

    def device_words(self, device=None):
        """S[0..capacity) as a CUDA int64 tensor (raw u64 bits), cached per device."""
        import torch

        dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
        t = self._dev.get(dev.index)
        if t is None:
            t = torch.empty(max(self.capacity, 1), dtype=torch.int64, device=dev)
            with torch.cuda.device(dev):
                st = torch.cuda.current_stream(dev).cuda_stream
                _lib.check(_lib.lib().hth_expand_seed(self.fold, 0, self.capacity, t.data_ptr(), st))
            self._dev[dev.index] = t
        return t


def expand_seed(master: bytes, needed: int) -> SeedBuffer:
    """Expand a 32-byte master into ``needed`` words (hasher.py:100-102)."""
    return SeedBuffer.from_master(master, needed)


@dataclass(frozen=True)
class SeedLayout:
    """Region partition of the expanded words for one length (hasher.py:105-123)."""

    levels: int
    ehc_start: int
    ehc_words: int
    tree_start: int
    tree_words_per_tree: int
    finalize_start: int
    finalize_words_per_tree: int
    remainder_start: int
    remainder_words: int
    total_words: int


def _check_params(params: HashParams) -> HashParams:
    if not isinstance(params, HashParams):
        raise ValueError("params must be a HashParams from variant()")
    return params


def instance_count(params: HashParams, n_bytes: int) -> int:
    return ((n_bytes + 7) // 8) // params.instance_words


def words_from_bytes(data: bytes) -> list:
    """Little-endian 64-bit words, the final partial word zero-padded
    (hasher.py:179-183): the word view every engine hashes."""
    data = bytes(data)
    if len(data) % 8:
        data += b"\x00" * (8 - len(data) % 8)
    return [int(x) for x in np.frombuffer(data, dtype="<u8")]


def hash_remainder(tail, remainder_words, k: int, half_bits: int = 32, counter=None) -> tuple:
    """The Toeplitz remainder (hasher.py:186-206) on the GPU: component i is
    NH of ``tail`` under ``remainder_words[i : i + len(tail)]``.

    As ``hash_bytes``, the GPU engine keeps no multiplication counter
    (``counter`` raises ``ValueError``) and works on 32-bit halves only.
    """
    if counter is not None:
        raise ValueError("multiplication counting is not available on the GPU engine")
    if half_bits != 32:
        raise ValueError("the GPU engine hashes 32-bit halves (half_bits=32)")
    n, k = len(tail), int(k)
    if len(remainder_words) < n + k - 1:
        raise ValueError("remainder key region too short")
    if k <= 0:
        return ()
    if n == 0:
        return (0,) * k
    import torch

    dev = torch.device("cuda", torch.cuda.current_device())
    as_dev = lambda v: torch.from_numpy(np.asarray(v, dtype=np.uint64).view(np.int64).copy()).to(dev)
    t, keys = as_dev(list(tail)), as_dev(list(remainder_words))
    out = torch.empty(k, dtype=torch.int64, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().hth_toeplitz_nh(t.data_ptr(), n, keys.data_ptr(), keys.numel(), k, out.data_ptr(),
                                              torch.cuda.current_stream(dev).cuda_stream))
    return tuple(int(x) for x in out.cpu().numpy().view(np.uint64))


def seed_layout(params: HashParams, n_bytes: int) -> SeedLayout:
    """Served by the C-ABI (hth_seed_layout) so host and device share one formula."""
    out = (ctypes.c_uint64 * 10)()
    _lib.check(_lib.lib().hth_seed_layout(_check_params(params).output_bytes, n_bytes, out))
    return SeedLayout(*[int(x) for x in out])


def seed_words_needed(params: HashParams, n_bytes: int) -> int:
    """Seed words needed to hash ``n_bytes`` (hasher.py:156-158)."""
    out = _lib.u64_out()
    _lib.check(_lib.lib().hth_seed_words_needed(_check_params(params).output_bytes, n_bytes, ctypes.byref(out)))
    return int(out.value)


def seed_for_input(master: bytes, params: HashParams, n_bytes: int) -> SeedBuffer:
    return expand_seed(master, seed_words_needed(params, n_bytes))


@dataclass(frozen=True)
class Digest:
    """k little-endian 64-bit words; ``output_bytes = 8 * k`` (hasher.py:165-176)."""

    words: tuple

    @property
    def bytes(self) -> bytes:
        return b"".join(w.to_bytes(8, "little") for w in self.words)

    def hex(self) -> str:
        return self.bytes.hex()


def _check_capacity(seed: SeedBuffer, params: HashParams, n_bytes: int) -> None:
    need = seed_words_needed(params, n_bytes)
    if seed.capacity < need:
        raise SeedSizeError(
            f"seed buffer holds {seed.capacity} words but this input needs {need}; "
            "expand with seed_words_needed()")


_OUT_T = {k: ctypes.c_uint64 * k for k in (2, 3, 4, 5)}  # digest words per variant

#: engine names accepted by hash_bytes: the GPU engine, and the reference's
#: two engine names as aliases of it (identical digests)
ENGINES = ("cuda", "lanes", "scalar")


def hash_bytes(data, seed: SeedBuffer, params: HashParams, engine: str = "cuda", counter=None,
               device=None) -> Digest:
    """One-shot hash of ``data`` under an expanded seed (hasher.py:434-453).

    ``data`` is a bytes-like object (host) or a CUDA uint8 tensor (device).
    Host data goes through ``hth_hash_host`` (H2D copy, on-device seed
    expansion, hash, D2H); device data through ``hth_hash_fixed``.
    """
    if engine not in ENGINES:
        raise ValueError(f"unknown engine {engine!r}; choose one of {', '.join(ENGINES)}")
    if counter is not None:
        # the reference counts multiplications only in its instrumented scalar
        # engine (hasher.py:447-449); the GPU engine has no such counter
        raise ValueError("multiplication counting is not available on the GPU engine")
    params = _check_params(params)
    k = params.output_words
    try:
        import torch
        is_tensor = isinstance(data, torch.Tensor)
    except ImportError:  # pragma: no cover
        is_tensor = False
    if is_tensor:
        from .batch import hash_fixed

        n = data.numel()
        _check_capacity(seed, params, n)
        out = hash_fixed(data.reshape(1, n), n, seed, params)
        return Digest(tuple(int(x) for x in out.cpu().numpy().view(np.uint64)[0]))
    buf = data if type(data) is bytes else bytes(data)
    out = _OUT_T[k]()
    dev = 0 if device is None else int(device)
    # the C-ABI checks the seed capacity itself (HTH_ESEEDSIZE -> SeedSizeError,
    # hasher.py:209-214), so the host path is a single foreign call
    rc = _lib.lib().hth_hash_host(params.output_bytes, buf, len(buf), seed.master, seed.capacity, out, dev)
    if rc:
        _lib.check(rc)
    return Digest(tuple(out))


def digest(data, master: bytes = b"\x00" * 32, output_bytes: int = 24) -> Digest:
    """Convenience one-shot (hasher.py:456-461)."""
    params = variant(output_bytes)
    return hash_bytes(data, seed_for_input(master, params, len(data)), params)


# ------------------------------------------------------------ batched seam
_MIX_1_INV = pow(_MIX_1, -1, 1 << 64)
_MIX_2_INV = pow(_MIX_2, -1, 1 << 64)


def _unshift_xor(y: np.ndarray, s: int) -> np.ndarray:
    """Inverse of x -> x ^ (x >> s) on uint64."""
    x = y.copy()
    t = s
    while t < 64:
        x ^= y >> np.uint64(t)
        t += s
    return x


def _unmix(z: np.ndarray) -> np.ndarray:
    """Inverse of the splitmix64 finalizer (a bijection of u64)."""
    with np.errstate(over="ignore"):
        z = _unshift_xor(z, 31) * np.uint64(_MIX_2_INV)
        z = _unshift_xor(z, 27) * np.uint64(_MIX_1_INV)
    return _unshift_xor(z, 30)


def _region_folds(seed_region, total: int):
    """Recover the seed stream(s) behind a ``seed_region(start, count)``.

    The engine computes seed words from a fold on the device
    (S[i] = mix(fold + (i+1) gamma), hasher.py:55-67), so a region is
    accepted when it is such a stream: a ``SeedBuffer.words_np`` (ours or
    the reference's: ``__self__`` with ``master``/``capacity``) or any
    callable returning ``_stream_words_np(folds, ...)`` with one fold or a
    (B, 1) array of folds (tests/test_hasher.py:254-310).  The folds are read
    off word 0 through the inverse finalizer and verified on the first and
    last words the layout uses.  Returns (folds (B,) or (1,), capacity or
    None).  ValueError for any other region; IndexError propagates from a
    region too small for the layout (SeedBuffer.words_np, hasher.py:94-97).
    """
    owner = getattr(seed_region, "__self__", None)
    if owner is not None and hasattr(owner, "master") and hasattr(owner, "capacity"):
        owner.words_np(max(total - 1, 0), 1)  # IndexError if the capacity is short
        return np.array([_master_fold(bytes(owner.master))], dtype=np.uint64), int(owner.capacity)
    head = np.asarray(seed_region(0, 1), dtype=np.uint64)
    if head.ndim == 1 and head.size == 1:
        head = head.reshape(1, 1)
    if head.ndim == 2 and head.shape[1] == 1:
        with np.errstate(over="ignore"):
            folds = _unmix(head[:, 0]) - np.uint64(GOLDEN_GAMMA)
    else:
        raise ValueError("seed_region(start, count) must return (count,) or (B, count) words")
    for start in {0, max(total - 2, 0)}:
        got = np.asarray(seed_region(start, 2 if total >= 2 else 1), dtype=np.uint64)
        want = _stream_words_np(folds[:, None], start, got.shape[-1])
        if not np.array_equal(got.reshape(-1, got.shape[-1]), want if got.ndim == 2 else want[:1]):
            raise ValueError("seed_region is not a splitmix seed stream (SeedBuffer.words_np or "
                             "_stream_words_np of master folds); the GPU engine cannot serve it")
    return folds, None


def _hash_words_np(words, n_bytes: int, seed_region, params: HashParams) -> np.ndarray:
    """The reference's batched seam (hasher.py:331-413) on the GPU engine.

    ``words``: (B, n_words) uint64 (a broadcast view of one row is hashed
    from one device copy).  ``seed_region(start, count)``: see
    ``_region_folds``.  Returns (B, k) uint64, row for row equal to the
    reference's ``_hash_words_np``.
    """
    params = _check_params(params)
    w = np.asarray(words)
    if w.ndim != 2:
        raise ValueError("words must be a (B, n_words) array")
    if w.dtype != np.uint64:
        w = w.astype(np.uint64)
    B = w.shape[0]
    nw = (n_bytes + 7) // 8
    if w.shape[1] < nw:
        raise ValueError(f"words hold {w.shape[1]} words but n_bytes={n_bytes} needs {nw}")
    total = seed_words_needed(params, n_bytes)
    folds, cap = _region_folds(seed_region, total)
    if B == 0:
        return np.zeros((0, params.output_words), dtype=np.uint64)
    import torch

    from .batch import hash_fixed, hash_fixed_folds

    one_row = B == 1 or w.strides[0] == 0
    rows = np.array(w[:1, :nw] if one_row else w[:, :nw], dtype=np.uint64, order="C")  # own, writable copy
    dev = torch.device("cuda", torch.cuda.current_device())
    t = torch.from_numpy(rows.view(np.uint8).reshape(-1)).to(dev)
    if folds.size == 1:
        seed = SeedBuffer(b"", cap if cap is not None else total, int(folds[0]))
        if one_row and B > 1:  # the same row under one seed: hash once
            out = hash_fixed(t, n_bytes, seed, params, n_strings=1).cpu().numpy().view(np.uint64)
            return np.repeat(out, B, axis=0)
        out = hash_fixed(t, n_bytes, seed, params, n_strings=B, stride=nw * 8)
    else:
        if folds.size != B:
            raise ValueError(f"seed_region gives {folds.size} seed rows for a batch of {B}")
        out = hash_fixed_folds(t, n_bytes, folds, params, n_strings=B, stride=0 if one_row else nw * 8)
    return out.cpu().numpy().view(np.uint64).copy()
