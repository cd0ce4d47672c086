"""Batched device entry points -- the GPU form of the reference's batched
seam ``_hash_words_np(words (B, n_words), n_bytes, seed_region, params)``
(halftimehash/hasher.py:331-413), plus a packed variable-length batch.

Inputs are CUDA tensors already resident in HBM; outputs are (B, k) int64
CUDA tensors holding the raw little-endian u64 digest words
(``out.cpu().numpy().view(np.uint64)`` gives the reference's uint64 array).
Work is stream-ordered on the current torch CUDA stream.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .hasher import SeedBuffer, _check_capacity, _check_params, seed_words_needed
from .params import HashParams

__all__ = ["hash_fixed", "hash_varlen", "varlen_status", "hash_words", "hash_fixed_host", "fill_bytes",
           "workspace_fixed", "workspace_varlen", "hash_fixed_folds", "hash_words_many_seeds", "release_host",
           "fill_strings"]


def _stream(dev) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _u64(x) -> int:
    return int(x) & ((1 << 64) - 1)


def workspace_fixed(params: HashParams, n_strings: int, n_bytes: int) -> int:
    out = ctypes.c_uint64(0)
    _lib.check(_lib.lib().hth_workspace_size_fixed(params.output_bytes, n_strings, n_bytes, ctypes.byref(out)))
    return int(out.value)


def workspace_varlen(params: HashParams, n_strings: int, total_bytes: int) -> int:
    out = ctypes.c_uint64(0)
    _lib.check(_lib.lib().hth_workspace_size_varlen(params.output_bytes, n_strings, total_bytes, ctypes.byref(out)))
    return int(out.value)


def _seed_ptr(seed, dev):
    """(device words, capacity, fold) of a SeedBuffer (hasher.py:70-97)."""
    if isinstance(seed, SeedBuffer):
        return seed.device_words(dev), seed.capacity, seed.fold
    raise ValueError("seed must be a SeedBuffer (expand_seed / seed_for_input)")


class _Workspace:
    """Reusable engine workspace per (device, stream).

    The C-ABI requires a zero-filled workspace on first use and leaves it
    zero-filled after every call (its counters and accumulators reset
    themselves), so one zeroed allocation serves all later calls.
    """

    def __init__(self):
        self.buf = {}

    def get(self, dev, nbytes):
        key = (dev.index, _stream(dev))
        t = self.buf.get(key)
        if t is None or t.numel() < nbytes:
            t = torch.zeros(max(nbytes, 256), dtype=torch.uint8, device=dev)
            self.buf[key] = t
        return t

    def drop(self, dev):
        """Forget this stream's workspace after a failed call: the next call
        starts from a fresh zero-filled one (the engine also re-zeroes a
        workspace whose launch failed)."""
        self.buf.pop((dev.index, _stream(dev)), None)


def _call(cache, dev, rc_fn):
    """Run one C-ABI call; on any error drop the cached workspace, then raise."""
    try:
        _lib.check(rc_fn())
    except Exception:
        if cache is not None:
            cache.drop(dev)
        raise


_WS = _Workspace()       # hash_fixed: zero-filled, kept zero by the engine
_WS_VAR = _Workspace()   # hash_varlen: zero-filled; the engine clears it per batch layout


def hash_fixed(data: torch.Tensor, n_bytes: int, seed, params: HashParams, n_strings: int = None,
               stride: int = None, out: torch.Tensor = None, workspace: torch.Tensor = None) -> torch.Tensor:
    """Hash ``n_strings`` strings of ``n_bytes`` each.

    ``data``: CUDA uint8 tensor; either 2-D (B, >= n_bytes) rows, or flat with
    explicit ``n_strings``/``stride``.  Returns (B, k) int64 (raw u64 bits).
    """
    params = _check_params(params)
    if not isinstance(data, torch.Tensor) or not data.is_cuda:
        raise ValueError("data must be a CUDA tensor (use hash_fixed_host for host buffers)")
    if data.dtype != torch.uint8:
        data = data.view(torch.uint8) if data.is_contiguous() else data.contiguous().view(torch.uint8)
    dev = data.device
    if data.dim() == 2 and n_strings is None:
        n_strings = data.shape[0]
        stride = data.stride(0) if stride is None else stride
        if data.stride(1) != 1:
            raise ValueError("rows must be contiguous")
    else:
        if n_strings is None:
            n_strings = 1
        stride = n_bytes if stride is None else stride
    if n_strings and (n_strings - 1) * stride + n_bytes > data.numel():
        raise ValueError("data tensor too small for n_strings * stride")
    seed_t, cap, fold = _seed_ptr(seed, dev)
    _check_capacity(seed, params, n_bytes)
    k = params.output_words
    if out is None:
        out = torch.empty((n_strings, k), dtype=torch.int64, device=dev)
    wsz = workspace_fixed(params, n_strings, n_bytes)
    ws = workspace if workspace is not None else (_WS.get(dev, wsz) if wsz else None)
    with torch.cuda.device(dev):
        _call(_WS if workspace is None else None, dev, lambda: _lib.lib().hth_hash_fixed(
            params.output_bytes, data.data_ptr(), n_strings, stride, n_bytes, fold, seed_t.data_ptr(), cap,
            out.data_ptr(), ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0,
            _stream(dev)))
    return out


def hash_varlen(data: torch.Tensor, offsets, seed, params: HashParams, max_n_bytes: int = None,
                out: torch.Tensor = None, workspace: torch.Tensor = None, check: bool = None) -> torch.Tensor:
    """Hash strings ``data[offsets[s]:offsets[s+1]]`` (packed, any alignment).

    ``offsets``: n+1 byte offsets, numpy array or CUDA int64 tensor.  With
    a numpy array the offsets are validated and the exact longest length is
    used for the seed check on the host; with a device tensor pass
    ``max_n_bytes`` (default: the buffer size) and the device validates them.

    ``check``: read the device's verdict after the call (one stream
    synchronize) and raise like the reference -- ``SeedSizeError`` if a
    string is longer than ``max_n_bytes`` (hasher.py:209-214), ``ValueError``
    for decreasing offsets or offsets past the buffer.  Default: on whenever
    the host could not validate (device offsets or a caller-supplied
    ``max_n_bytes``).  Pass ``False`` inside CUDA-graph capture and call
    ``varlen_status(workspace)`` afterwards.
    """
    params = _check_params(params)
    if not isinstance(data, torch.Tensor) or not data.is_cuda:
        raise ValueError("data must be a CUDA tensor")
    if data.dtype != torch.uint8:
        data = data.view(torch.uint8) if data.is_contiguous() else data.contiguous().view(torch.uint8)
    if data.dim() != 1:
        data = data.reshape(-1)
    dev = data.device
    if check is None:
        check = isinstance(offsets, torch.Tensor) or max_n_bytes is not None
    if isinstance(offsets, torch.Tensor):
        d_off = offsets.to(device=dev, dtype=torch.int64)
        if max_n_bytes is None:
            max_n_bytes = data.numel()
    else:
        off = np.asarray(offsets, dtype=np.uint64)
        if off.ndim != 1 or off.size < 1 or np.any(off[1:] < off[:-1]):
            raise ValueError("offsets must be a non-decreasing 1-D array")
        if off[-1] > data.numel():
            raise ValueError("offsets exceed the data tensor")
        if max_n_bytes is None:
            max_n_bytes = int(np.max(off[1:] - off[:-1])) if off.size > 1 else 0
        d_off = torch.from_numpy(off.view(np.int64)).to(dev, non_blocking=False)
    n = d_off.numel() - 1
    seed_t, cap, fold = _seed_ptr(seed, dev)
    _check_capacity(seed, params, max_n_bytes)
    k = params.output_words
    if out is None:
        out = torch.empty((max(n, 0), k), dtype=torch.int64, device=dev)
    total = data.numel()
    wsz = workspace_varlen(params, max(n, 0), total)
    ws = workspace if workspace is not None else _WS_VAR.get(dev, wsz)
    if workspace is not None and workspace.numel() < wsz:
        raise ValueError(f"workspace too small: {workspace.numel()} < {wsz} bytes")
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().hth_hash_varlen(
            params.output_bytes, data.data_ptr(), d_off.data_ptr(), n, max_n_bytes, total, fold, seed_t.data_ptr(),
            cap, out.data_ptr(), ws.data_ptr(), ws.numel(), _stream(dev)))
        if check and n > 0:
            _lib.check(_lib.lib().hth_varlen_status(ws.data_ptr(), _stream(dev)))
    return out


def varlen_status(workspace: torch.Tensor) -> None:
    """Raise the error (if any) the device recorded for the last
    ``hash_varlen`` call on ``workspace`` (synchronizes its stream)."""
    dev = workspace.device
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().hth_varlen_status(workspace.data_ptr(), _stream(dev)))


def hash_fixed_folds(data: torch.Tensor, n_bytes: int, folds, params: HashParams, n_strings: int = None,
                     stride: int = None, out: torch.Tensor = None) -> torch.Tensor:
    """Many seeds: string s hashed under the seed stream of folds[s]
    (``_hash_words_np`` with a (B, 1) fold array, tests/test_hasher.py:254-310).
    ``stride=0`` hashes one input under every fold.  Returns (B, k) int64."""
    params = _check_params(params)
    if not isinstance(data, torch.Tensor) or not data.is_cuda:
        raise ValueError("data must be a CUDA tensor")
    dev = data.device
    f = folds if isinstance(folds, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(folds, dtype=np.uint64)).view(np.int64))
    f = f.to(device=dev, dtype=torch.int64).contiguous()
    n_strings = f.numel() if n_strings is None else n_strings
    if f.numel() < n_strings:
        raise ValueError("need one fold per string")
    stride = n_bytes if stride is None else stride
    if n_strings and (n_strings - 1) * stride + n_bytes > data.numel():
        raise ValueError("data tensor too small")
    k = params.output_words
    if out is None:
        out = torch.empty((n_strings, k), dtype=torch.int64, device=dev)
    wsz = workspace_fixed(params, n_strings, n_bytes)
    ws = _WS.get(dev, wsz)
    with torch.cuda.device(dev):
        _call(_WS, dev, lambda: _lib.lib().hth_hash_fixed_folds(
            params.output_bytes, data.data_ptr(), n_strings, stride, n_bytes, f.data_ptr(), out.data_ptr(),
            ws.data_ptr(), ws.numel(), _stream(dev)))
    return out


def hash_words_many_seeds(words, n_bytes: int, folds, params: HashParams, device=None) -> np.ndarray:
    """One (n_words,) input -- or a (B, n_words) batch -- under B seed folds.
    Returns (B, k) uint64 like the reference seam with a (B, 1) fold region."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    folds = np.asarray(folds, dtype=np.uint64).reshape(-1)
    t = torch.from_numpy(w.view(np.uint8).reshape(-1)).cuda(device)
    stride = 0 if w.ndim == 1 else w.shape[1] * 8
    out = hash_fixed_folds(t, n_bytes, folds, params, n_strings=folds.size, stride=stride)
    return out.cpu().numpy().view(np.uint64)


def hash_words(words, n_bytes: int, seed, params: HashParams, device=None) -> np.ndarray:
    """GPU form of ``_hash_words_np`` (hasher.py:331-413) for one shared seed.

    ``words``: (B, ceil(n_bytes/8)) uint64 array (numpy or CUDA tensor).
    Returns (B, k) uint64 numpy.
    """
    if isinstance(words, torch.Tensor):
        t = words if words.is_cuda else words.cuda(device)
        t = t.contiguous().view(torch.uint8).reshape(t.shape[0], -1)
    else:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        t = torch.from_numpy(w.view(np.uint8).reshape(w.shape[0], -1)).cuda(device)
    out = hash_fixed(t, n_bytes, seed, params)
    return out.cpu().numpy().view(np.uint64)


def hash_fixed_host(data, n_strings: int, n_bytes: int, master: bytes, params: HashParams, stride: int = None,
                    seed_capacity: int = None, device: int = 0) -> np.ndarray:
    """End-to-end batch from HOST memory (``hth_hash_fixed_host``): chunked
    H2D copies pipelined against hashing on three streams.  ``data`` may be a
    numpy array, bytes, or a (pinned) CPU torch tensor.  ``seed_capacity``
    plays SeedBuffer.capacity (``SeedSizeError`` below the layout); None
    sizes the seed stream exactly (seed_for_input).  Returns (B, k) uint64."""
    params = _check_params(params)
    stride = n_bytes if stride is None else stride
    if isinstance(data, torch.Tensor):
        ptr, nb = data.data_ptr(), data.numel() * data.element_size()
    else:
        arr = np.frombuffer(data, dtype=np.uint8) if isinstance(data, (bytes, bytearray)) else np.asarray(data)
        ptr, nb = arr.ctypes.data, arr.nbytes
    if n_strings and (n_strings - 1) * stride + n_bytes > nb:
        raise ValueError("host buffer too small")
    out = np.zeros((n_strings, params.output_words), dtype=np.uint64)
    if len(master) != 32:
        raise ValueError("master seed must be exactly 32 bytes")
    cap = _lib.SEED_AUTO if seed_capacity is None else int(seed_capacity)
    _lib.check(_lib.lib().hth_hash_fixed_host(params.output_bytes, ptr, n_strings, stride, n_bytes, bytes(master),
                                              cap, out.ctypes.data, device))
    return out


def fill_bytes(n_bytes: int, fill_seed: int = 0x243F6A8885A308D3, word_offset: int = 0, device=None,
               out: torch.Tensor = None) -> torch.Tensor:
    """Device form of the reference generator ``cli.fill_bytes`` (cli.py:48-53)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
    if out is None:
        out = torch.empty(((n_bytes + 15) // 16) * 16, dtype=torch.uint8, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.lib().hth_fill_splitmix(_u64(fill_seed), word_offset, n_bytes, out.data_ptr(), _stream(dev)))
    return out


def release_host() -> None:
    """Free the calling thread's host-path streams and buffers (``hth_host_release``)."""
    _lib.check(_lib.lib().hth_host_release())


def fill_strings(n_strings: int, n_bytes: int, first: int = 0, step: int = 1, fill_seed: int = 0x243F6A8885A308D3,
                 out: torch.Tensor = None, stride: int = None, device=None) -> torch.Tensor:
    """One launch: local string i = global string ``first + i * step`` of the
    packed ``fill_bytes`` stream of ``n_bytes``-strings (a round-robin or
    blocked shard of a batch; ``n_bytes % 8 == 0``)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else torch.device(device).index or 0)
    stride = n_bytes if stride is None else stride
    if out is None:
        out = torch.empty(max(n_strings * stride, 16), dtype=torch.uint8, device=dev)
    if n_strings and (n_strings - 1) * stride + n_bytes > out.numel():
        raise ValueError("output tensor too small")
    with torch.cuda.device(out.device):
        _lib.check(_lib.lib().hth_fill_splitmix_strings(_u64(fill_seed), n_strings, n_bytes, first, step,
                                                        out.data_ptr(), stride, _stream(out.device)))
    return out
