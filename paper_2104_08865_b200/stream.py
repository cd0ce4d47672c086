"""Incremental hashing of one long string (absent from the reference, which
is one-shot: pkg/README.md:121).

The digest equals ``hash_bytes`` on the concatenated input.  The reference's
seed layout depends on the total length (tree and finalize regions shift
with the level count, hasher.py:130-153), so the total length is declared up
front, as with any length-keyed hash.  Because the stack construction groups
blocks front-aligned (tree.py:63-100), every complete run of 8^c instances
reduces to level-c roots independently of what follows: the stream hashes
each such slice on the GPU as soon as its bytes have arrived
(``hth_hash_slice``), keeps the roots and the partial finalize sums, and
finishes with the last slice (ragged end + tail) and ``hth_hash_merge``.
The last slice always contains the string's last job, so it is never hashed
early.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .hasher import Digest, SeedBuffer, _check_capacity
from .params import HashParams


class StreamHasher:
    """``h = StreamHasher(params, seed, total_length); h.update(b1); ...; h.digest()``.

    ``update`` accepts bytes-like objects, numpy uint8 arrays or uint8 torch
    tensors (host or CUDA).  Work is stream-ordered on the current CUDA stream
    of the device; the staging buffer holds one slice (~``slice_bytes``,
    rounded down to whole level-c subtrees).
    """

    def __init__(self, params: HashParams, seed: SeedBuffer, total_length: int, device=None,
                 slice_bytes: int = 64 << 20):
        import torch

        _check_capacity(seed, params, total_length)
        self.params, self.seed, self.n = params, seed, int(total_length)
        idx = torch.cuda.current_device() if device is None else torch.device(device).index or 0
        self.dev = torch.device("cuda", idx)
        self.ib = params.instance_words * 8
        self.n_inst = ((self.n + 7) // 8) // params.instance_words
        c = 3 if self.n_inst >= 512 else 2  # >= the engine's job level (hth_hash_slice requirement)
        while (8 ** (c + 1)) * self.ib <= slice_bytes:
            c += 1
        self.level, self.sub = c, 8 ** c
        self.keep = (self.n_inst >> (3 * c)) & ~7  # non-leftover level-c roots of the whole string
        self.slice_len = self.sub * self.ib
        size = self.slice_len + self.ib + 32 if self.n_inst >= self.sub else self.n + 32
        self.buf = torch.empty(((size + 15) // 16) * 16, dtype=torch.uint8, device=self.dev)
        self.fill = 0       # bytes staged for the current slice
        self.consumed = 0   # bytes of completed slices
        self.inst_done = 0  # first instance of the current slice
        self.frontiers, self.partials = [], []
        self.k = params.output_words
        ws = ctypes.c_uint64()
        _lib.check(_lib.lib().hth_workspace_size_slice(params.output_bytes, self.n, ctypes.byref(ws)))
        self.ws = torch.zeros(max(ws.value, 256), dtype=torch.uint8, device=self.dev)
        self._digest = None

    def _last(self) -> bool:
        return self.inst_done + self.sub >= self.n_inst

    def _hash_staged(self, a: int, b: int):
        import torch

        cnt = max(0, min(b >> (3 * self.level), self.keep) - (a >> (3 * self.level)))
        fr = torch.empty((max(cnt, 1), 8 * self.k), dtype=torch.int64, device=self.dev)
        part = torch.empty(self.k, dtype=torch.int64, device=self.dev)
        with torch.cuda.device(self.dev):
            _lib.check(_lib.lib().hth_hash_slice(
                self.params.output_bytes, self.buf.data_ptr(), self.n, a, b, self.level, self.seed.fold,
                self.seed.device_words(self.dev).data_ptr(), self.seed.capacity, fr.data_ptr(), part.data_ptr(),
                self.ws.data_ptr(), self.ws.numel(), torch.cuda.current_stream(self.dev).cuda_stream))
        if cnt:
            self.frontiers.append(fr[:cnt])
        self.partials.append(part)

    def update(self, data) -> "StreamHasher":
        import torch

        if self._digest is not None:
            raise ValueError("digest() already taken")
        if isinstance(data, torch.Tensor):
            t = data.reshape(-1).view(torch.uint8) if data.dtype != torch.uint8 else data.reshape(-1)
        else:
            arr = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else \
                np.ascontiguousarray(data).reshape(-1).view(np.uint8)
            t = torch.from_numpy(np.array(arr, copy=True))
        if self.consumed + self.fill + t.numel() > self.n:
            raise ValueError("more bytes than the declared total length")
        pos, total = 0, t.numel()
        while pos < total:
            need = (self.n - self.consumed) if self._last() else self.slice_len
            take = min(need - self.fill, total - pos)
            self.buf[self.fill:self.fill + take].copy_(t[pos:pos + take], non_blocking=True)
            self.fill += take
            pos += take
            if not self._last() and self.fill == self.slice_len:
                # a complete run of 8^c instances followed by more instances
                self._hash_staged(self.inst_done, self.inst_done + self.sub)
                self.inst_done += self.sub
                self.consumed += self.fill
                self.fill = 0
        return self

    def digest(self) -> Digest:
        import torch

        if self._digest is None:
            if self.consumed + self.fill != self.n:
                raise ValueError(f"received {self.consumed + self.fill} of {self.n} declared bytes")
            self._hash_staged(self.inst_done, self.n_inst)
            fr = torch.cat(self.frontiers) if self.frontiers else torch.zeros((1, 8 * self.k), dtype=torch.int64,
                                                                                device=self.dev)
            nf = sum(int(f.shape[0]) for f in self.frontiers)
            pa = torch.stack(self.partials).contiguous()
            out = torch.empty(self.k, dtype=torch.int64, device=self.dev)
            tmp = torch.empty(2 * (nf // 8 + 8) * 8 * self.k * 8, dtype=torch.uint8, device=self.dev)
            with torch.cuda.device(self.dev):
                _lib.check(_lib.lib().hth_hash_merge(
                    self.params.output_bytes, self.n, self.level, fr.data_ptr(), nf, pa.data_ptr(), pa.shape[0],
                    self.seed.fold, self.seed.device_words(self.dev).data_ptr(), self.seed.capacity, out.data_ptr(),
                    tmp.data_ptr(), tmp.numel(), torch.cuda.current_stream(self.dev).cuda_stream))
            self._digest = Digest(tuple(int(x) for x in out.cpu().numpy().view(np.uint64)))
        return self._digest
