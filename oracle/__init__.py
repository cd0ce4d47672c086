"""HalftimeHash CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two independent restatements of the reference hash path
(/root/reference/pkg/src/halftimehash, halftimehash 0.1.0):

* ``oracle.oracle_np`` -- numpy, mirrors the reference's batched lane engine
  (hasher.py:331-413); small and medium sizes, and the ``--impl reference``
  CPU baseline (it runs at the reference's own numpy speed).
* ``oracle.c`` -- scalar C (halftime_oracle.c, built by oracle/Makefile into
  oracle/liboracle.so) for multi-GiB checks, e.g. config 5's 16 GiB string.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package, and
only as the checker / CPU baseline.  The product package never does.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import oracle_np  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build(force: bool = False) -> str:
    path = os.path.join(_HERE, "liboracle.so")
    src = os.path.join(_HERE, "halftime_oracle.c")
    if force or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return path


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        u64, vp, i32 = ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int
        L.hto_splitmix.argtypes = [u64, u64, u64, vp, i32]
        L.hto_splitmix.restype = None
        L.hto_seed_words_needed.argtypes = [i32, u64]
        L.hto_seed_words_needed.restype = u64
        L.hto_hash_one.argtypes = [i32, vp, u64, vp, u64, vp]
        L.hto_hash_fixed.argtypes = [i32, vp, u64, u64, u64, vp, u64, vp, i32]
        L.hto_hash_varlen.argtypes = [i32, vp, vp, u64, vp, u64, vp, i32]
        L.hto_hash_huge.argtypes = [i32, vp, u64, vp, u64, vp, i32]
        L.hto_slice.argtypes = [i32, vp, u64, u64, u64, i32, vp, u64, vp, vp]
        L.hto_merge.argtypes = [i32, u64, i32, vp, u64, vp, u64, vp, u64, vp]
        for f in (L.hto_hash_one, L.hto_hash_fixed, L.hto_hash_varlen, L.hto_hash_huge, L.hto_slice, L.hto_merge):
            f.restype = i32
        _LIB = L
    return _LIB


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _threads(t):
    return t if t else (os.cpu_count() or 1)


class c:
    """ctypes front end of the C restatement."""

    @staticmethod
    def splitmix(fold: int, start: int, count: int, threads: int = 0) -> np.ndarray:
        out = np.empty(count, dtype=np.uint64)
        lib().hto_splitmix(fold & ((1 << 64) - 1), start, count, _ptr(out), _threads(threads))
        return out

    @staticmethod
    def seed_words_needed(out_bytes: int, n_bytes: int) -> int:
        return int(lib().hto_seed_words_needed(out_bytes, n_bytes))

    @staticmethod
    def _k(out_bytes):
        return out_bytes // 8

    @staticmethod
    def _rc(rc):
        if rc == -2:
            raise ValueError("seed buffer too small")
        if rc:
            raise ValueError(f"oracle error {rc}")

    @classmethod
    def hash_one(cls, out_bytes: int, data, seeds: np.ndarray) -> np.ndarray:
        buf = np.frombuffer(bytes(data), dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        out = np.zeros(cls._k(out_bytes), dtype=np.uint64)
        cls._rc(lib().hto_hash_one(out_bytes, _ptr(buf), buf.nbytes, _ptr(seeds), seeds.size, _ptr(out)))
        return out

    @classmethod
    def hash_fixed(cls, out_bytes, data: np.ndarray, n_strings, stride, n_bytes, seeds, threads=0):
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        out = np.zeros((n_strings, cls._k(out_bytes)), dtype=np.uint64)
        cls._rc(lib().hto_hash_fixed(out_bytes, _ptr(data), n_strings, stride, n_bytes,
                                     _ptr(seeds), seeds.size, _ptr(out), _threads(threads)))
        return out

    @classmethod
    def hash_varlen(cls, out_bytes, data: np.ndarray, offsets: np.ndarray, seeds, threads=0):
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
        n = offsets.size - 1
        out = np.zeros((n, cls._k(out_bytes)), dtype=np.uint64)
        cls._rc(lib().hto_hash_varlen(out_bytes, _ptr(data), _ptr(offsets), n, _ptr(seeds),
                                      seeds.size, _ptr(out), _threads(threads)))
        return out

    @classmethod
    def hash_huge(cls, out_bytes, data: np.ndarray, seeds, threads=0):
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        out = np.zeros(cls._k(out_bytes), dtype=np.uint64)
        cls._rc(lib().hto_hash_huge(out_bytes, _ptr(data), data.nbytes, _ptr(seeds), seeds.size,
                                    _ptr(out), _threads(threads)))
        return out

    @classmethod
    def slice(cls, out_bytes, data: np.ndarray, n_bytes, inst_begin, inst_end, level, count, seeds):
        """Frontier (count, k*8) and partial (k,) of one slice; `data` is the whole string."""
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        k = cls._k(out_bytes)
        fr = np.zeros((max(count, 1), k * 8), dtype=np.uint64)
        part = np.zeros(k, dtype=np.uint64)
        cls._rc(lib().hto_slice(out_bytes, _ptr(data), n_bytes, inst_begin, inst_end, level, _ptr(seeds),
                                seeds.size, _ptr(fr), _ptr(part)))
        return fr[:count], part

    @classmethod
    def merge(cls, out_bytes, n_bytes, level, frontier: np.ndarray, partials: np.ndarray, seeds):
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64)
        fr = np.ascontiguousarray(frontier, dtype=np.uint64)
        pa = np.ascontiguousarray(partials, dtype=np.uint64)
        out = np.zeros(cls._k(out_bytes), dtype=np.uint64)
        cls._rc(lib().hto_merge(out_bytes, n_bytes, level, _ptr(fr), fr.shape[0], _ptr(pa), pa.shape[0],
                                _ptr(seeds), seeds.size, _ptr(out)))
        return out

