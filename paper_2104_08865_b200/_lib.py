"""ctypes binding of libhalftime_b200.so (C-ABI: include/halftime_b200.h).

The product path has no CPU fallback: if the shared library is missing or
CUDA is unavailable, calls raise instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes
import os
import threading

from ._errors import SeedSizeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HTH_LIB") or os.path.join(_HERE, "libhalftime_b200.so")

HTH_OK, HTH_EINVAL, HTH_ESEEDSIZE, HTH_ERANGE, HTH_ECUDA, HTH_ENOMEM = 0, -1, -2, -3, -4, -5

#: every entry point declared in include/halftime_b200.h
EXPORTS = (
    "hth_last_error", "hth_version", "hth_variant_geometry", "hth_seed_words_needed",
    "hth_seed_layout", "hth_master_fold", "hth_expand_seed", "hth_fill_splitmix",
    "hth_workspace_size_fixed", "hth_hash_fixed", "hth_workspace_size_varlen",
    "hth_hash_varlen", "hth_varlen_status", "hth_hash_host", "hth_hash_fixed_host",
    "hth_slice_plan", "hth_workspace_size_slice", "hth_hash_slice", "hth_hash_merge", "hth_hash_fixed_folds",
    "hth_ipc_get_handle", "hth_ipc_open_handle", "hth_ipc_close_handle", "hth_host_release",
    "hth_workspace_reset", "hth_hash_slice_ex", "hth_hash_merge_ex", "hth_signal", "hth_wait_flag",
    "hth_fill_splitmix_strings", "hth_toeplitz_nh",
)

HTH_SLICE_ACCUMULATE = 1

#: seed_capacity sentinel of the host entry points (HTH_SEED_AUTO)
SEED_AUTO = (1 << 64) - 1

_lock = threading.Lock()
_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the CUDA engine has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        u64, i32, vp = ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
        pu64 = ctypes.POINTER(ctypes.c_uint64)
        pi32 = ctypes.POINTER(ctypes.c_int)
        L.hth_last_error.restype = ctypes.c_char_p
        L.hth_last_error.argtypes = []
        L.hth_version.restype = i32
        sigs = {
            "hth_variant_geometry": [i32, pi32, pi32, pi32, pi32, pi32],
            "hth_seed_words_needed": [i32, u64, pu64],
            "hth_seed_layout": [i32, u64, pu64],
            "hth_master_fold": [ctypes.c_char_p, pu64],
            "hth_expand_seed": [u64, u64, u64, vp, vp],
            "hth_fill_splitmix": [u64, u64, u64, vp, vp],
            "hth_workspace_size_fixed": [i32, u64, u64, pu64],
            "hth_hash_fixed": [i32, vp, u64, u64, u64, u64, vp, u64, vp, vp, u64, vp],
            "hth_workspace_size_varlen": [i32, u64, u64, pu64],
            "hth_hash_varlen": [i32, vp, vp, u64, u64, u64, u64, vp, u64, vp, vp, u64, vp],
            "hth_varlen_status": [vp, vp],
            "hth_hash_host": [i32, vp, u64, ctypes.c_char_p, u64, vp, i32],
            "hth_hash_fixed_host": [i32, vp, u64, u64, u64, ctypes.c_char_p, u64, vp, i32],
            "hth_slice_plan": [i32, u64, u64, vp, pi32, vp],
            "hth_hash_fixed_folds": [i32, vp, u64, u64, u64, vp, vp, vp, u64, vp],
            "hth_workspace_size_slice": [i32, u64, pu64],
            "hth_hash_slice": [i32, vp, u64, u64, u64, i32, u64, vp, u64, vp, vp, vp, u64, vp],
            "hth_hash_merge": [i32, u64, i32, vp, u64, vp, u64, u64, vp, u64, vp, vp, u64, vp],
            "hth_ipc_get_handle": [vp, vp, pu64],
            "hth_ipc_open_handle": [vp, ctypes.POINTER(ctypes.c_void_p)],
            "hth_ipc_close_handle": [vp],
            "hth_host_release": [],
            "hth_workspace_reset": [vp, u64, vp],
            "hth_hash_slice_ex": [i32, vp, u64, u64, u64, i32, u64, vp, u64, vp, vp, vp, u64, i32, vp, u64, vp],
            "hth_hash_merge_ex": [i32, u64, i32, vp, u64, vp, u64, vp, u64, vp, vp, u64, vp, u64, vp, vp, u64, vp],
            "hth_signal": [vp, u64, vp],
            "hth_wait_flag": [vp, u64, u64, vp, vp],
            "hth_fill_splitmix_strings": [u64, u64, u64, u64, u64, vp, u64, vp],
            "hth_toeplitz_nh": [vp, u64, vp, u64, i32, vp, vp],
        }
        for name, args in sigs.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = i32
        _lib = L
        return L


def check(rc: int) -> None:
    if rc == HTH_OK:
        return
    msg = lib().hth_last_error().decode(errors="replace")
    if rc == HTH_ESEEDSIZE:
        raise SeedSizeError(msg)
    if rc == HTH_EINVAL:
        raise ValueError(msg)
    if rc == HTH_ERANGE:
        raise IndexError(msg)
    if rc == HTH_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"halftime_b200 CUDA error: {msg}")


def u64_out() -> ctypes.c_uint64:
    return ctypes.c_uint64(0)
