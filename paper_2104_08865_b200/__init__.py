"""paper_2104_08865_b200 -- B200-native HalftimeHash engine.

A drop-in for the hash path of the reference package ``halftimehash`` 0.1.0
(arXiv 2104.08865): same public names as ``halftimehash/__init__.py:9-37``,
with ``hash_bytes(..., engine="cuda")`` and the batched device entry points
``hash_fixed`` / ``hash_varlen`` (the GPU form of ``_hash_words_np``).
All hashing runs in hand-written sm_100a CUDA kernels in
``libhalftime_b200.so`` (C-ABI: include/halftime_b200.h); there is no CPU
fallback.
"""

from ._errors import SeedSizeError
from .hasher import (
    ENGINES,
    Digest,
    SeedBuffer,
    SeedLayout,
    digest,
    expand_seed,
    hash_bytes,
    instance_count,
    seed_for_input,
    seed_layout,
    seed_words_needed,
)
from .params import (
    SUPPORTED_COEFFICIENTS,
    VARIANTS,
    ErasureCode,
    HashParams,
    TransformMatrix,
    coefficient_multiply,
    variant,
)

__version__ = "0.1.0"

__all__ = [
    "Digest", "ErasureCode", "HashParams", "SeedBuffer", "SeedLayout", "SeedSizeError", "TransformMatrix",
    "VARIANTS", "digest", "expand_seed", "hash_bytes", "instance_count", "seed_for_input", "seed_layout",
    "seed_words_needed", "variant", "hash_fixed", "hash_varlen", "hash_words", "hash_fixed_host", "fill_bytes",
    "hash_fixed_folds", "hash_words_many_seeds", "StreamHasher", "varlen_status", "release_host", "fill_strings", "ENGINES",
    "SUPPORTED_COEFFICIENTS", "coefficient_multiply",
    "__version__",
]


def __getattr__(name):
    # batch entry points import torch lazily so host-only use stays light
    if name in ("hash_fixed", "hash_varlen", "hash_words", "hash_fixed_host", "fill_bytes", "hash_fixed_folds",
                "hash_words_many_seeds", "varlen_status", "release_host", "fill_strings"):
        from . import batch

        return getattr(batch, name)
    if name == "StreamHasher":
        from .stream import StreamHasher

        return StreamHasher
    raise AttributeError(name)
