"""Exceptions mirroring the reference (halftimehash/hasher.py:36-37)."""


class SeedSizeError(ValueError):
    """Seed buffer capacity below what this input length requires."""
