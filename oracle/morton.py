"""Numpy restatement of the reference's Morton order -- TEST INFRASTRUCTURE ONLY.

Follows lodstream/io.py:419-446 (``_spread_bits``, ``morton_key``,
``morton_sort``) operation for operation; pinned by
tests/test_oracle_golden.py against keys and orders produced by the reference
itself (tests/golden/morton.npz).
"""
from __future__ import annotations

import numpy as np


def spread_bits(v: np.ndarray) -> np.ndarray:
    """io.py:418-427: space 21-bit integers so consecutive bits land 3 apart."""
    v = v.astype(np.uint64)
    v &= np.uint64(0x1FFFFF)
    for shift, mask in ((32, 0x1F00000000FFFF), (16, 0x1F0000FF0000FF), (8, 0x100F00F00F00F00F),
                        (4, 0x10C30C30C30C30C3), (2, 0x1249249249249249)):
        v = (v | (v << np.uint64(shift))) & np.uint64(mask)
    return v


def morton_key(xyz: np.ndarray, bmin, size: float, bits: int = 21) -> np.ndarray:
    """io.py:430-440."""
    scale = (1 << bits) / size
    top = (1 << bits) - 1
    keys = np.zeros(len(xyz), np.uint64)
    for axis in range(3):
        with np.errstate(invalid="ignore"):
            q = ((xyz[:, axis].astype(np.float64) - bmin[axis]) * scale).astype(np.int64)
        np.clip(q, 0, top, out=q)
        keys |= spread_bits(q) << np.uint64(axis)
    return keys


def morton_order(xyz: np.ndarray, bmin, size: float) -> np.ndarray:
    """io.py:443-446: the stable argsort behind morton_sort."""
    return np.argsort(morton_key(xyz, bmin, size), kind="stable")
