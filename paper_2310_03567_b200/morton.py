"""Device Morton order (reference: lodstream/io.py:419-446).

``morton_key`` / ``morton_sort`` keep the reference's signatures and results
(64-bit keys, x at bit 0 then y, z; stable reorder) and run as one call into
the CUDA library (``lod_morton_sort``: key kernel + LSD onesweep radix passes +
one gather).  Pre-sorting a stream along the curve is the paper's locality
gain for insertion (the CLI's ``sort-morton``, cli.py:282-292).
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .octree import CubeBounds


def _morton(xyz, rgba, bounds: CubeBounds, bits: int, device: int, keys: bool, records: bool):
    L = _lib.require_device(device)
    if not 1 <= bits <= 21:
        raise ValueError("bits must be in 1..21")
    xyz = np.ascontiguousarray(xyz, np.float32).reshape(-1, 3)
    n = len(xyz)
    rg = np.ascontiguousarray(rgba, np.uint32).reshape(-1) if rgba is not None else None
    if rg is not None and len(rg) != n:
        raise ValueError("xyz and rgba lengths differ")
    ko = np.empty(n, np.uint64) if keys else None
    xo = np.empty_like(xyz) if records else None
    ro = np.empty_like(rg) if (records and rg is not None) else None
    if n:
        scale = (1 << bits) / bounds.size  # io.py:432, the same Python float expression
        bmin = np.ascontiguousarray(bounds.min, np.float64)
        p = _lib.ptr
        _lib.check(L.lod_morton_sort(device, p(bmin), float(scale), int(bits), p(xyz), p(rg), n, p(xo), p(ro),
                                     p(ko), 0), "morton_sort")
    return ko, xo, ro


def morton_key(xyz, bounds: CubeBounds, bits: int = 21, device: int = 0) -> np.ndarray:
    """64-bit Morton codes: x at bit 0, then y, then z, interleaved (io.py:430-440)."""
    return _morton(xyz, None, bounds, bits, device, keys=True, records=False)[0]


def morton_sort(xyz, rgba, bounds: CubeBounds, device: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Stable reorder of a point set by Morton key (io.py:443-446)."""
    _, xo, ro = _morton(xyz, rgba, bounds, 21, device, keys=False, records=True)
    return xo, ro
