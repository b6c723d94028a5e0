"""Seeded synthetic point clouds for the benchmark configs (BASELINE.json).

* ``gen_uniform`` / ``gen_surface`` restate the reference generators
  (lodstream/synth.py:20-40) so configs 1, 2 and 5 see the same inputs;
* ``gen_mesh`` (config 3) and ``gen_skew`` (config 4) are new: the reference
  has no generator for them.

Input generation is outside the timed region; it runs on the host with numpy.
"""
from __future__ import annotations

import numpy as np


def _pack(r, g, b) -> np.ndarray:
    out = r.astype(np.uint32)
    out |= g.astype(np.uint32) << 8
    out |= b.astype(np.uint32) << 16
    out |= np.uint32(255) << 24
    return out


def gen_uniform(n: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """Uniform in the unit cube, uniform rgb, a=255 (synth.py:20-24)."""
    rng = np.random.default_rng(seed)
    xyz = rng.random((n, 3), np.float32)
    rgb = rng.integers(0, 256, (n, 3), np.uint32)
    return xyz, _pack(rgb[:, 0], rgb[:, 1], rgb[:, 2])


def gen_surface(n: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    """2.5D LIDAR-like height field + noise (synth.py:27-40)."""
    rng = np.random.default_rng(seed)
    x = rng.random(n)
    y = rng.random(n)
    z = 0.5 + 0.18 * np.sin(5.1 * x + 1.7) * np.cos(4.3 * y) + 0.08 * np.sin(11.0 * x * y)
    z += rng.normal(0.0, 0.004, n)
    xyz = np.empty((n, 3), np.float32)
    xyz[:, 0] = x
    xyz[:, 1] = y
    xyz[:, 2] = np.clip(z, 0.0, 0.999)
    shade = (np.clip(z, 0.0, 1.0) * 255).astype(np.uint32)
    return xyz, _pack((x * 255).astype(np.uint32), (y * 255).astype(np.uint32), shade)


def mesh_scene(n_tri: int = 20_000, seed: int = 7) -> tuple[np.ndarray, np.ndarray]:
    """A fixed random triangle soup in the unit cube with per-vertex rgb:
    vertices (n_tri, 3, 3) f64 and colours (n_tri, 3, 3) f64 in [0, 255]."""
    rng = np.random.default_rng(seed)
    centres = rng.random((n_tri, 1, 3)) * 0.9 + 0.05
    verts = np.clip(centres + rng.normal(0.0, 0.02, (n_tri, 3, 3)), 0.0, 0.999)
    cols = rng.random((n_tri, 3, 3)) * 255.0
    return verts, cols


def gen_mesh(n: int, seed: int, scene=None) -> tuple[np.ndarray, np.ndarray]:
    """Photogrammetry-style surface samples (config 3): area-weighted triangle
    choice, uniform barycentrics (sqrt trick), interpolated rgb, a=255."""
    verts, cols = scene if scene is not None else mesh_scene()
    a, b, c = verts[:, 0], verts[:, 1], verts[:, 2]
    area = 0.5 * np.linalg.norm(np.cross(b - a, c - a), axis=1)
    p = area / area.sum()
    rng = np.random.default_rng(seed)
    tri = rng.choice(len(p), size=n, p=p)
    r1 = np.sqrt(rng.random(n))
    r2 = rng.random(n)
    w0, w1, w2 = 1.0 - r1, r1 * (1.0 - r2), r1 * r2
    pts = w0[:, None] * a[tri] + w1[:, None] * b[tri] + w2[:, None] * c[tri]
    rgb = w0[:, None] * cols[tri, 0] + w1[:, None] * cols[tri, 1] + w2[:, None] * cols[tri, 2]
    rgb = np.clip(np.rint(rgb), 0, 255).astype(np.uint32)
    xyz = np.clip(pts, 0.0, 0.999).astype(np.float32)
    return xyz, _pack(rgb[:, 0], rgb[:, 1], rgb[:, 2])


SKEW_CORNER = (0.61, 0.23, 0.47)
SKEW_SIDE = 1e-4 ** (1.0 / 3.0)  # a 1e-4-volume cube


def gen_skew(n: int, seed: int, frac: float = 0.9) -> tuple[np.ndarray, np.ndarray]:
    """Density-skew stress (config 4): ``frac`` of the points uniform in a cube
    of volume 1e-4 at SKEW_CORNER, the rest uniform in the unit cube, shuffled."""
    rng = np.random.default_rng(seed)
    k = int(round(n * frac))
    dense = rng.random((k, 3)) * SKEW_SIDE + np.asarray(SKEW_CORNER)
    sparse = rng.random((n - k, 3))
    pts = np.concatenate([dense, sparse])[rng.permutation(n)]
    rgb = rng.integers(0, 256, (n, 3), np.uint32)
    return pts.astype(np.float32), _pack(rgb[:, 0], rgb[:, 1], rgb[:, 2])


GENERATORS = {"uniform": gen_uniform, "surface": gen_surface, "mesh": gen_mesh, "skew": gen_skew}


def generate(kind: str, n: int, seed: int) -> tuple[np.ndarray, np.ndarray]:
    try:
        gen = GENERATORS[kind]
    except KeyError:
        raise ValueError(f"unknown generator {kind!r}, have {sorted(GENERATORS)}") from None
    return gen(n, seed)
