"""Independent numpy oracles -- TEST INFRASTRUCTURE ONLY.

Restatements of the reference test suite's oracles (pkg/tests/oracles.py),
which share no code with the engine: a top-down rebuild of the settled tree
from the whole dataset (oracles.py:55-96), path-keyed comparison
(oracles.py:99-147) and a numpy min-scatter rasterizer (oracles.py:258-286).
Formulas that the contract pins bit-exactly (cells, routing, depth) keep the
reference's operation order.
"""
from __future__ import annotations

import numpy as np


def ref_cells(px, py, pz, bx, by, bz, s, g):
    """Clamped occupancy cells (oracles.py:18-26)."""
    c = [np.clip(np.floor(g * (p - b) / s), 0, g - 1).astype(np.int64) for p, b in ((px, bx), (py, by), (pz, bz))]
    return (c[2] * g + c[1]) * g + c[0]


class RefNode:
    __slots__ = ("inner", "level", "xyz", "rgba", "cells", "colors")

    def __init__(self, inner, level):
        self.inner, self.level = inner, level
        self.xyz = self.rgba = self.cells = self.colors = None


def build_reference(xyz, rgba, bmin, size, *, grid_res, leaf_threshold, max_depth):
    """{octant path: RefNode} of the settled tree (oracles.py:55-96).

    Inner regions (more than T points, above the depth cap) keep the first
    point per occupied cell in dataset order, listed in claim order; leaves
    keep their points in dataset order.
    """
    g = grid_res
    p64 = np.asarray(xyz, np.float64)
    out = {}
    work = [((), np.arange(len(rgba)), float(bmin[0]), float(bmin[1]), float(bmin[2]), float(size), 0)]
    while work:
        path, idx, bx, by, bz, s, level = work.pop()
        if len(idx) > leaf_threshold and level < max_depth:
            node = RefNode(True, level)
            px, py, pz = p64[idx, 0], p64[idx, 1], p64[idx, 2]
            cell = ref_cells(px, py, pz, bx, by, bz, s, g)
            _, first = np.unique(cell, return_index=True)
            first.sort()
            node.cells, node.colors = cell[first], rgba[idx[first]]
            out[path] = node
            h = s * 0.5
            oct_ = (px >= bx + h).astype(np.int8) | ((py >= by + h).astype(np.int8) << 1) | (
                (pz >= bz + h).astype(np.int8) << 2)
            for o in range(8):
                work.append((path + (o,), idx[oct_ == o], bx + h if o & 1 else bx, by + h if o & 2 else by,
                             bz + h if o & 4 else bz, h, level + 1))
        else:
            node = RefNode(False, level)
            node.xyz, node.rgba = xyz[idx], rgba[idx]
            out[path] = node
    return out


def tree_paths(inner, children) -> dict:
    """{octant path: node id} walked from the root (oracles.py:99-110)."""
    out = {(): 0}
    todo = [((), 0)]
    while todo:
        path, nid = todo.pop()
        if inner[nid]:
            for o in range(8):
                kid = int(children[nid, o])
                out[path + (o,)] = kid
                todo.append((path + (o,), kid))
    return out


def assert_matches_reference(tree, ref) -> None:
    """Topology, leaf sequences, voxel colours / centres / bitgrids by path (oracles.py:113-147)."""
    paths = tree_paths(tree.inner, tree.children)
    assert set(paths) == set(ref), f"topology differs: {len(paths)} vs {len(ref)} nodes"
    g = tree.grid_res
    for path, nid in paths.items():
        want = ref[path]
        assert bool(tree.inner[nid]) == want.inner, f"kind differs at {path}"
        got_xyz, got_rgba = tree.gather_samples(nid)
        if not want.inner:
            assert np.array_equal(got_xyz, want.xyz), f"leaf points at {path}"
            assert np.array_equal(got_rgba, want.rgba), f"leaf colors at {path}"
        else:
            assert np.array_equal(got_rgba, want.colors), f"voxel colors at {path}"
            bx, by, bz = tree.bmin[nid]
            step = tree.node_size(nid) / g
            cx, cy, cz = want.cells % g, (want.cells // g) % g, want.cells // (g * g)
            centers = np.stack([bx + (cx + 0.5) * step, by + (cy + 0.5) * step, bz + (cz + 0.5) * step],
                               axis=-1).astype(np.float32).reshape(-1, 3)
            assert np.array_equal(got_xyz, centers), f"voxel centers at {path}"
            assert np.array_equal(np.sort(tree.occupied_cells(nid)), np.sort(want.cells)), f"bitgrid at {path}"


def ref_render(xyz, rgba, cam, width, height):
    """numpy projection + unordered np.minimum.at scatter (oracles.py:258-286).

    ``cam`` is the 18-double Camera.packed() block.
    """
    pos, right, up, fwd = cam[0:3], cam[3:6], cam[6:9], cam[9:12]
    tan_half, aspect, near, far = cam[12], cam[13], cam[14], cam[15]
    p = np.asarray(xyz, np.float64)
    dx, dy, dz = p[:, 0] - pos[0], p[:, 1] - pos[1], p[:, 2] - pos[2]
    zv = dx * fwd[0] + dy * fwd[1] + dz * fwd[2]
    xv = dx * right[0] + dy * right[1] + dz * right[2]
    yv = dx * up[0] + dy * up[1] + dz * up[2]
    keep = (zv > near) & (zv < far)
    with np.errstate(divide="ignore", invalid="ignore"):
        ndc_x = np.where(keep, xv / (zv * tan_half * aspect), 0.0)
        ndc_y = np.where(keep, yv / (zv * tan_half), 0.0)
        depth = far * (zv - near) / ((far - near) * np.where(zv == 0.0, 1.0, zv))
        px = np.floor((ndc_x + 1.0) * 0.5 * width).astype(np.int64)
        py = np.floor((1.0 - ndc_y) * 0.5 * height).astype(np.int64)
    keep &= (px >= 0) & (px < width) & (py >= 0) & (py < height)
    bits = depth.astype(np.float32).view(np.uint32).astype(np.uint64)
    packed = (bits << np.uint64(32)) | np.asarray(rgba).astype(np.uint64)
    fb = np.full(width * height, np.uint64(0xFFFFFFFFFFFFFFFF))
    np.minimum.at(fb, (py * width + px)[keep], packed[keep])
    return fb
