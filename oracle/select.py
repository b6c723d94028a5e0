"""Host restatement of the reference's LOD selection -- TEST INFRASTRUCTURE ONLY.

``select_visible`` follows lodstream/render.py:127-200 line for line with the
same numpy operations (frustum_planes, frustum_intersects, screen_size, the
octant-ordered stack walk), over plain node columns (``inner``, ``count``,
``children``, ``bmin``, ``level``) so it runs on the product's host mirror or
on the oracle tree alike.  The GPU selection (lod_select_visible) is checked
against it; ``decision_margins`` reports how close each visited node's
frustum / pixel-size decision was, to tell float-order ties from real bugs.
"""
from __future__ import annotations

import math

import numpy as np


def basis(position, target, up):
    pos = np.asarray(position, np.float64)
    fwd = np.asarray(target, np.float64) - pos
    fwd = fwd / np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, np.float64))
    right = right / np.linalg.norm(right)
    return right, np.cross(right, fwd), fwd


def corners(bmin, size):
    out = np.empty((8, 3), dtype=np.float64)
    for i in range(8):
        out[i, 0] = bmin[0] + (size if i & 1 else 0.0)
        out[i, 1] = bmin[1] + (size if i & 2 else 0.0)
        out[i, 2] = bmin[2] + (size if i & 4 else 0.0)
    return out


def frustum_planes(cam) -> np.ndarray:
    """render.py:127-148."""
    right, up, fwd = basis(cam.position, cam.target, cam.up)
    pos = np.asarray(cam.position, np.float64)
    th = math.tan(math.radians(cam.fov_deg) * 0.5)
    asp = cam.width / cam.height
    planes = np.empty((6, 4), np.float64)

    def put(i, n, through):
        n = n / np.linalg.norm(n)
        planes[i, :3] = n
        planes[i, 3] = -n @ through

    put(0, fwd, pos + fwd * cam.near)
    put(1, -fwd, pos + fwd * cam.far)
    put(2, right + fwd * (th * asp), pos)
    put(3, -right + fwd * (th * asp), pos)
    put(4, up + fwd * th, pos)
    put(5, -up + fwd * th, pos)
    return planes


def frustum_intersects(c, planes) -> bool:
    """render.py:151-157."""
    for i in range(6):
        if (c @ planes[i, :3] + planes[i, 3] < 0.0).all():
            return False
    return True


def screen_size(c, cam) -> float:
    """render.py:160-174."""
    right, up, fwd = basis(cam.position, cam.target, cam.up)
    th = math.tan(math.radians(cam.fov_deg) * 0.5)
    asp = cam.width / cam.height
    d = c - np.asarray(cam.position, np.float64)
    zv = d @ fwd
    if (zv <= cam.near).any():
        return math.inf
    sx = (d @ right / (zv * th * asp) + 1.0) * 0.5 * cam.width
    sy = (1.0 - d @ up / (zv * th)) * 0.5 * cam.height
    return float(max(sx.max() - sx.min(), sy.max() - sy.min()))


def select_visible(cols: dict, size0: float, cam, threshold: float = 128.0) -> list[int]:
    """render.py:177-200 over node columns."""
    inner, count, children, bmin, level = (cols[k] for k in ("inner", "count", "children", "bmin", "level"))
    if not inner[0] and count[0] == 0:
        return []
    planes = frustum_planes(cam)
    out: list[int] = []
    stack = [0]
    while stack:
        nid = stack.pop()
        c = corners(bmin[nid], size0 * (0.5 ** int(level[nid])))
        if not frustum_intersects(c, planes):
            continue
        if inner[nid] and screen_size(c, cam) > threshold:
            for o in range(7, -1, -1):
                stack.append(int(children[nid, o]))
        else:
            out.append(nid)
    return out


def decision_margins(cols: dict, size0: float, cam, threshold: float, nodes) -> dict:
    """Per node: (frustum margin = max over planes of the smallest |max corner
    distance|, relative pixel-size margin |size - threshold| / threshold)."""
    planes = frustum_planes(cam)
    out = {}
    for nid in nodes:
        c = corners(cols["bmin"][nid], size0 * (0.5 ** int(cols["level"][nid])))
        fm = min(abs(float((c @ planes[i, :3] + planes[i, 3]).max())) for i in range(6))
        ss = screen_size(c, cam)
        sm = abs(ss - threshold) / max(abs(threshold), 1.0) if math.isfinite(ss) else math.inf
        out[nid] = (fm, sm)
    return out
