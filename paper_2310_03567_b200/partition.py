"""Octant-prefix partitioning of a point stream across GPUs.

The key is the octant path of a point over the first ``depth`` levels of the
root cube, computed with the reference's exact float64 descent rule
(``x >= bx + h`` per axis, _kernels.py:44-56) -- not a quantised Morton key,
whose rounding could route boundary points differently (io.py:431-440).
Prefixes are assigned to ranks greedily by descending count (LPT): level-1
octants balance 2 and 4 ranks, level-2 prefixes balance 8.
Each rank keeps its points in global order, so its subtrees see exactly the
ingestion order of a single-device run.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def prefix_of(xyz: np.ndarray, depth: int, bmin=(0.0, 0.0, 0.0), size: float = 1.0) -> np.ndarray:
    """Octant path of every point over ``depth`` levels, as a base-8 integer
    (first octant most significant)."""
    p = np.asarray(xyz, np.float64).reshape(-1, 3)
    b = np.tile(np.asarray(bmin, np.float64), (len(p), 1))
    s = float(size)
    key = np.zeros(len(p), np.int64)
    for _ in range(depth):
        h = s * 0.5
        o = np.zeros(len(p), np.int64)
        for axis in range(3):
            up = p[:, axis] >= b[:, axis] + h
            o |= up.astype(np.int64) << axis
            b[:, axis] = np.where(up, b[:, axis] + h, b[:, axis])
        s = h
        key = key * 8 + o
    return key


@dataclass
class Plan:
    depth: int
    owner: np.ndarray  # (8**depth,) rank per prefix
    load: np.ndarray   # (world,) sample points per rank


def plan_owners(sample_batches, world: int, depth: int | None = None, bmin=(0.0, 0.0, 0.0),
                size: float = 1.0) -> Plan:
    """LPT assignment of prefixes to ranks from a sample of the stream."""
    if depth is None:
        depth = 1 if world <= 4 else 2
    counts = np.zeros(8 ** depth, np.int64)
    for x, _ in sample_batches:
        counts += np.bincount(prefix_of(x, depth, bmin, size), minlength=8 ** depth)
    owner = np.zeros(8 ** depth, np.int32)
    load = np.zeros(world, np.int64)
    for pre in np.argsort(-counts, kind="stable"):
        r = int(np.argmin(load))
        owner[pre] = r
        load[r] += counts[pre]
    return Plan(depth, owner, load)


def take(plan: Plan, xyz: np.ndarray, rgba: np.ndarray, rank: int, bmin=(0.0, 0.0, 0.0), size: float = 1.0):
    """This rank's points of a batch, in global order."""
    mask = plan.owner[prefix_of(xyz, plan.depth, bmin, size)] == rank
    return np.ascontiguousarray(xyz[mask]), np.ascontiguousarray(rgba[mask])


def imbalance(plan: Plan) -> float:
    """max / mean load of the plan."""
    m = plan.load.mean()
    return float(plan.load.max() / m) if m > 0 else 1.0
