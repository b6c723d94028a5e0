"""Per-call wall latency of insert_batch for tiny batches (C1's regime:
test_acceptance.py:81-101 makes 1.52M calls of 1..1000 points at G=16,
T=100, C=1000, max depth 12).  Prints one JSON line per batch size."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2310_03567_b200 import Arena, ChunkPool, CubeBounds, Octree, UpdateConfig, UpdateState, insert_batch


def run(bs: int, total: int) -> dict:
    rng = np.random.default_rng(bs)
    xyz = rng.random((total, 3)).astype(np.float32)
    rgba = rng.integers(0, 1 << 32, total, dtype=np.uint64).astype(np.uint32)
    arena = Arena(256 << 20)
    tree = Octree(CubeBounds((0.0, 0.0, 0.0), 1.0), arena, ChunkPool(arena, 1000), grid_res=16,
                  leaf_threshold=100, max_depth=12)
    state = UpdateState(UpdateConfig())
    parts = [(xyz[i:i + bs], rgba[i:i + bs]) for i in range(0, total, bs)]
    for x, c in parts[:20]:
        insert_batch(tree, x, c, state)
    t0 = time.perf_counter()
    for x, c in parts[20:]:
        insert_batch(tree, x, c, state)
    _ = tree.num_nodes  # settle
    dt = time.perf_counter() - t0
    calls = len(parts) - 20
    return {"batch": bs, "calls": calls, "us_per_call": round(dt / calls * 1e6, 2),
            "points_per_s": round((total - 20 * bs) / dt, 1), "nodes": tree.num_nodes}


if __name__ == "__main__":
    for bs, total in ((1, 20_000), (7, 70_000), (100, 200_000), (1000, 200_000)):
        print(json.dumps(run(bs, total)), flush=True)
