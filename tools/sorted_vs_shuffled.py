"""Acceptance C10's workload (test_acceptance.py:349-374): 1M uniform points
in 100k-point batches, Morton-sorted vs shuffled, per-phase device times
(LOD_FLAG_PROFILE) and the settled wall time per ordering."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2310_03567_b200 import Arena, ChunkPool, CubeBounds, Octree, UpdateConfig, UpdateState, insert_batch, synth
from paper_2310_03567_b200.morton import morton_sort


def build(xyz, rgba, profile):
    arena = Arena(1 << 30)
    tree = Octree(CubeBounds((0.0, 0.0, 0.0), 1.0), arena, ChunkPool(arena, 1000), grid_res=128,
                  leaf_threshold=50_000, max_depth=20)
    state = UpdateState(UpdateConfig())
    phases = {}
    t0 = time.perf_counter()
    for i in range(0, len(rgba), 100_000):
        insert_batch(tree, xyz[i:i + 100_000], rgba[i:i + 100_000], state, profile=profile)
        if profile:
            for k, v in state.last["phase_ms"].items():
                phases[k] = phases.get(k, 0.0) + v
    st = state.stats
    wall = time.perf_counter() - t0
    tree.close()
    return wall, st.update_seconds, phases


if __name__ == "__main__":
    xyz, rgba = synth.gen_uniform(1_000_000, 10)
    sx, sr = morton_sort(xyz, rgba, CubeBounds((0.0, 0.0, 0.0), 1.0))
    perm = np.random.default_rng(100).permutation(len(rgba))
    hx, hr = xyz[perm].copy(), rgba[perm].copy()
    build(hx, hr, False)
    for name, (x, c) in (("sorted", (sx, sr)), ("shuffled", (hx, hr))):
        walls = [build(x, c, False)[:2] for _ in range(5)]
        _, _, ph = build(x, c, True)
        print(json.dumps({"order": name, "wall_s": [round(w, 5) for w, _ in walls],
                          "update_seconds": [round(u, 5) for _, u in walls],
                          "phase_ms": {k: round(v, 3) for k, v in ph.items()}}))
