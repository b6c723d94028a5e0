"""Acceptance C9's workload (test_acceptance.py:317-346): 1M uniform points
into trees of chunk capacity 500..10000, rasterize at the bench camera; wall
time per render (min of 7) and the device-side split (selection + splat)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2310_03567_b200 import Arena, ChunkPool, CubeBounds, Octree, UpdateConfig, UpdateState, insert_batch, synth
from paper_2310_03567_b200.render import Camera, rasterize

xyz, rgba = synth.generate("uniform", 1_000_000, 9)
cam = Camera(position=(0.5, 0.5, -1.5), target=(0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=100.0, width=1024,
             height=768)
for cs in (500, 1000, 2000, 5000, 10000):
    arena = Arena(1 << 30)
    tree = Octree(CubeBounds((0.0, 0.0, 0.0), 1.0), arena, ChunkPool(arena, cs), grid_res=128, leaf_threshold=50_000,
                  max_depth=20)
    st = UpdateState(UpdateConfig())
    for i in range(0, 1_000_000, 100_000):
        insert_batch(tree, xyz[i:i + 100_000], rgba[i:i + 100_000], st)
    times = []
    for _ in range(7):
        t0 = time.perf_counter()
        fb, rep = rasterize(tree, cam, threshold=128.0)
        times.append(time.perf_counter() - t0)
    print(json.dumps({"C": cs, "best_ms": round(min(times) * 1e3, 3), "all_ms": [round(t * 1e3, 3) for t in times],
                      "chunks": tree.pool.allocated_total, "nodes_drawn": rep.nodes_drawn,
                      "samples": rep.samples_drawn}))
    tree.close()
