"""Small-path split of a tiny-batch stream: wall per call vs device time per
call (the kernels' own globaltimer spans, folded by lod_tree_settle) vs the
host-side cost of the call (the Python facade + C ABI, measured with the
device idle)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2310_03567_b200 import Arena, ChunkPool, CubeBounds, Octree, UpdateConfig, UpdateState, insert_batch

for bs, total in ((1, 30_000), (7, 70_000)):
    rng = np.random.default_rng(bs)
    xyz = rng.random((total, 3)).astype(np.float32)
    rgba = rng.integers(0, 1 << 32, total, dtype=np.uint64).astype(np.uint32)
    arena = Arena(256 << 20)
    tree = Octree(CubeBounds((0.0, 0.0, 0.0), 1.0), arena, ChunkPool(arena, 1000), grid_res=16, leaf_threshold=100,
                  max_depth=12)
    state = UpdateState(UpdateConfig())
    parts = [(xyz[i:i + bs], rgba[i:i + bs]) for i in range(0, total, bs)]
    for x, c in parts[:50]:
        insert_batch(tree, x, c, state)
    s0 = state.stats.device_seconds
    t0 = time.perf_counter()
    for x, c in parts[50:]:
        insert_batch(tree, x, c, state)
    t_host = time.perf_counter() - t0
    st = state.stats
    t_all = time.perf_counter() - t0
    calls = len(parts) - 50
    print(json.dumps({"batch": bs, "wall_us_per_call": round(t_all / calls * 1e6, 2),
                      "host_loop_us_per_call": round(t_host / calls * 1e6, 2),
                      "device_us_per_call": round((st.device_seconds - s0) / calls * 1e6, 2), "calls": calls}))

# the C ABI alone (no facade): same stream, a fresh tree, prebuilt arguments
import ctypes  # noqa: E402

from paper_2310_03567_b200 import _lib  # noqa: E402

for bs, total in ((1, 30_000), (7, 70_000)):
    rng = np.random.default_rng(bs)
    xyz = rng.random((total, 3)).astype(np.float32)
    rgba = rng.integers(0, 1 << 32, total, dtype=np.uint64).astype(np.uint32)
    arena = Arena(256 << 20)
    tree = Octree(CubeBounds((0.0, 0.0, 0.0), 1.0), arena, ChunkPool(arena, 1000), grid_res=16, leaf_threshold=100,
                  max_depth=12)
    state = UpdateState(UpdateConfig())
    for i in range(0, 50 * bs, bs):
        insert_batch(tree, xyz[i:i + bs], rgba[i:i + bs], state)
    state.stats
    h = tree.handle
    lim = state._limits
    bst = state._bstats
    fn = tree._L.lod_insert_batch
    args = [(xyz.ctypes.data + 12 * i, rgba.ctypes.data + 4 * i) for i in range(50 * bs, total - bs + 1, bs)]
    lr, br = ctypes.byref(lim), ctypes.byref(bst)
    t0 = time.perf_counter()
    for px, pc in args:
        fn(h, px, pc, bs, lr, 0, br)
    t_host = time.perf_counter() - t0
    _lib.check(tree._L.lod_tree_settle(h, ctypes.byref(_lib.LodSettleStats())), "settle")
    t_all = time.perf_counter() - t0
    print(json.dumps({"batch": bs, "abi_only": True, "wall_us_per_call": round(t_all / len(args) * 1e6, 2),
                      "host_loop_us_per_call": round(t_host / len(args) * 1e6, 2), "calls": len(args)}))
