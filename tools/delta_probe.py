"""Where collect_delta's time goes: device cycle with LOD_FLAG_DELTA, the
delta D2H (lod_read_delta), the host assembly (structure / voxel / point lists)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_03567_b200 import _lib, insert_batch, synth, update, wait_settled  # noqa: E402
from bench import new_tree  # noqa: E402

tree, state = new_tree(0, 8 << 30)
NW = int(os.environ.get("NW", 30))
bs = [synth.gen_surface(1_000_000, 1000 + i) for i in range(NW + 10)]
db = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in bs]
for i in range(NW):
    insert_batch(tree, *db[i], state)
wait_settled(tree, state)
orig = update._read_delta
t_read = []


def timed_read(t):
    t0 = time.perf_counter()
    info = _lib.LodDeltaInfo()
    _lib.check(t._L.lod_delta_info(t.handle, ctypes.byref(info)))
    t1 = time.perf_counter()
    d = orig(t)
    t2 = time.perf_counter()
    t_read.append((t1 - t0, t2 - t1, info.n_voxels, info.n_voxel_groups, info.n_splits))
    return d


update._read_delta = timed_read
for i in range(NW, NW + 10):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    insert_batch(tree, *db[i], state, collect_delta=bool(i % 2))
    wait_settled(tree, state)
    t1 = time.perf_counter()
    print(f"batch {i} delta={bool(i % 2)} total {1e3 * (t1 - t0):.3f} ms", t_read[-1] if i % 2 else "")
# split the read: D2H only vs assembly
info = _lib.LodDeltaInfo()
_lib.check(tree._L.lod_delta_info(tree.handle, ctypes.byref(info)))
nv = info.n_voxels
for kind in ("pageable", "pinned"):
    a = np.empty(nv, np.uint32) if kind == "pageable" else _lib.pinned_empty(nv, np.uint32)
    b = np.empty(nv, np.uint32) if kind == "pageable" else _lib.pinned_empty(nv, np.uint32)
    for _ in range(3):
        t0 = time.perf_counter()
        _lib.check(tree._L.lod_read_delta(tree.handle, None, None, None, None, _lib.ptr(a), _lib.ptr(b), None, None,
                                          None))
        t1 = time.perf_counter()
    print(kind, "cells+rgba D2H", nv, f"{1e3 * (t1 - t0):.3f} ms")
t0 = time.perf_counter()
_ = tree.children
t1 = time.perf_counter()
tree._invalidate()
_ = tree.children
t2 = time.perf_counter()
print(f"children cached {1e3 * (t1 - t0):.3f} ms, refresh {1e3 * (t2 - t1):.3f} ms, nodes {tree.num_nodes}")
