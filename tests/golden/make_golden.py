"""Generate golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports ``lodstream`` from /root/reference/pkg/src (read-only, numba JIT),
replays a set of scenarios that cover the reference test suite's pinned cases
 and writes one compressed ``.npz`` per scenario next to this
script.  The fixtures hold the inputs, the reference's complete observable
tree state after the last batch (node table, pool tables, counters, every
node's sample sequence, every inner node's occupied cells) and framebuffers.
Nothing on the GPU box reads /root/reference; the tests read these files.
"""
from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _import_ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF)
    from lodstream import octree, render, store, update, errors  # noqa: F401

    return octree, render, store, update, errors


def cloud(n, seed=0, kind="uniform"):
    """Same construction as the reference suite's conftest.cloud (conftest.py:66-79)."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        xyz = rng.random((n, 3)).astype(np.float32)
    elif kind == "surface":
        xy = rng.random((n, 2))
        z = 0.5 + 0.2 * np.sin(6.0 * xy[:, 0]) * np.cos(5.0 * xy[:, 1])
        xyz = np.column_stack([xy[:, 0], xy[:, 1], z]).astype(np.float32)
    elif kind == "skew":
        k = int(n * 0.9)
        dense = rng.random((k, 3)) * 0.0464 + np.array([0.61, 0.23, 0.47])
        xyz = np.concatenate([dense, rng.random((n - k, 3))])[rng.permutation(n)].astype(np.float32)
    else:
        raise ValueError(kind)
    np.clip(xyz, 0.0, np.nextafter(np.float32(1.0), np.float32(0.0)), out=xyz)
    rgba = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    return xyz, rgba


def pack_rgba(r, g, b, a=255):
    return (r & 0xFF) | (g & 0xFF) << 8 | (b & 0xFF) << 16 | (a & 0xFF) << 24


RED, GREEN, BLUE = pack_rgba(255, 0, 0), pack_rgba(0, 255, 0), pack_rgba(0, 0, 255)


def canonical():
    return (np.array([[0.1, 0.1, 0.1], [0.2, 0.2, 0.2], [0.8, 0.8, 0.8]], np.float32),
            np.array([RED, GREEN, BLUE], np.uint32))


def ten_points():
    lo = [(0.05, 0.05, 0.05), (0.1, 0.1, 0.1), (0.15, 0.15, 0.15), (0.2, 0.2, 0.2)]
    mid = [(0.3, 0.3, 0.3)]
    hi = [(0.6, 0.6, 0.6), (0.7, 0.65, 0.8), (0.9, 0.9, 0.55), (0.8, 0.8, 0.8), (0.55, 0.95, 0.7)]
    return np.array(lo + mid + hi, np.float32), np.arange(10, dtype=np.uint32) + 1


def scenarios():
    """(name, params, [batches]) -- params: tree + update config."""
    out = []
    base = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=64 << 20, chunk_capacity=1000,
                grid_res=16, leaf_threshold=100, max_depth=12,
                backlog_capacity=10_000_000, spill_capacity=100_000_000)

    def P(**kw):
        d = dict(base)
        d.update(kw)
        return d

    x, c = canonical()
    out.append(("canonical", P(chunk_capacity=2, grid_res=4, leaf_threshold=2), [(x, c)]))
    out.append(("canonical_1by1", P(chunk_capacity=2, grid_res=4, leaf_threshold=2),
                [(x[i:i + 1], c[i:i + 1]) for i in range(3)]))
    x, c = ten_points()
    more = (np.array([[0.28, 0.29, 0.3], [0.31, 0.27, 0.26]], np.float32), np.array([100, 101], np.uint32))
    out.append(("ten_points_spill", P(chunk_capacity=4, grid_res=4, leaf_threshold=5), [(x, c), more]))
    out.append(("depth_cap", P(grid_res=4, leaf_threshold=2, max_depth=3),
                [(np.full((7, 3), 0.3, np.float32), np.arange(7, dtype=np.uint32))]))
    rng = np.random.default_rng(3)
    out.append(("colocated", P(grid_res=4, leaf_threshold=5),
                [((rng.random((10, 3)) * 0.02).astype(np.float32), np.arange(10, dtype=np.uint32))]))
    for bs in (2000, 333, 31):
        x, c = cloud(2000, seed=13)
        out.append((f"rebuild_bs{bs}", P(grid_res=8, leaf_threshold=50),
                    [(x[i:i + bs], c[i:i + bs]) for i in range(0, 2000, bs)]))
    x, c = cloud(300, seed=14)
    out.append(("replay_bs37", P(grid_res=4, leaf_threshold=10, max_depth=6),
                [(x[i:i + 37], c[i:i + 37]) for i in range(0, 300, 37)]))
    x, c = cloud(4000, seed=4)
    out.append(("chunks_c50", P(chunk_capacity=50, grid_res=8, leaf_threshold=20),
                [(x[i:i + 137], c[i:i + 137]) for i in range(0, 4000, 137)]))
    x, c = cloud(4000, seed=3, kind="surface")
    out.append(("surface_253", P(arena_bytes=128 << 20, grid_res=4, leaf_threshold=10, max_depth=8),
                [(x[i:i + 253], c[i:i + 253]) for i in range(0, 4000, 253)]))
    x, c = cloud(20000, seed=21, kind="uniform")
    edgy = np.array([[0.5, 0.5, 0.5], [0.25, 0.5, 0.75], [0.5, 0.0, 0.999], [0.5, 0.25, 0.5]], np.float32)
    x = np.concatenate([x, edgy])
    c = np.concatenate([c, np.arange(4, dtype=np.uint32)])
    out.append(("uniform_g16_c7", P(chunk_capacity=7, grid_res=16, leaf_threshold=100),
                [(x[i:i + 997], c[i:i + 997]) for i in range(0, len(c), 997)]))
    x, c = cloud(12000, seed=22, kind="skew")
    out.append(("skew_g8", P(chunk_capacity=64, grid_res=8, leaf_threshold=40, max_depth=14),
                [(x[i:i + 3000], c[i:i + 3000]) for i in range(0, len(c), 3000)]))
    x, c = cloud(30000, seed=23, kind="surface")
    out.append(("surface_g32_big_batches", P(chunk_capacity=100, grid_res=32, leaf_threshold=500),
                [(x[i:i + 10000], c[i:i + 10000]) for i in range(0, len(c), 10000)]))
    # fatal paths (exception type only)
    x, c = canonical()
    out.append(("spill_overflow", P(grid_res=4, leaf_threshold=2, spill_capacity=1),
                [(x, c), (np.array([[0.15, 0.15, 0.15]], np.float32), np.array([9], np.uint32))]))
    out.append(("backlog_overflow", P(grid_res=4, leaf_threshold=2, backlog_capacity=1), [(x, c)]))
    x, c = cloud(500, seed=24)
    out.append(("out_of_arena", P(arena_bytes=4096, chunk_capacity=16, grid_res=8, leaf_threshold=20), [(x, c)]))
    return out


def run_scenario(mods, params, batches):
    octree, render, store, update, errors = mods
    arena = store.Arena(params["arena_bytes"])
    pool = store.ChunkPool(arena, params["chunk_capacity"])
    tree = octree.Octree(octree.CubeBounds(tuple(params["bmin"]), params["size"]), arena, pool,
                         grid_res=params["grid_res"], leaf_threshold=params["leaf_threshold"],
                         max_depth=params["max_depth"])
    st = update.UpdateState(update.UpdateConfig(backlog_capacity=params["backlog_capacity"],
                                                spill_capacity=params["spill_capacity"]))
    error = ""
    per_batch = []
    for x, c in batches:
        try:
            update.insert_batch(tree, x, c, st)
        except (errors.OutOfArena, errors.SpillOverflow, errors.BacklogOverflow) as e:
            error = type(e).__name__
            break
        per_batch.append([st.stats.voxels_created, st.stats.splits, st.stats.nodes,
                          st.stats.backlog_high_water, st.stats.spill_high_water])
    return tree, st, error, per_batch


def tree_state(tree) -> dict:
    n = tree.num_nodes
    c = tree.pool.allocated_total
    d = {
        "num_nodes": n, "splits_total": tree.splits_total, "max_level": tree.max_level,
        "allocated_total": c, "released_total": tree.pool.released_total,
        "free_count": tree.pool.free_count, "arena_offset": tree.arena.offset,
        "parent": tree.parent[:n].copy(), "octant": tree.octant[:n].copy(), "level": tree.level[:n].copy(),
        "children": tree.children[:n].copy(), "inner": tree.inner[:n].copy(), "final": tree.final[:n].copy(),
        "count": tree.count[:n].copy(), "pending": tree.pending[:n].copy(),
        "chunk_head": tree.chunk_head[:n].copy(), "chunk_tail": tree.chunk_tail[:n].copy(),
        "chunk_count": tree.chunk_count[:n].copy(), "grid_off": tree.grid_off[:n].copy(),
        "bmin": tree.bmin[:n].copy(), "next": tree.pool.next[:c].copy(),
        "occupied": tree.pool.occupied[:c].copy(), "payload_off": tree.pool.payload_off[:c].copy(),
        "free_list": np.asarray(tree.pool._free, np.int32),
    }
    offs = np.zeros(n + 1, np.int64)
    recs = []
    cell_offs = np.zeros(n + 1, np.int64)
    cells = []
    for nid in range(n):
        xyz, rgba = tree.gather_samples(nid)
        r = np.empty((len(rgba), 4), np.float32)
        r[:, :3] = xyz
        r[:, 3] = rgba.view(np.float32)
        recs.append(r)
        offs[nid + 1] = offs[nid] + len(rgba)
        oc = tree.occupied_cells(nid).astype(np.int64) if tree.inner[nid] else np.empty(0, np.int64)
        cells.append(oc)
        cell_offs[nid + 1] = cell_offs[nid] + len(oc)
    d["rec_offsets"] = offs
    d["records"] = np.concatenate(recs) if recs else np.empty((0, 4), np.float32)
    d["cell_offsets"] = cell_offs
    d["cells"] = np.concatenate(cells) if cells else np.empty(0, np.int64)
    return d


RASTER_CAMS = [
    dict(position=(0.5, 0.5, -1.0), target=(0.5, 0.5, 0.5), fov_deg=90.0, near=0.1, far=100.0,
         width=1000, height=1000),
    dict(position=(1.6, 1.2, -0.8), target=(0.5, 0.5, 0.5), fov_deg=70.0, near=0.05, far=50.0,
         width=256, height=256),
    dict(position=(0.4, 0.6, -1.4), target=(0.5, 0.5, 0.5), fov_deg=80.0, near=0.05, far=60.0,
         width=320, height=240),
]


def sparse_fb(cells):
    idx = np.flatnonzero(cells != np.uint64(0xFFFFFFFFFFFFFFFF))
    return idx.astype(np.int64), cells[idx]


DELTA_SCENARIOS = ("canonical", "canonical_1by1", "ten_points_spill", "depth_cap", "chunks_c50", "surface_253",
                   "uniform_g16_c7", "skew_g8", "surface_g32_big_batches", "rebuild_bs333")


def flatten_deltas(deltas) -> dict:
    """BatchDelta list -> flat arrays: structure rows (kind 0 = split, 1 =
    create; node, parent, octant, level), voxel groups (node, count) with the
    concatenated cells / colours, point ranges (node, start, count); *_off
    give each batch's rows."""
    ev, vg, cells, cols, pts = [], [], [], [], []
    off = {"ev": [0], "vg": [0], "vc": [0], "pt": [0]}
    for d in deltas:
        for e in d.structure:
            ev.append([0, e[1], -1, -1, -1] if e[0] == "split" else [1, e[1], e[2], e[3], e[4]])
        for node, c, r in d.voxels:
            vg.append([node, len(c)])
            cells.append(np.asarray(c, np.uint32))
            cols.append(np.asarray(r, np.uint32))
        for node, start, count in d.points:
            pts.append([node, start, count])
        off["ev"].append(len(ev))
        off["vg"].append(len(vg))
        off["vc"].append(sum(len(c) for c in cells))
        off["pt"].append(len(pts))
    out = {
        "events": np.array(ev, np.int64).reshape(-1, 5),
        "vgroups": np.array(vg, np.int64).reshape(-1, 2),
        "vcells": np.concatenate(cells) if cells else np.empty(0, np.uint32),
        "vrgba": np.concatenate(cols) if cols else np.empty(0, np.uint32),
        "points": np.array(pts, np.int64).reshape(-1, 3),
    }
    for k, v in off.items():
        out[k + "_off"] = np.array(v, np.int64)
    return out


def make_deltas(mods) -> None:
    """deltas.npz: the reference's BatchDelta (insert_batch(collect_delta=True),
    update.py:333-355) for every batch of the DELTA_SCENARIOS."""
    octree, render, store, update, errors = mods
    blob = {}
    for name, params, batches in scenarios():
        if name not in DELTA_SCENARIOS:
            continue
        arena = store.Arena(params["arena_bytes"])
        pool = store.ChunkPool(arena, params["chunk_capacity"])
        tree = octree.Octree(octree.CubeBounds(tuple(params["bmin"]), params["size"]), arena, pool,
                             grid_res=params["grid_res"], leaf_threshold=params["leaf_threshold"],
                             max_depth=params["max_depth"])
        st = update.UpdateState(update.UpdateConfig(backlog_capacity=params["backlog_capacity"],
                                                    spill_capacity=params["spill_capacity"]))
        deltas = [update.insert_batch(tree, x, c, st, collect_delta=True) for x, c in batches]
        for k, v in flatten_deltas(deltas).items():
            blob[f"{name}__{k}"] = v
    np.savez_compressed(os.path.join(HERE, "deltas.npz"), **blob)
    print("deltas.npz:", ", ".join(DELTA_SCENARIOS))


def make_morton() -> None:
    """morton.npz: the reference's morton_key / morton_sort (io.py:419-446) on
    clouds with duplicates, boundary and out-of-cube coordinates, several bit
    widths and an offset non-unit root."""
    sys.path.insert(0, REF)
    from lodstream import io as lio
    from lodstream.octree import CubeBounds

    out = {}
    rng = np.random.default_rng(41)
    xyz, rgba = cloud(6000, seed=42)
    dup = xyz[rng.integers(0, len(xyz), 600)]
    edge = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0], [0.5, 0.5, 0.5], [-0.25, 0.5, 1.75], [0.999999, 0.0, 0.5],
                     [np.nextafter(np.float32(1), np.float32(0))] * 3], np.float32)
    x = np.concatenate([xyz, dup, edge]).astype(np.float32)
    c = np.concatenate([rgba, rgba[:600], np.arange(len(edge), dtype=np.uint32)]).astype(np.uint32)
    out["xyz"], out["rgba"] = x, c
    unit = CubeBounds((0.0, 0.0, 0.0), 1.0)
    for bits in (1, 2, 5, 10, 11, 16, 21):
        out[f"keys_b{bits}"] = lio.morton_key(x, unit, bits=bits)
    sx, sr = lio.morton_sort(x, c, unit)
    out["sorted_xyz"], out["sorted_rgba"] = sx, sr
    off = CubeBounds((-3.0, 2.5, 10.0), 6.5)
    xo = (x.astype(np.float64) * 6.5 + np.array([-3.0, 2.5, 10.0])).astype(np.float32)
    out["off_xyz"] = xo
    out["off_keys"] = lio.morton_key(xo, off)
    out["off_sorted_rgba"] = lio.morton_sort(xo, c, off)[1]
    np.savez_compressed(os.path.join(HERE, "morton.npz"), **out)
    print("morton.npz:", len(x), "points")


def main():
    mods = _import_ref()
    if "--only-deltas" in sys.argv:
        make_deltas(mods)
        return
    if "--only-morton" in sys.argv:
        make_morton()
        return
    make_deltas(mods)
    make_morton()
    octree, render, store, update, errors = mods
    manifest = {}
    for name, params, batches in scenarios():
        tree, st, error, per_batch = run_scenario(mods, params, batches)
        blob = {
            "params": np.frombuffer(json.dumps(params).encode(), np.uint8),
            "batch_sizes": np.array([len(c) for _, c in batches], np.int64),
            "xyz": np.concatenate([x for x, _ in batches]).astype(np.float32),
            "rgba": np.concatenate([c for _, c in batches]).astype(np.uint32),
            "error": np.frombuffer(error.encode() or b" ", np.uint8),
            "per_batch": np.array(per_batch, np.int64).reshape(-1, 5),
        }
        if not error:
            for k, v in tree_state(tree).items():
                blob["s_" + k] = np.asarray(v)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **blob)
        manifest[name] = {"nodes": int(tree.num_nodes), "error": error}
    # rasterizer fixtures: brute force + LOD at two thresholds on a tree
    x, c = cloud(5000, seed=31)
    fbs = {}
    for ci, cam_kw in enumerate(RASTER_CAMS):
        cam = render.Camera(**cam_kw)
        fb = render.brute_force_render(x, c, cam)
        fbs[f"brute{ci}_idx"], fbs[f"brute{ci}_val"] = sparse_fb(fb.cells)
        fbs[f"cam{ci}"] = cam.packed()
    arena = store.Arena(64 << 20)
    pool = store.ChunkPool(arena, 1000)
    tree = octree.Octree(octree.CubeBounds((0.0, 0.0, 0.0), 1.0), arena, pool, grid_res=16, leaf_threshold=64,
                         max_depth=12)
    st = update.UpdateState()
    update.insert_batch(tree, x, c, st)
    for ci, cam_kw in enumerate(RASTER_CAMS):
        cam = render.Camera(**cam_kw)
        for thr in (-1.0, 128.0, 20.0):
            fb, rep = render.rasterize(tree, cam, threshold=thr)
            key = f"lod{ci}_{int(thr)}"
            fbs[key + "_idx"], fbs[key + "_val"] = sparse_fb(fb.cells)
            fbs[key + "_sel"] = np.asarray(rep.selected, np.int32)
            fbs[key + "_samples"] = np.array([rep.samples_drawn], np.int64)
    # hand-worked pixel + tie cases (test_render.py:43-83)
    fbs["xyz"], fbs["rgba"] = x, c
    np.savez_compressed(os.path.join(HERE, "raster.npz"), **fbs)
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
        json.dump(manifest, f, indent=1, sort_keys=True)
    print(json.dumps(manifest, indent=1))


if __name__ == "__main__":
    main()
