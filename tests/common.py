"""Test helpers: golden fixtures, oracle / product runners and comparators."""
from __future__ import annotations

import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")

STATE_SCALARS = ("num_nodes", "splits_total", "max_level", "allocated_total", "released_total",
                 "free_count", "arena_offset")
NODE_COLS_ID_FREE = ("parent", "octant", "level", "children", "inner", "final", "count", "pending",
                     "chunk_count", "grid_off", "bmin")
CHUNK_ID_COLS = ("chunk_head", "chunk_tail", "next", "occupied", "payload_off", "free_list")


def golden_names() -> list[str]:
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f not in ("raster.npz", "deltas.npz", "morton.npz"))


def load_golden(name: str) -> dict:
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    d = {k: z[k] for k in z.files}
    d["params"] = json.loads(bytes(d["params"]).decode())
    d["error"] = bytes(d["error"]).decode().strip()
    sizes = d["batch_sizes"]
    offs = np.concatenate([[0], np.cumsum(sizes)])
    d["batches"] = [(d["xyz"][a:b], d["rgba"][a:b]) for a, b in zip(offs[:-1], offs[1:])]
    d["state"] = {k[2:]: v for k, v in d.items() if k.startswith("s_")}
    return d


def load_raster() -> dict:
    z = np.load(os.path.join(GOLDEN, "raster.npz"))
    return {k: z[k] for k in z.files}


DELTA_KEYS = ("events", "vgroups", "vcells", "vrgba", "points", "ev_off", "vg_off", "vc_off", "pt_off")


def delta_names() -> list[str]:
    z = np.load(os.path.join(GOLDEN, "deltas.npz"))
    return sorted({k.split("__")[0] for k in z.files})


def load_deltas(name: str) -> dict:
    """The reference's BatchDelta of every batch of a scenario (make_golden.make_deltas)."""
    z = np.load(os.path.join(GOLDEN, "deltas.npz"))
    return {k: z[f"{name}__{k}"] for k in DELTA_KEYS}


def flatten_deltas(deltas) -> dict:
    """[(structure, voxels, points)] or [BatchDelta] -> the deltas.npz layout."""
    ev, vg, cells, cols, pts = [], [], [], [], []
    off = {"ev": [0], "vg": [0], "vc": [0], "pt": [0]}
    nvc = 0
    for d in deltas:
        structure, voxels, points = (d.structure, d.voxels, d.points) if hasattr(d, "structure") else d
        for e in structure:
            ev.append([0, e[1], -1, -1, -1] if e[0] == "split" else [1, e[1], e[2], e[3], e[4]])
        for node, c, r in voxels:
            assert np.asarray(c).dtype == np.uint32 and np.asarray(r).dtype == np.uint32
            vg.append([node, len(c)])
            cells.append(np.asarray(c, np.uint32))
            cols.append(np.asarray(r, np.uint32))
            nvc += len(c)
        for node, start, count in points:
            pts.append([node, start, count])
        off["ev"].append(len(ev))
        off["vg"].append(len(vg))
        off["vc"].append(nvc)
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


def assert_same_deltas(got: dict, want: dict, what: str = "") -> None:
    for k in DELTA_KEYS:
        assert np.array_equal(np.asarray(got[k]), np.asarray(want[k])), f"{what}: delta {k} differs"


def dense_fb(idx, val, n):
    fb = np.full(n, np.uint64(0xFFFFFFFFFFFFFFFF))
    fb[idx] = val
    return fb


# -- oracle ----------------------------------------------------------------------------


def run_oracle(params: dict, batches):
    import oracle

    t = oracle.OracleTree(
        params["bmin"], params["size"], grid_res=params["grid_res"], leaf_threshold=params["leaf_threshold"],
        max_depth=params["max_depth"], chunk_capacity=params["chunk_capacity"],
        arena_bytes=params["arena_bytes"], backlog_capacity=params["backlog_capacity"],
        spill_capacity=params["spill_capacity"],
    )
    error = ""
    per_batch = []
    hw_b = hw_s = 0
    for x, c in batches:
        try:
            s = t.insert_batch(x, c)
        except oracle.OracleError as e:
            error = e.kind
            break
        hw_b, hw_s = max(hw_b, s["n_voxels"]), max(hw_s, s["n_spill"])
        st = t.state()
        per_batch.append([t.voxels_created, st["splits_total"], st["num_nodes"], hw_b, hw_s])
    return t, error, per_batch


def oracle_state(t) -> dict:
    d = t.state()
    n = d["num_nodes"]
    offs = np.zeros(n + 1, np.int64)
    recs, cells = [], []
    cell_offs = np.zeros(n + 1, np.int64)
    for nid in range(n):
        xyz, rgba = t.gather_samples(nid)
        r = np.empty((len(rgba), 4), np.float32)
        r[:, :3] = xyz
        r[:, 3] = rgba.view(np.float32)
        recs.append(r)
        offs[nid + 1] = offs[nid] + len(rgba)
        oc = t.occupied_cells(nid).astype(np.int64) if d["inner"][nid] else np.empty(0, np.int64)
        cells.append(oc)
        cell_offs[nid + 1] = cell_offs[nid] + len(oc)
    d["rec_offsets"] = offs
    d["records"] = np.concatenate(recs) if recs else np.empty((0, 4), np.float32)
    d["cell_offsets"] = cell_offs
    d["cells"] = np.concatenate(cells) if cells else np.empty(0, np.int64)
    return d


# -- product ---------------------------------------------------------------------------


def make_product(params: dict, device: int = 0):
    from paper_2310_03567_b200 import Arena, ChunkPool, CubeBounds, Octree, UpdateConfig, UpdateState

    arena = Arena(params["arena_bytes"])
    pool = ChunkPool(arena, params["chunk_capacity"])
    tree = Octree(CubeBounds(tuple(params["bmin"]), params["size"]), arena, pool, grid_res=params["grid_res"],
                  leaf_threshold=params["leaf_threshold"], max_depth=params["max_depth"], device=device)
    state = UpdateState(UpdateConfig(backlog_capacity=params["backlog_capacity"],
                                     spill_capacity=params["spill_capacity"]))
    return tree, state


def run_product(params: dict, batches):
    from paper_2310_03567_b200 import BacklogOverflow, OutOfArena, SpillOverflow, insert_batch

    tree, state = make_product(params)
    error = ""
    per_batch = []
    for x, c in batches:
        try:
            insert_batch(tree, x, c, state)
        except (OutOfArena, SpillOverflow, BacklogOverflow) as e:
            error = type(e).__name__
            break
        s = state.stats
        per_batch.append([s.voxels_created, s.splits, s.nodes, s.backlog_high_water, s.spill_high_water])
    return tree, state, error, per_batch


def product_state(tree) -> dict:
    n = tree.num_nodes
    d = {
        "num_nodes": n, "splits_total": tree.splits_total, "max_level": tree.max_level,
        "allocated_total": tree.pool.allocated_total, "released_total": tree.pool.released_total,
        "free_count": tree.pool.free_count, "arena_offset": tree.arena.offset,
    }
    for k in NODE_COLS_ID_FREE + ("chunk_head", "chunk_tail"):
        d[k] = getattr(tree, k)[:n].copy()
    c = d["allocated_total"]
    for k in ("next", "occupied", "payload_off"):
        d[k] = getattr(tree.pool, k)[:c].copy()
    d["free_list"] = tree.pool.free_list.copy()
    offs, rec = tree.dump_records()
    d["rec_offsets"], d["records"] = offs, rec
    cells, cell_offs = [], np.zeros(n + 1, np.int64)
    for nid in range(n):
        oc = tree.occupied_cells(nid).astype(np.int64) if d["inner"][nid] else np.empty(0, np.int64)
        cells.append(oc)
        cell_offs[nid + 1] = cell_offs[nid] + len(oc)
    d["cell_offsets"] = cell_offs
    d["cells"] = np.concatenate(cells) if cells else np.empty(0, np.int64)
    return d


def assert_same_state(got: dict, want: dict, *, chunk_ids: bool, label: str = "") -> None:
    """Bit-exact comparison of two observable tree states.

    ``chunk_ids=False`` skips the columns that name chunk ids / payload offsets
    (their assignment order is an implementation detail: SURVEY 8(a) item 4);
    counts of chunks, arena growth, free-list length and every node's sample
    sequence are always compared.
    """
    for k in STATE_SCALARS:
        assert int(got[k]) == int(want[k]), f"{label}: {k} {got[k]} != {want[k]}"
    n = int(want["num_nodes"])
    cols = NODE_COLS_ID_FREE + (CHUNK_ID_COLS if chunk_ids else ())
    for k in cols:
        a, b = np.asarray(got[k]), np.asarray(want[k])
        if k in ("chunk_head", "chunk_tail") or k in NODE_COLS_ID_FREE:
            a, b = a[:n], b[:n]
        assert a.shape == b.shape, f"{label}: {k} shape {a.shape} != {b.shape}"
        if k == "bmin":
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), f"{label}: bmin bits differ"
        else:
            if not np.array_equal(a, b):
                diff = np.flatnonzero((a != b).reshape(len(a), -1).any(axis=1)) if a.size else []
                raise AssertionError(f"{label}: {k} differs at rows {list(diff[:8])}")
    assert np.array_equal(got["rec_offsets"], want["rec_offsets"]), f"{label}: per-node counts differ"
    ra = np.ascontiguousarray(got["records"]).view(np.uint32)
    rb = np.ascontiguousarray(want["records"]).view(np.uint32)
    if not np.array_equal(ra, rb):
        bad = np.flatnonzero((ra != rb).any(axis=1))
        node = int(np.searchsorted(want["rec_offsets"], bad[0], side="right") - 1)
        raise AssertionError(f"{label}: {len(bad)} sample records differ, first at node {node}")
    assert np.array_equal(got["cell_offsets"], want["cell_offsets"]), f"{label}: bitgrid popcounts differ"
    assert np.array_equal(got["cells"], want["cells"]), f"{label}: occupied cells differ"


# -- multi-GPU protocol, emulated on one GPU -------------------------------------------


def emulate_partitioned(params: dict, batches, plan, merge: bool = True):
    """The warm-up / hand-off / partitioned protocol (multigpu.py) with
    len(plan.load) ranks as trees on one GPU: every batch goes into the single
    tree `g`; rank 0 takes whole batches until the top is inner, its packed
    state is unpacked into the other ranks; later batches are routed by exact
    octant prefix (partition.take: global order within a rank) and, with
    `merge`, the top-node voxels of every batch are merged across ranks by the
    winners' global indices (multigpu.merge_top_voxels).  Returns
    (g, ranks [(tree, state)], handed_off_at)."""
    from paper_2310_03567_b200 import insert_batch, multigpu, partition

    world = len(plan.load)
    g, gs = make_product(params)
    ranks = [make_product(params) for _ in range(world)]
    handed = None
    for bi, (x, c) in enumerate(batches):
        insert_batch(g, x, c, gs)
        if handed is None:
            insert_batch(ranks[0][0], x, c, ranks[0][1])
            if multigpu.top_is_inner(ranks[0][0], plan.depth):
                buf = multigpu.pack_tree(ranks[0][0])
                for r in range(1, world):
                    multigpu.unpack_tree(ranks[r][0], buf)
                handed = bi
            continue
        owner = plan.owner[partition.prefix_of(x, plan.depth, params["bmin"], params["size"])]
        everyone, own_nodes = [], []
        for r in range(world):
            pos = np.flatnonzero(owner == r)
            if len(pos):
                insert_batch(ranks[r][0], np.ascontiguousarray(x[pos]), np.ascontiguousarray(c[pos]), ranks[r][1])
                node, cell, rgba, win = multigpu.last_top_voxels(ranks[r][0], plan.depth)
                everyone.append((node, cell, rgba, pos[win]))
                own_nodes.append(node)
            else:
                everyone.append((np.empty(0, np.int32),) * 2 + (np.empty(0, np.uint32), np.empty(0, np.int64)))
                own_nodes.append(np.empty(0, np.int32))
        if merge:
            for r in range(world):
                multigpu.merge_top_voxels(ranks[r][0], own_nodes[r], everyone)
    return g, ranks, handed


def assert_union_equals_single(g, ranks, plan, label: str = "") -> int:
    """Node for node, by octant path: prefix subtrees on their owner, and the
    replicated top nodes on EVERY rank, equal the single tree (kind, sample
    sequence, occupied cells).  Returns the nodes compared."""
    from oracle.rebuild import tree_paths

    gp = tree_paths(g.inner, g.children)
    g_off, g_rec = g.dump_records()
    rp = [tree_paths(t.inner, t.children) for t, _ in ranks]
    dumps = [t.dump_records() for t, _ in ranks]
    checked = 0
    for path, nid in gp.items():
        if len(path) < plan.depth:
            holders = range(len(ranks))
        else:
            prefix = 0
            for o in path[:plan.depth]:
                prefix = prefix * 8 + o
            holders = [int(plan.owner[prefix])]
        want = g_rec[g_off[nid]:g_off[nid + 1]].view(np.uint32)
        for r in holders:
            t = ranks[r][0]
            assert path in rp[r], f"{label}: rank {r} lacks {path}"
            rid = rp[r][path]
            assert bool(t.inner[rid]) == bool(g.inner[nid]), f"{label}: kind at {path} on rank {r}"
            ro, rr = dumps[r]
            got = rr[ro[rid]:ro[rid + 1]].view(np.uint32)
            assert got.shape == want.shape and np.array_equal(got, want), f"{label}: samples at {path} on rank {r}"
            if g.inner[nid]:
                assert np.array_equal(t.occupied_cells(rid), g.occupied_cells(nid)), f"{label}: cells {path} r{r}"
            checked += 1
    return checked
