"""Octree facade over the device-resident node table (reference: lodstream/octree.py).

Geometry conventions are the reference's (octree.py:1-24): cubic root, octant
bit 0 = x, 1 = y, 2 = z, set when the coordinate is >= the node centre; child
bounds ``min + half * offset`` in float64; cells ``floor(g * (p - min) / size)``
clamped, linearised ``cx + g*cy + g*g*cz``; voxels at cell centres.

Storage is the B200 layout: the node table is a struct-of-arrays
in HBM with the same column types and shapes as the reference's numpy columns
(octree.py:169-182), mutated only by the update kernels.  The attributes below
(``count``, ``inner``, ``children``, ...) are host mirrors refreshed lazily
from the device after each update (one D2H of the live rows), so callers and
tests read them exactly like the reference's arrays.  Writing into a mirror
does not change the tree.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .store import NO_CHUNK, Arena, ChunkPool

NO_NODE = -1
POINT_DTYPE = np.dtype(
    [("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("r", "u1"), ("g", "u1"), ("b", "u1"), ("a", "u1")]
)


@dataclass(frozen=True)
class CubeBounds:
    """Axis-aligned cube: minimum corner and edge length (octree.py:39-72)."""

    min: tuple[float, float, float]
    size: float

    @property
    def center(self) -> tuple[float, float, float]:
        h = self.size * 0.5
        return (self.min[0] + h, self.min[1] + h, self.min[2] + h)

    def child(self, octant: int) -> "CubeBounds":
        h = self.size * 0.5
        return CubeBounds(
            (
                self.min[0] + (h if octant & 1 else 0.0),
                self.min[1] + (h if octant & 2 else 0.0),
                self.min[2] + (h if octant & 4 else 0.0),
            ),
            h,
        )

    def contains(self, p) -> bool:
        return all(self.min[i] <= p[i] <= self.min[i] + self.size for i in range(3))

    def corners(self) -> np.ndarray:
        """(8, 3) float64 corners; corner i sits at octant offset i."""
        bits = np.arange(8)
        out = np.empty((8, 3), dtype=np.float64)
        for axis in range(3):
            on = (bits >> axis) & 1
            out[:, axis] = np.where(on == 1, self.min[axis] + self.size, self.min[axis] + 0.0)
        return out


def cubify(mins, maxs) -> CubeBounds:
    """Smallest cube covering an AABB, centred on it along the short axes (octree.py:75-85)."""
    lo_in = np.asarray(mins, dtype=np.float64)
    hi_in = np.asarray(maxs, dtype=np.float64)
    extent = hi_in - lo_in
    size = float(extent.max())
    if size <= 0.0:
        size = 1.0
    lo = lo_in - (size - extent) * 0.5
    return CubeBounds((float(lo[0]), float(lo[1]), float(lo[2])), size)


def octant_of(p, bounds: CubeBounds) -> int:
    """Routing octant; points on a split plane go to the upper child (octree.py:88-98)."""
    c = bounds.center
    return int(p[0] >= c[0]) | int(p[1] >= c[1]) << 1 | int(p[2] >= c[2]) << 2


def cell_of(p, bounds: CubeBounds, g: int) -> int:
    """Clamped linear grid cell (octree.py:101-107)."""
    out = 0
    for axis, mul in ((0, 1), (1, g), (2, g * g)):
        c = int(np.floor(g * (float(p[axis]) - bounds.min[axis]) / bounds.size))
        out += mul * min(max(c, 0), g - 1)
    return out


def cell_coords(cell: int, g: int) -> tuple[int, int, int]:
    return cell % g, (cell // g) % g, cell // (g * g)


def voxel_center(cell: int, bounds: CubeBounds, g: int) -> np.ndarray:
    """float64 centre of a cell (octree.py:114-125)."""
    step = bounds.size / g
    idx = cell_coords(cell, g)
    return np.array([bounds.min[a] + (idx[a] + 0.5) * step for a in range(3)], dtype=np.float64)


def pack_rgba(r: int, g: int, b: int, a: int = 255) -> int:
    return (r & 0xFF) | (g & 0xFF) << 8 | (b & 0xFF) << 16 | (a & 0xFF) << 24


_DUMP_CACHE_MAX = 8 << 20    # samples: trees up to 128 MB of records are read back whole for gathers
_ARENA_CACHE_MAX = 128 << 20  # bytes: arenas up to this much in use are read back whole for grids

_NODE_COLS = (
    # name, dtype, per-row shape, fill beyond the live rows (octree.py:169-182)
    ("parent", np.int32, (), NO_NODE),
    ("octant", np.uint8, (), 0),
    ("level", np.int32, (), 0),
    ("children", np.int32, (8,), NO_NODE),
    ("inner", np.bool_, (), False),
    ("final", np.bool_, (), False),
    ("count", np.int64, (), 0),
    ("pending", np.int64, (), 0),
    ("chunk_head", np.int32, (), NO_CHUNK),
    ("chunk_tail", np.int32, (), NO_CHUNK),
    ("chunk_count", np.int32, (), 0),
    ("grid_off", np.int64, (), -1),
    ("bmin", np.float64, (3,), 0.0),
)


class Octree:
    """Device-resident octree with the reference's constructor and accessors."""

    def __init__(
        self,
        bounds: CubeBounds,
        arena: Arena,
        pool: ChunkPool,
        *,
        grid_res: int = 128,
        leaf_threshold: int = 50000,
        max_depth: int = 20,
        device: int = 0,
    ) -> None:
        if grid_res < 2 or grid_res & 1:
            raise ValueError("grid_res must be even, so the bitgrid is whole bytes")
        if pool.arena is not arena:
            raise ValueError("the chunk pool must draw from the same arena")
        L = _lib.require_device(device)
        self.bounds = bounds
        self.arena = arena
        self.pool = pool
        self.grid_res = grid_res
        self.grid_bytes = grid_res ** 3 // 8
        self.leaf_threshold = leaf_threshold
        self.max_depth = max_depth
        self.device = device
        self.size_by_level = bounds.size * 0.5 ** np.arange(max_depth + 2)
        p = _lib.LodParams()
        p.bmin[0], p.bmin[1], p.bmin[2] = (float(v) for v in bounds.min)
        p.size = float(bounds.size)
        p.grid_res, p.leaf_threshold, p.max_depth = grid_res, leaf_threshold, max_depth
        p.chunk_capacity = pool.capacity
        p.arena_bytes = arena.capacity
        p.device = device
        h = ctypes.c_void_p()
        _lib.check(L.lod_tree_create(ctypes.byref(p), ctypes.byref(h)), "lod_tree_create")
        self._h = h
        self._L = L
        arena._bind(self)
        pool._bind(self)
        self._gen = 0
        self._cache: dict = {}
        self._arena_edits: list = []  # (offset, host copy handed out, snapshot) of pool.records() views

    # -- lifetime -----------------------------------------------------------------
    def close(self) -> None:
        h = getattr(self, "_h", None)
        if h:
            self._L.lod_tree_destroy(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> ctypes.c_void_p:
        """The C handle; host edits of the mirrors reach the device first."""
        if self._cache or self._arena_edits:
            self._sync_edits()
        return self._h

    def _invalidate(self) -> None:
        self._gen += 1
        self._cache.clear()
        self._arena_edits.clear()  # payload copies handed out before a device update are detached

    def _sync_edits(self) -> None:
        """Write host edits of the mirrored columns back to the device.

        Callers may edit ``tree.count``, ``pool.occupied``, the arrays
        ``pool.records(cid)`` returned, ... in place, as the reference's unit
        tests do with its numpy-backed tree; the mirrors are compared with
        the snapshot taken when they were read, and changed columns are
        written back (lod_write_nodes / lod_write_pool / lod_write_arena,
        which rebuild the device-only indexes) before the next device call."""
        c = self._cache
        if "cols" in c:
            cols, snap = c["cols"], c["cols_snap"]
            n = len(snap["count"])
            changed = {k for k in snap if not np.array_equal(cols[k][:n], snap[k])}
            if changed:
                keep = [np.ascontiguousarray(cols[k][:n]) if k in changed else None for k, *_ in _NODE_COLS]
                _lib.check(self._L.lod_write_nodes(self._h, n, *(_lib.ptr(a) for a in keep)), "lod_write_nodes")
                for k in changed:
                    snap[k] = cols[k][:n].copy()
                c.pop("info", None)
                c["_edited"] = True
        if "pool" in c:
            pc, snap = c["pool"], c["pool_snap"]
            n = len(snap["occupied"])
            changed = {k for k in snap if not np.array_equal(pc[k][:n], snap[k])}
            if changed:
                args = [np.ascontiguousarray(pc[k][:n]) if k in changed else None
                        for k in ("next", "payload_off", "occupied")]
                _lib.check(self._L.lod_write_pool(self._h, n, *(_lib.ptr(a) for a in args)), "lod_write_pool")
                for k in changed:
                    snap[k] = pc[k][:n].copy()
                c["_edited"] = True
        wrote = False
        for off, raw, snap in self._arena_edits:
            if not np.array_equal(raw, snap):
                _lib.check(self._L.lod_write_arena(self._h, off, raw.nbytes, _lib.ptr(raw)), "lod_write_arena")
                snap[...] = raw
                wrote = True
        if wrote or c.pop("_edited", False):
            for k in ("dump", "dump_gen", "arena", "arena_gen"):
                c.pop(k, None)


    # -- mirrors ----------------------------------------------------------------------
    def _info(self) -> _lib.LodTreeInfo:
        if "info" not in self._cache:
            info = _lib.LodTreeInfo()
            _lib.check(self._L.lod_tree_info(self._h, ctypes.byref(info)), "lod_tree_info")
            self._cache["info"] = info
        return self._cache["info"]

    def _cols(self) -> dict:
        if "cols" not in self._cache:
            n = int(self._info().num_nodes)
            cap = max(1024, 1 << max(n - 1, 1).bit_length())
            cols = {}
            for name, dt, shape, fill in _NODE_COLS:
                cols[name] = np.full((cap,) + shape, fill, dtype=dt)
            args = [_lib.ptr(cols[name]) for name, *_ in _NODE_COLS]
            _lib.check(self._L.lod_read_nodes(self._h, n, *args), "lod_read_nodes")
            self._cache["cols"] = cols
            self._cache["cols_snap"] = {name: cols[name][:n].copy() for name, *_ in _NODE_COLS}
        return self._cache["cols"]

    def _pool_cols(self) -> dict:
        if "pool" not in self._cache:
            info = self._info()
            n, nf = int(info.allocated_total), int(info.free_count)
            cap = max(1024, 1 << max(n - 1, 1).bit_length())
            nxt = np.full(cap, NO_CHUNK, np.int32)
            poff = np.zeros(cap, np.int64)
            occ = np.zeros(cap, np.int32)
            free = np.zeros(nf, np.int32)
            _lib.check(self._L.lod_read_pool(self._h, n, _lib.ptr(nxt), _lib.ptr(poff), _lib.ptr(occ),
                                             _lib.ptr(free), nf), "lod_read_pool")
            self._cache["pool"] = {"next": nxt, "payload_off": poff, "occupied": occ, "free_list": free}
            self._cache["pool_snap"] = {"next": nxt[:n].copy(), "payload_off": poff[:n].copy(),
                                        "occupied": occ[:n].copy()}
        return self._cache["pool"]

    def _arena_bytes(self, off: int, size: int) -> np.ndarray:
        out = np.empty(size, np.uint8)
        if size:
            _lib.check(self._L.lod_read_arena(self.handle, off, size, _lib.ptr(out)), "lod_read_arena")
        return out

    def _live_chunks(self) -> int:
        n = self.num_nodes
        return int(self.chunk_count[:n].sum())

    num_nodes = property(lambda self: int(self._info().num_nodes))
    splits_total = property(lambda self: int(self._info().splits_total))
    max_level = property(lambda self: int(self._info().max_level))
    parent = property(lambda self: self._cols()["parent"])
    octant = property(lambda self: self._cols()["octant"])
    level = property(lambda self: self._cols()["level"])
    children = property(lambda self: self._cols()["children"])
    inner = property(lambda self: self._cols()["inner"])
    final = property(lambda self: self._cols()["final"])
    count = property(lambda self: self._cols()["count"])
    pending = property(lambda self: self._cols()["pending"])
    chunk_head = property(lambda self: self._cols()["chunk_head"])
    chunk_tail = property(lambda self: self._cols()["chunk_tail"])
    chunk_count = property(lambda self: self._cols()["chunk_count"])
    grid_off = property(lambda self: self._cols()["grid_off"])
    bmin = property(lambda self: self._cols()["bmin"])

    # -- per-node access ---------------------------------------------------------------
    def node_size(self, nid: int) -> float:
        return self.bounds.size * (0.5 ** int(self.level[nid]))

    def node_bounds(self, nid: int) -> CubeBounds:
        b = self.bmin[nid]
        return CubeBounds((float(b[0]), float(b[1]), float(b[2])), self.node_size(nid))

    def grid(self, nid: int) -> np.ndarray:
        """Copy of an inner node's occupancy bitgrid bytes (octree.py:275-279)."""
        off = int(self.grid_off[nid])
        assert off >= 0, "leaf nodes have no grid"
        cached = self._cached_arena()
        if cached is not None:
            return cached[off: off + self.grid_bytes].copy()
        return self._arena_bytes(off, self.grid_bytes)

    def grid_popcount(self, nid: int) -> int:
        return int(np.unpackbits(self.grid(nid), bitorder="little").sum())

    def occupied_cells(self, nid: int) -> np.ndarray:
        """Sorted linear cells with their bit set (octree.py:293-296)."""
        return np.nonzero(np.unpackbits(self.grid(nid), bitorder="little"))[0]

    def gather_samples(self, nid: int, start: int = 0) -> tuple[np.ndarray, np.ndarray]:
        """Samples [start, count) in storage (= insertion) order (octree.py:298-326).

        Trees up to _DUMP_CACHE_MAX samples are read back whole once per
        update (lod_dump_records) and served from that copy, so walking every
        node (as the reference's oracles do) costs one device round trip,
        not one per node."""
        total = int(self.count[nid])
        k = max(total - start, 0)
        if k and self._cached_dump() is not None:
            off, rec = self._cache["dump"]
            r = rec[off[nid] + start: off[nid + 1]]
            return np.ascontiguousarray(r[:, :3]), r[:, 3].view(np.uint32).copy()
        xyz = np.empty((k, 3), dtype=np.float32)
        rgba = np.empty(k, dtype=np.uint32)
        if k:
            _lib.check(self._L.lod_gather(self.handle, nid, start, _lib.ptr(xyz), _lib.ptr(rgba)), "lod_gather")
        return xyz, rgba

    def _cached_dump(self):
        if self._cache.get("dump_gen") != self._gen:
            n = self.num_nodes
            total = int(self.count[:n].sum())
            self._cache["dump"] = self.dump_records() if total <= _DUMP_CACHE_MAX else None
            self._cache["dump_gen"] = self._gen
        return self._cache["dump"]

    def _cached_arena(self):
        """The used arena bytes (grids and payloads), one read per update, for small trees."""
        if self._cache.get("arena_gen") != self._gen:
            used = self.arena.offset
            self._cache["arena"] = self._arena_bytes(0, used) if used <= _ARENA_CACHE_MAX else None
            self._cache["arena_gen"] = self._gen
        return self._cache["arena"]

    def chunk_directory(self) -> list[np.ndarray]:
        """Every node's chunk ids in list order as the device directory holds
        them (the spill gather and the render read chunks through it)."""
        n = self.num_nodes
        top = ctypes.c_uint64(0)
        _lib.check(self._L.lod_read_directory(self._h, 0, None, None, None, 0, ctypes.byref(top)), "directory")
        off, cap = np.zeros(n, np.int64), np.zeros(n, np.int32)
        cdir = np.zeros(max(int(top.value), 1), np.int32)
        _lib.check(self._L.lod_read_directory(self._h, n, _lib.ptr(off), _lib.ptr(cap), _lib.ptr(cdir), len(cdir),
                                              ctypes.byref(top)), "directory")
        cc = self.chunk_count[:n]
        assert np.all(cc <= cap), "directory region smaller than the chunk list"
        return [cdir[off[i]:off[i] + cc[i]] for i in range(n)]

    def dump_records(self) -> tuple[np.ndarray, np.ndarray]:
        """All samples packed by node id: (offsets (n+1,), records (total, 4) as f32 view)."""
        n = self.num_nodes
        offsets = np.zeros(n + 1, np.int64)
        _lib.check(self._L.lod_dump_records(self.handle, n, _lib.ptr(offsets), None), "lod_dump_records")
        rec = np.empty((int(offsets[-1]), 4), np.float32)
        _lib.check(self._L.lod_dump_records(self._h, n, _lib.ptr(offsets), _lib.ptr(rec)), "lod_dump_records")
        return offsets, rec

    # -- structure outside the update cycle -------------------------------------------
    def split(self, nid: int, spill) -> list[int]:
        """Turn a leaf into an inner node with 8 fresh leaf children
        (octree.py:222-264): stored samples go to ``spill`` in storage order
        (SpillOverflow past its capacity), the chunks back to the pool in walk
        order, the node gets a zeroed grid (OutOfArena past the arena).  The
        device kernel is the same split the update cycle performs."""
        assert not self.inner[nid], "split target must be a leaf"
        assert self.level[nid] < self.max_depth, "cannot split at max depth"
        if int(self.count[nid]):
            xyz, rgba = self.gather_samples(nid)
            spill.append(xyz, rgba)
        first = ctypes.c_int32(0)
        rc = self._L.lod_split_node(self.handle, nid, ctypes.byref(first))
        self._invalidate()
        _lib.check(rc, "split")
        return list(range(first.value, first.value + 8))

    def append_chunk(self, nid: int) -> int:
        """Link one freshly acquired chunk at the tail of a node's list
        (octree.py:328-337; LIFO reuse before the arena, store.py:110-123)."""
        cid = ctypes.c_int32(0)
        rc = self._L.lod_append_chunk(self.handle, nid, ctypes.byref(cid))
        self._invalidate()
        _lib.check(rc, "append_chunk")
        return int(cid.value)

    def grid_test_and_set(self, nid: int, cell: int) -> bool:
        """Set a cell bit; True when the cell was previously empty (octree.py:281-288)."""
        assert int(self.grid_off[nid]) >= 0, "leaf nodes have no grid"
        was = ctypes.c_int32(0)
        rc = self._L.lod_grid_test_and_set(self.handle, nid, int(cell), ctypes.byref(was))
        self._invalidate()
        _lib.check(rc, "grid_test_and_set")
        return bool(was.value)

    # -- whole-tree helpers (octree.py:341-377) ---------------------------------------
    def leaves(self) -> np.ndarray:
        return np.nonzero(~self.inner[: self.num_nodes])[0]

    def inner_nodes(self) -> np.ndarray:
        return np.nonzero(self.inner[: self.num_nodes])[0]

    def total_points(self) -> int:
        n = self.num_nodes
        return int(self.count[:n][~self.inner[:n]].sum())

    def total_voxels(self) -> int:
        n = self.num_nodes
        return int(self.count[:n][self.inner[:n]].sum())

    def validate(self) -> None:
        """Structural consistency sweep (octree.py:355-377); raises AssertionError."""
        n = self.num_nodes
        cap = self.pool.capacity
        count, ccount, head = self.count, self.chunk_count, self.chunk_head
        inner, children, grid_off = self.inner, self.children, self.grid_off
        nxt, occ = self.pool.next, self.pool.occupied
        dirs = self.chunk_directory()  # device-only index of every chunk list (B200 extra)
        for nid in range(n):
            cnt = int(count[nid])
            want = (cnt + cap - 1) // cap
            assert ccount[nid] == want, (nid, cnt, int(ccount[nid]))
            walked = []
            cid = int(head[nid])
            seen = cnt
            while cid != NO_CHUNK:
                walked.append(cid)
                got = int(occ[cid])
                assert got == min(seen, cap), (nid, cid, got)
                seen -= got
                cid = int(nxt[cid])
            assert len(walked) == want
            assert walked == dirs[nid].tolist(), (nid, "chunk directory differs from the list")
            if inner[nid]:
                assert all(children[nid, o] != NO_NODE for o in range(8))
                assert self.grid_popcount(nid) == cnt, (nid, cnt)
            else:
                assert grid_off[nid] == -1
                assert all(children[nid, o] == NO_NODE for o in range(8))
        self.pool.check_ledger()
