"""lodstream/_b200.py -- the binding a `lodstream` maintainer would add.

Self-contained ctypes binding of the C ABI in ``include/lod_b200.h``
(``paper_2310_03567_b200/_lodb200.so``): only ``ctypes`` and ``numpy``, no
import of the facade package.  It replaces the orchestration entry points of
the reference's hot path:

* ``update.insert_batch``      (update.py:252-393)  -> :func:`insert_batch`
* ``update.run_frame_updates`` (update.py:396-417)  -> :func:`prefetch` before each insert
* ``render.rasterize``         (render.py:213-225)  -> :func:`rasterize`
* ``render.brute_force_render`` (render.py:228-239) -> :func:`brute_force_render`
* ``Octree.gather_samples``    (octree.py:298-326)  -> :func:`gather`
* node-table mirrors           (octree.py:169-182)  -> :func:`read_nodes`

The structure layouts below are checked against the C header by
``tests/test_integration.py`` (compiled ``offsetof`` / ``sizeof`` of every
field), so this file cannot drift from ``include/lod_b200.h`` silently.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_DEFAULT_LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2310_03567_b200",
                            "_lodb200.so")

# status codes (lod_b200.h) -> the reference's exception names (errors.py:10-19)
LOD_OK = 0
ERRORS = {1: "OutOfArena", 2: "SpillOverflow", 3: "BacklogOverflow"}
# flags
FLAG_DEVICE_INPUT, FLAG_DEVICE_FB, FLAG_PROFILE, FLAG_DELTA = 1, 2, 4, 8
FLAG_PACKED, FLAG_INPUT_STREAM, FLAG_FB_CLEAR = 16, 32, 64
NPHASE = 10


class LodParams(ctypes.Structure):
    _fields_ = [("bmin", ctypes.c_double * 3), ("size", ctypes.c_double),
                ("grid_res", ctypes.c_int64), ("leaf_threshold", ctypes.c_int64),
                ("max_depth", ctypes.c_int64), ("chunk_capacity", ctypes.c_int64),
                ("arena_bytes", ctypes.c_uint64), ("device", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class LodLimits(ctypes.Structure):
    _fields_ = [("backlog_capacity", ctypes.c_int64), ("spill_capacity", ctypes.c_int64),
                ("input_stream", ctypes.c_void_p)]  # with FLAG_INPUT_STREAM, for device inputs


class LodBatchStats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in (
        "n_batch", "n_spill", "n_voxels", "n_splits", "iterations", "num_nodes",
        "splits_total", "max_level", "allocated_total", "free_count", "released_total")] + [
        ("arena_offset", ctypes.c_uint64), ("launches", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
        ("device_ms", ctypes.c_float), ("device_ms_prev", ctypes.c_float),
        ("phase_ms", ctypes.c_float * NPHASE)]


class LodTreeInfo(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in (
        "num_nodes", "node_capacity", "splits_total", "max_level", "allocated_total", "free_count",
        "released_total", "chunk_capacity_rows")] + [
        ("arena_offset", ctypes.c_uint64), ("arena_capacity", ctypes.c_uint64),
        ("grid_bytes", ctypes.c_int64), ("chunk_capacity", ctypes.c_int64)]


class LodDeltaInfo(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in ("n_splits", "n_voxel_groups", "n_voxels", "n_point_groups")]


class LodSettleStats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in ("calls", "n_voxels", "n_voxels_max", "n_spill_max", "n_splits",
                                              "num_nodes", "splits_total", "max_level")] + [
        ("device_ms", ctypes.c_float), ("error", ctypes.c_int32)]


STRUCTS = (LodParams, LodLimits, LodBatchStats, LodTreeInfo, LodDeltaInfo, LodSettleStats)

_P, _I64 = ctypes.c_void_p, ctypes.c_int64
_SIGS = {
    "lod_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "lod_tree_create": (ctypes.c_int, [ctypes.POINTER(LodParams), ctypes.POINTER(_P)]),
    "lod_tree_destroy": (ctypes.c_int, [_P]),
    "lod_tree_info": (ctypes.c_int, [_P, ctypes.POINTER(LodTreeInfo)]),
    "lod_insert_batch": (ctypes.c_int, [_P, _P, _P, _I64, ctypes.POINTER(LodLimits), ctypes.c_int,
                                        ctypes.POINTER(LodBatchStats)]),
    "lod_tree_wait": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_float)]),
    "lod_tree_settle": (ctypes.c_int, [_P, ctypes.POINTER(LodSettleStats)]),
    "lod_prefetch_batch": (ctypes.c_int, [_P, _P, _P, _I64]),
    "lod_prefetch_drain": (ctypes.c_int, [_P]),
    "lod_read_nodes": (ctypes.c_int, [_P, _I64] + [_P] * 13),
    "lod_gather": (ctypes.c_int, [_P, _I64, _I64, _P, _P]),
    "lod_delta_info": (ctypes.c_int, [_P, ctypes.POINTER(LodDeltaInfo)]),
    "lod_read_delta": (ctypes.c_int, [_P] + [_P] * 9),
    "lod_render": (ctypes.c_int, [_P, _P, _P, ctypes.c_double, _P, _I64, _I64, ctypes.c_int, _P, _I64,
                                  ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "lod_raster_points": (ctypes.c_int, [ctypes.c_int32, _P, _P, _I64, _P, _P, _I64, _I64, ctypes.c_int]),
}

_L = None


def lib(path: str | None = None) -> ctypes.CDLL:
    """Load and type the library (no GPU is needed to load it)."""
    global _L
    if _L is None or path:
        L = ctypes.CDLL(path or os.environ.get("LODSTREAM_B200_LIB", _DEFAULT_LIB))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype, fn.argtypes = res, args
        _L = L
    return _L


class B200Error(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        self.kind = ERRORS.get(code)
        super().__init__(f"{what}: {lib().lod_strerror(code).decode()}")


def _check(rc: int, what: str, errors_module=None) -> None:
    """Raise the reference's exception for its three fatal codes (when the
    caller passes ``lodstream.errors``), else B200Error."""
    if rc == LOD_OK:
        return
    if errors_module is not None and rc in ERRORS:
        raise getattr(errors_module, ERRORS[rc])(lib().lod_strerror(rc).decode())
    raise B200Error(rc, what)


def create(bounds_min, bounds_size, arena_bytes, chunk_capacity, grid_res, leaf_threshold, max_depth,
           device: int = 0) -> ctypes.c_void_p:
    """Octree(bounds, Arena(arena_bytes), ChunkPool(arena, chunk_capacity), ...) on the device
    (octree.py:148-188)."""
    p = LodParams((ctypes.c_double * 3)(*bounds_min), float(bounds_size), grid_res, leaf_threshold, max_depth,
                  chunk_capacity, arena_bytes, device, 0)
    h = ctypes.c_void_p()
    _check(lib().lod_tree_create(ctypes.byref(p), ctypes.byref(h)), "lod_tree_create")
    return h


def destroy(h) -> None:
    _check(lib().lod_tree_destroy(h), "lod_tree_destroy")


def insert_batch(h, xyz, rgba, backlog_capacity=10_000_000, spill_capacity=100_000_000, collect_delta=False,
                 errors_module=None) -> LodBatchStats:
    """update.insert_batch (update.py:252-393) for host arrays: xyz (n, 3)
    float32, rgba (n,) uint32.  The returned stats feed UpdateStats
    (n_voxels -> voxels_created, num_nodes, splits_total, n_spill)."""
    xyz = np.ascontiguousarray(xyz, np.float32).reshape(-1, 3)
    rgba = np.ascontiguousarray(rgba, np.uint32).reshape(-1)
    if len(xyz) != len(rgba):
        raise ValueError("xyz and rgba lengths differ")
    st = LodBatchStats()
    if len(rgba) == 0:  # update.py:266-268
        return st
    lim = LodLimits(backlog_capacity, spill_capacity, None)
    flags = FLAG_DELTA if collect_delta else 0
    _check(lib().lod_insert_batch(h, xyz.ctypes.data, rgba.ctypes.data, len(rgba), ctypes.byref(lim), flags,
                                  ctypes.byref(st)), "lod_insert_batch", errors_module)
    return st


def insert_batch_device(h, xyz_ptr: int, rgba_ptr: int, n: int, stream: int, backlog_capacity=10_000_000,
                        spill_capacity=100_000_000, errors_module=None) -> LodBatchStats:
    """Batch already resident in HBM (device pointers, e.g. torch's
    ``data_ptr()``) produced on CUDA stream ``stream``: the tree's stream
    waits on it by event, no host synchronisation first."""
    st = LodBatchStats()
    lim = LodLimits(backlog_capacity, spill_capacity, ctypes.c_void_p(stream))
    _check(lib().lod_insert_batch(h, ctypes.c_void_p(xyz_ptr), ctypes.c_void_p(rgba_ptr), n, ctypes.byref(lim),
                                  FLAG_DEVICE_INPUT | FLAG_INPUT_STREAM, ctypes.byref(st)),
           "lod_insert_batch", errors_module)
    return st


def settle(h) -> LodSettleStats:
    """Wait for every queued cycle of the tree (tiny batches return once their
    one-kernel cycle is queued, with n_voxels = -1) and get what those cycles
    did: fold calls / n_voxels / n_voxels_max / n_spill_max / n_splits into
    UpdateStats (update.py:382-392)."""
    out = LodSettleStats()
    _check(lib().lod_tree_settle(h, ctypes.byref(out)), "lod_tree_settle")
    return out


def wait(h) -> float:
    """Block until the tree's last update has fully run (its device ms, or -1)."""
    ms = ctypes.c_float(-1.0)
    _check(lib().lod_tree_wait(h, ctypes.byref(ms)), "lod_tree_wait")
    return float(ms.value)


def prefetch(h, xyz, rgba) -> None:
    """run_frame_updates' ingest feed: stage queued batch k+1 (page-locked
    host arrays, kept unchanged until inserted) while batch k updates."""
    _check(lib().lod_prefetch_batch(h, xyz.ctypes.data, rgba.ctypes.data, len(rgba)), "lod_prefetch_batch")


def info(h) -> LodTreeInfo:
    i = LodTreeInfo()
    _check(lib().lod_tree_info(h, ctypes.byref(i)), "lod_tree_info")
    return i


def read_nodes(h, n: int) -> dict:
    """The Octree SoA columns (octree.py:169-182), rows [0, n)."""
    cols = {
        "parent": np.empty(n, np.int32), "octant": np.empty(n, np.uint8), "level": np.empty(n, np.int32),
        "children": np.empty((n, 8), np.int32), "inner": np.empty(n, np.bool_), "final": np.empty(n, np.bool_),
        "count": np.empty(n, np.int64), "pending": np.empty(n, np.int64), "chunk_head": np.empty(n, np.int32),
        "chunk_tail": np.empty(n, np.int32), "chunk_count": np.empty(n, np.int32),
        "grid_off": np.empty(n, np.int64), "bmin": np.empty((n, 3), np.float64),
    }
    _check(lib().lod_read_nodes(h, n, *(c.ctypes.data for c in cols.values())), "lod_read_nodes")
    return cols


def gather(h, nid: int, start: int, count: int):
    """Octree.gather_samples(nid, start) given the node's count."""
    k = max(count - start, 0)
    xyz, rgba = np.empty((k, 3), np.float32), np.empty(k, np.uint32)
    if k:
        _check(lib().lod_gather(h, nid, start, xyz.ctypes.data, rgba.ctypes.data), "lod_gather")
    return xyz, rgba


def read_delta(h):
    """BatchDelta of the last insert made with collect_delta=True
    (update.py:183-194, 333-355): (splits, voxel groups, point groups)."""
    d = LodDeltaInfo()
    _check(lib().lod_delta_info(h, ctypes.byref(d)), "lod_delta_info")
    ns, nvg, nv, npg = d.n_splits, d.n_voxel_groups, d.n_voxels, d.n_point_groups
    out = {"splits": np.empty(ns, np.int32), "vnode": np.empty(nvg, np.int32), "vstart": np.empty(nvg, np.int64),
           "vcount": np.empty(nvg, np.int64), "vcells": np.empty(nv, np.uint32), "vrgba": np.empty(nv, np.uint32),
           "pnode": np.empty(npg, np.int32), "pstart": np.empty(npg, np.int64), "pcount": np.empty(npg, np.int64)}
    _check(lib().lod_read_delta(h, *(a.ctypes.data for a in out.values())), "lod_read_delta")
    return out


def rasterize(h, num_nodes: int, planes, cam_packed, threshold: float, fb_cells, width: int, height: int,
              fresh: bool = False):
    """render.rasterize (render.py:213-225): device selection + splat into
    ``fb_cells`` (uint64, width*height, updated in place).  ``planes`` =
    render.frustum_planes(camera) (6 x 4 f64), ``cam_packed`` =
    Camera.packed() (18 f64).  ``fresh``: the framebuffer is all sentinel,
    so the device fills its target instead of uploading it.  Returns
    (selected node ids in visit order, samples drawn)."""
    planes = np.ascontiguousarray(planes, np.float64)
    cam = np.ascontiguousarray(cam_packed, np.float64)
    sel = np.empty(max(num_nodes, 1), np.int32)
    n, drawn = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().lod_render(h, planes.ctypes.data, cam.ctypes.data, float(threshold), fb_cells.ctypes.data, width,
                            height, FLAG_FB_CLEAR if fresh else 0, sel.ctypes.data, len(sel), ctypes.byref(n),
                            ctypes.byref(drawn)), "lod_render")
    return sel[: n.value].tolist(), int(drawn.value)


def brute_force_render(xyz, rgba, cam_packed, fb_cells, width: int, height: int, device: int = 0) -> None:
    """render.brute_force_render (render.py:228-239) into fb_cells (in place)."""
    xyz = np.ascontiguousarray(xyz, np.float32)
    rgba = np.ascontiguousarray(rgba, np.uint32)
    cam = np.ascontiguousarray(cam_packed, np.float64)
    _check(lib().lod_raster_points(device, xyz.ctypes.data, rgba.ctypes.data, len(rgba), cam.ctypes.data,
                                   fb_cells.ctypes.data, width, height, 0), "lod_raster_points")
