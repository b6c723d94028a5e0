"""ctypes binding of the C ABI in include/lod_b200.h (``_lodb200.so``).

There is deliberately no CPU fallback: if the CUDA library is missing, or no
CUDA device is visible, every entry point that needs the GPU raises
``NativeUnavailable`` with the reason.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import BacklogOverflow, OutOfArena, SpillOverflow

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LOD_B200_LIB") or os.path.join(_HERE, "_lodb200.so")  # override: A/B experiments

LOD_OK = 0
LOD_E_OUT_OF_ARENA = 1
LOD_E_SPILL_OVERFLOW = 2
LOD_E_BACKLOG_OVERFLOW = 3
LOD_E_CUDA = 4
LOD_E_ARG = 5
LOD_E_NOMEM = 6
LOD_E_NO_DEVICE = 7

LOD_FLAG_DEVICE_INPUT = 1
LOD_FLAG_DEVICE_FB = 2
LOD_FLAG_PROFILE = 4
LOD_FLAG_DELTA = 8
LOD_FLAG_PACKED = 16
LOD_FLAG_INPUT_STREAM = 32
LOD_FLAG_FB_CLEAR = 64
LOD_NPHASE = 10
LOD_IPC_HANDLE_BYTES = 64
LOD_WINDOW_HEADER_BYTES = 2 * 64 * 64 * 8 + 6 * 64 * 8
PHASES = ("count", "split", "resolve", "backlog", "alloc", "sort", "delta", "epilogue", "h2d", "total")


class NativeUnavailable(RuntimeError):
    """The sm_100a CUDA library or a CUDA device is not available."""


class LodError(RuntimeError):
    pass


class LodParams(ctypes.Structure):
    _fields_ = [
        ("bmin", ctypes.c_double * 3),
        ("size", ctypes.c_double),
        ("grid_res", ctypes.c_int64),
        ("leaf_threshold", ctypes.c_int64),
        ("max_depth", ctypes.c_int64),
        ("chunk_capacity", ctypes.c_int64),
        ("arena_bytes", ctypes.c_uint64),
        ("device", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class LodLimits(ctypes.Structure):
    _fields_ = [("backlog_capacity", ctypes.c_int64), ("spill_capacity", ctypes.c_int64),
                ("input_stream", ctypes.c_void_p)]


class LodBatchStats(ctypes.Structure):
    _fields_ = [
        ("n_batch", ctypes.c_int64), ("n_spill", ctypes.c_int64), ("n_voxels", ctypes.c_int64),
        ("n_splits", ctypes.c_int64), ("iterations", ctypes.c_int64),
        ("num_nodes", ctypes.c_int64), ("splits_total", ctypes.c_int64), ("max_level", ctypes.c_int64),
        ("allocated_total", ctypes.c_int64), ("free_count", ctypes.c_int64),
        ("released_total", ctypes.c_int64), ("arena_offset", ctypes.c_uint64),
        ("launches", ctypes.c_int64), ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
        ("device_ms", ctypes.c_float), ("device_ms_prev", ctypes.c_float),
        ("phase_ms", ctypes.c_float * LOD_NPHASE),
    ]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "phase_ms"}
        d["phase_ms"] = dict(zip(PHASES, list(self.phase_ms)))
        return d


class LodTreeInfo(ctypes.Structure):
    _fields_ = [
        ("num_nodes", ctypes.c_int64), ("node_capacity", ctypes.c_int64),
        ("splits_total", ctypes.c_int64), ("max_level", ctypes.c_int64),
        ("allocated_total", ctypes.c_int64), ("free_count", ctypes.c_int64),
        ("released_total", ctypes.c_int64), ("chunk_capacity_rows", ctypes.c_int64),
        ("arena_offset", ctypes.c_uint64), ("arena_capacity", ctypes.c_uint64),
        ("grid_bytes", ctypes.c_int64), ("chunk_capacity", ctypes.c_int64),
    ]


class LodSettleStats(ctypes.Structure):
    _fields_ = [("calls", ctypes.c_int64), ("n_voxels", ctypes.c_int64), ("n_voxels_max", ctypes.c_int64),
                ("n_spill_max", ctypes.c_int64), ("n_splits", ctypes.c_int64), ("num_nodes", ctypes.c_int64),
                ("splits_total", ctypes.c_int64), ("max_level", ctypes.c_int64), ("device_ms", ctypes.c_float),
                ("error", ctypes.c_int32)]


class LodSimInfo(ctypes.Structure):
    _fields_ = [("file_bytes", ctypes.c_uint64), ("bytes_read", ctypes.c_uint64), ("read_seconds", ctypes.c_double),
                ("direct", ctypes.c_int32), ("pinned", ctypes.c_int32)]


class LodDeltaInfo(ctypes.Structure):
    _fields_ = [("n_splits", ctypes.c_int64), ("n_voxel_groups", ctypes.c_int64), ("n_voxels", ctypes.c_int64),
                ("n_point_groups", ctypes.c_int64)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64

# name -> (restype, argtypes); kept in sync with include/lod_b200.h
SIGNATURES = {
    "lod_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "lod_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "lod_tree_create": (ctypes.c_int, [ctypes.POINTER(LodParams), ctypes.POINTER(_P)]),
    "lod_tree_destroy": (ctypes.c_int, [_P]),
    "lod_tree_info": (ctypes.c_int, [_P, ctypes.POINTER(LodTreeInfo)]),
    "lod_insert_batch": (ctypes.c_int, [_P, _P, _P, _I64, ctypes.POINTER(LodLimits), ctypes.c_int,
                                        ctypes.POINTER(LodBatchStats)]),
    "lod_prefetch_batch": (ctypes.c_int, [_P, _P, _P, _I64]),
    "lod_prefetch_drain": (ctypes.c_int, [_P]),
    "lod_prefetch_records": (ctypes.c_int, [_P, _P, _I64]),
    "lod_sim_open": (ctypes.c_int, [ctypes.c_char_p, _I64, ctypes.c_int32, ctypes.POINTER(_P)]),
    "lod_sim_next": (ctypes.c_int, [_P, ctypes.POINTER(_P), ctypes.POINTER(_I64)]),
    "lod_sim_release": (ctypes.c_int, [_P, _P]),
    "lod_sim_info": (ctypes.c_int, [_P, ctypes.POINTER(LodSimInfo)]),
    "lod_sim_close": (ctypes.c_int, [_P]),
    "lod_tree_wait": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_float)]),
    "lod_tree_settle": (ctypes.c_int, [_P, ctypes.POINTER(LodSettleStats)]),
    "lod_read_nodes": (ctypes.c_int, [_P, _I64] + [_P] * 13),
    "lod_read_pool": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _I64]),
    "lod_gather": (ctypes.c_int, [_P, _I64, _I64, _P, _P]),
    "lod_read_directory": (ctypes.c_int, [_P, _I64, _P, _P, _P, _I64, ctypes.POINTER(ctypes.c_uint64)]),
    "lod_split_node": (ctypes.c_int, [_P, _I64, ctypes.POINTER(ctypes.c_int32)]),
    "lod_append_chunk": (ctypes.c_int, [_P, _I64, ctypes.POINTER(ctypes.c_int32)]),
    "lod_grid_test_and_set": (ctypes.c_int, [_P, _I64, _I64, ctypes.POINTER(ctypes.c_int32)]),
    "lod_write_nodes": (ctypes.c_int, [_P, _I64] + [_P] * 13),
    "lod_write_pool": (ctypes.c_int, [_P, _I64, _P, _P, _P]),
    "lod_write_arena": (ctypes.c_int, [_P, ctypes.c_uint64, ctypes.c_uint64, _P]),
    "lod_dump_records": (ctypes.c_int, [_P, _I64, _P, _P]),
    "lod_delta_info": (ctypes.c_int, [_P, ctypes.POINTER(LodDeltaInfo)]),
    "lod_read_delta": (ctypes.c_int, [_P] + [_P] * 9),
    "lod_read_arena": (ctypes.c_int, [_P, ctypes.c_uint64, ctypes.c_uint64, _P]),
    "lod_rasterize": (ctypes.c_int, [_P, _P, _I64, _P, _P, _I64, _I64, ctypes.c_int, ctypes.POINTER(_I64)]),
    "lod_select_visible": (ctypes.c_int, [_P, _P, _P, ctypes.c_double, _P, _I64, ctypes.POINTER(_I64)]),
    "lod_render": (ctypes.c_int, [_P, _P, _P, ctypes.c_double, _P, _I64, _I64, ctypes.c_int, _P, _I64,
                                  ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    "lod_raster_points": (ctypes.c_int, [ctypes.c_int32, _P, _P, _I64, _P, _P, _I64, _I64, ctypes.c_int]),
    "lod_morton_sort": (ctypes.c_int, [ctypes.c_int32, _P, ctypes.c_double, ctypes.c_int32, _P, _P, _I64, _P, _P,
                                       _P, ctypes.c_int]),
    "lod_route_bucket": (ctypes.c_int, [ctypes.c_int32, _P, ctypes.c_double, ctypes.c_int32, _P, ctypes.c_int32, _P, _P,
                                        _I64, _P, _P, _P, _P, _P]),
    "lod_last_voxels": (ctypes.c_int, [_P, ctypes.c_int32, _I64, _P, _P, _P, _P, ctypes.POINTER(_I64)]),
    "lod_last_voxels_count": (ctypes.c_int, [_P, ctypes.c_int32, _P, _P]),
    "lod_last_voxels_log": (ctypes.c_int, [_P, ctypes.c_int32, _P, _I64, _P, _P, _P, _P, _I64, _P, _P]),
    "lod_merge_voxels": (ctypes.c_int, [_P, _I64, _P, _P, _P, _P, _P]),
    "lod_ipc_alloc": (ctypes.c_int, [ctypes.c_int32, ctypes.c_uint64, ctypes.POINTER(_P), _P]),
    "lod_ipc_open": (ctypes.c_int, [ctypes.c_int32, _P, ctypes.POINTER(_P)]),
    "lod_ipc_close": (ctypes.c_int, [_P]),
    "lod_route_peers_begin": (ctypes.c_int, [ctypes.c_int32, _P, ctypes.c_double, ctypes.c_int32, _P, ctypes.c_int32,
                                             ctypes.c_int32, _P, _I64, _P, ctypes.c_int32, ctypes.c_uint64, _P, _P,
                                             _P, ctypes.c_int32, _P]),
    "lod_route_peers_finish": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _P, _I64, _P,
                                              ctypes.c_int32, _I64, ctypes.c_uint64, ctypes.c_int32, _P]),
    "lod_composite_min_peers": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _P, _I64, _P]),
    "lod_device_alloc": (ctypes.c_int, [ctypes.c_int32, ctypes.c_uint64, ctypes.POINTER(_P)]),
    "lod_device_free": (ctypes.c_int, [_P]),
    "lod_memcpy_h2d": (ctypes.c_int, [_P, _P, ctypes.c_uint64]),
    "lod_memcpy_d2h": (ctypes.c_int, [_P, _P, ctypes.c_uint64]),
    "lod_host_alloc": (ctypes.c_int, [ctypes.c_uint64, ctypes.POINTER(_P)]),
    "lod_host_free": (ctypes.c_int, [_P]),
    "lod_fb_fill": (ctypes.c_int, [ctypes.c_int32, _P, _I64, ctypes.c_uint64]),
    "lod_l2_flush": (ctypes.c_int, [ctypes.c_int32]),
    "lod_tree_pack_size": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_uint64)]),
    "lod_tree_pack": (ctypes.c_int, [_P, _P, ctypes.c_uint64]),
    "lod_tree_unpack": (ctypes.c_int, [_P, _P, ctypes.c_uint64]),
}

_lib = None


def load(path: str | None = None) -> ctypes.CDLL:
    """Load the CUDA library (no GPU needed just to load it)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise NativeUnavailable(
            f"{p} is missing: build it with `python -m paper_2310_03567_b200.build` "
            "(there is no CPU fallback)"
        )
    L = ctypes.CDLL(p)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = L
    return L


def device_count() -> int:
    n = ctypes.c_int(0)
    load().lod_device_count(ctypes.byref(n))
    return int(n.value)


def require_device(device: int = 0) -> ctypes.CDLL:
    L = load()
    n = device_count()
    if n <= device:
        raise NativeUnavailable(f"CUDA device {device} not available ({n} visible); no CPU fallback")
    return L


def check(rc: int, what: str = "") -> None:
    if rc == LOD_OK:
        return
    msg = load().lod_strerror(rc).decode()
    if what:
        msg = f"{what}: {msg}"
    if rc == LOD_E_OUT_OF_ARENA:
        raise OutOfArena(msg)
    if rc == LOD_E_SPILL_OVERFLOW:
        raise SpillOverflow(msg)
    if rc == LOD_E_BACKLOG_OVERFLOW:
        raise BacklogOverflow(msg)
    if rc == LOD_E_NO_DEVICE:
        raise NativeUnavailable(msg)
    if rc == LOD_E_ARG:
        raise ValueError(msg)
    if rc == LOD_E_NOMEM:
        raise MemoryError(msg)
    raise LodError(msg)


def ptr(a) -> ctypes.c_void_p:
    if a is None:
        return ctypes.c_void_p(0)
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    if hasattr(a, "data_ptr"):  # torch tensor
        return ctypes.c_void_p(a.data_ptr())
    if isinstance(a, int):
        return ctypes.c_void_p(a)
    raise TypeError(f"cannot take a pointer of {type(a)!r}")


# -- page-locked host arrays ---------------------------------------------------
# Results the device writes out wholesale (framebuffers, BatchDelta columns)
# land in page-locked memory, so the D2H is a DMA at link speed instead of a
# staged pageable copy.  Buffers come from a per-size-class pool (powers of
# two) and return to it when the last numpy view of them dies.
_PINNED_FREE: dict[int, list[int]] = {}
_PINNED_KEEP = 4


def _pinned_release(nbytes: int, addr: int) -> None:
    free = _PINNED_FREE.setdefault(nbytes, [])
    if len(free) < _PINNED_KEEP:
        free.append(addr)
    else:
        load().lod_host_free(ctypes.c_void_p(addr))


def pinned_empty(n: int, dtype) -> np.ndarray:
    """An uninitialised page-locked numpy array of n elements."""
    import weakref

    dt = np.dtype(dtype)
    need = max(int(n) * dt.itemsize, 1)
    nbytes = 1 << (need - 1).bit_length()
    free = _PINNED_FREE.get(nbytes)
    if free:
        addr = free.pop()
    else:
        p = ctypes.c_void_p()
        check(load().lod_host_alloc(nbytes, ctypes.byref(p)), "pinned host buffer")
        addr = int(p.value)
    buf = (ctypes.c_uint8 * nbytes).from_address(addr)
    weakref.finalize(buf, _pinned_release, nbytes, addr)
    return np.frombuffer(buf, dt, count=int(n))
