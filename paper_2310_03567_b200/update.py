"""Incremental batch insertion on the B200 (reference: lodstream/update.py).

``insert_batch`` runs one full update cycle of the reference's contract
(update.py:1-27) -- expansion (count <-> split until settled), sampling
(first-come voxel claims), allocation, store, cleanup -- as one call into the
CUDA library (``lod_insert_batch``).  The semantics, including the exact node
ids, per-node point/voxel sequences, chunk counts, arena growth and overflow
points, are the reference's; see DESIGN.md for how each pass maps to kernels.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .octree import Octree

__all__ = [
    "UpdateConfig",
    "UpdateState",
    "UpdateStats",
    "BatchDelta",
    "BudgetClock",
    "SpillBuffer",
    "VoxelBacklog",
    "chunks_needed",
    "insert_batch",
    "insert_records",
    "run_frame_updates",
]


def chunks_needed(count: int, capacity: int) -> int:
    """Chunks required to hold ``count`` records: ceil(count / capacity)."""
    return (count + capacity - 1) // capacity


@dataclass
class UpdateConfig:
    batch_size: int = 1_000_000
    budget_ms: float = 10.0
    backlog_capacity: int = 10_000_000
    spill_capacity: int = 100_000_000


@dataclass
class UpdateStats:
    batches: int = 0
    frames: int = 0
    points: int = 0
    voxels_created: int = 0
    nodes: int = 0
    splits: int = 0
    update_seconds: float = 0.0
    max_batch_ms: float = 0.0
    frame_ms_total: float = 0.0
    frame_ms_max: float = 0.0
    backlog_high_water: int = 0
    spill_high_water: int = 0
    device_seconds: float = 0.0  # CUDA-event time of the update kernels (B200 extra)
    launches: int = 0  # kernels launched by the updates (B200 extra)
    h2d_bytes: int = 0  # host->device bytes copied by the updates (B200 extra)
    d2h_bytes: int = 0  # device->host bytes read back by the updates (B200 extra)

    def throughput_mps(self) -> float:
        """Million points ingested per update-second (update.py:82-86)."""
        if self.update_seconds <= 0.0:
            return 0.0
        return self.points / self.update_seconds / 1e6


class BudgetClock:
    """Wall-clock frame budget, checked between batches (update.py:89-103)."""

    def __init__(self, budget_ms: float) -> None:
        self.budget_ms = budget_ms
        self._start = time.perf_counter()

    def restart(self) -> None:
        self._start = time.perf_counter()

    def elapsed_ms(self) -> float:
        return (time.perf_counter() - self._start) * 1e3

    def exceeded(self) -> bool:
        return self.elapsed_ms() >= self.budget_ms


class SpillBuffer:
    """Spill buffer (update.py:106-140).  Inside insert_batch the spilled
    records live in an HBM buffer of the tree for one cycle; between cycles
    the buffer is empty, which is all callers of the update can observe.
    Host segments are held only for ``Octree.split`` called directly
    (octree.py:222-264), which appends the split leaf's samples here."""

    def __init__(self, capacity: int) -> None:
        self.capacity = capacity
        self.total = 0
        self.high_water = 0
        self._xyz: list[np.ndarray] = []
        self._rgba: list[np.ndarray] = []

    def append(self, xyz: np.ndarray, rgba: np.ndarray) -> None:
        from .errors import SpillOverflow

        if self.total + len(rgba) > self.capacity:
            raise SpillOverflow(f"spill buffer past capacity {self.capacity}")
        self._xyz.append(xyz)
        self._rgba.append(rgba)
        self.total += len(rgba)
        self.high_water = max(self.high_water, self.total)

    def concat(self) -> tuple[np.ndarray, np.ndarray]:
        if not self._xyz:
            return np.empty((0, 3), np.float32), np.empty(0, np.uint32)
        return np.concatenate(self._xyz), np.concatenate(self._rgba)

    def clear(self) -> None:
        self._xyz.clear()
        self._rgba.clear()
        self.total = 0

    def __len__(self) -> int:
        return self.total


class VoxelBacklog:
    """Backlog accounting; the (node, cell, rgba) triples live in HBM for one
    cycle (update.py:143-171)."""

    def __init__(self, capacity: int) -> None:
        self.capacity = capacity
        self.length = 0
        self.high_water = 0

    def clear(self) -> None:
        self.length = 0


@dataclass
class BatchDelta:
    """What one cycle changed, in stream emission order (update.py:183-194):
    ``structure`` interleaves ("split", node) and ("create", node, parent,
    octant, level) events in split order; ``voxels`` lists (node, cells u32,
    rgba u32) and ``points`` (node, start, count) in ascending node id."""

    structure: list[tuple] = field(default_factory=list)
    voxels: list[tuple[int, np.ndarray, np.ndarray]] = field(default_factory=list)
    points: list[tuple[int, int, int]] = field(default_factory=list)


class UpdateState:
    """Per-tree transient state and statistics (update.py:197-223).

    Cycles the device has not run yet (a tiny batch's one-kernel cycle queued
    by an insert that could not fail, or an early-returning insert's tail) are
    folded into ``stats`` on the first read: the read waits for them
    (lod_tree_settle), adds their counts, and adds the wait to
    ``update_seconds`` -- so ``update_seconds`` is the wall time until the
    tree was settled, as in the reference, whose insert_batch returns settled."""

    def __init__(self, config: UpdateConfig | None = None) -> None:
        self.config = config or UpdateConfig()
        self.spill = SpillBuffer(self.config.spill_capacity)
        self.backlog = VoxelBacklog(self.config.backlog_capacity)
        self._stats = UpdateStats()
        self.clock = BudgetClock(self.config.budget_ms)
        self.last: dict | None = None  # LodBatchStats of the last call
        self._limits = _lib.LodLimits()
        self._bstats = _lib.LodBatchStats()
        self._unsettled: dict[int, Octree] = {}  # trees with work the device has not run yet

    @property
    def stats(self) -> UpdateStats:
        if self._unsettled:
            self.settle()
        return self._stats

    @stats.setter
    def stats(self, value: UpdateStats) -> None:
        self._stats = value

    def settle(self) -> None:
        """Wait for every queued cycle of this state's trees and fold their counts in."""
        st = self._stats
        for tree in list(self._unsettled.values()):
            t0 = time.perf_counter()
            out = _lib.LodSettleStats()
            rc = tree._L.lod_tree_settle(tree.handle, ctypes.byref(out))
            tree._invalidate()
            st.update_seconds += time.perf_counter() - t0
            st.device_seconds += float(out.device_ms) * 1e-3
            if out.calls:
                st.voxels_created += int(out.n_voxels)
                self.backlog.high_water = max(self.backlog.high_water, int(out.n_voxels_max))
                self.spill.high_water = max(self.spill.high_water, int(out.n_spill_max))
                st.backlog_high_water = self.backlog.high_water
                st.spill_high_water = self.spill.high_water
            st.splits = int(out.splits_total)
            st.nodes = int(out.num_nodes)
            _lib.check(rc, "settle")
        self._unsettled.clear()


def _as_input(a, dtype, shape_tail):
    """numpy / torch input -> (object keeping the buffer alive, is_device)."""
    if hasattr(a, "is_cuda") and a.is_cuda:
        import torch  # only when the caller already uses torch

        want = {np.float32: torch.float32, np.uint32: torch.int32}[dtype]
        if a.dtype not in (want, torch.uint32 if dtype is np.uint32 else want):
            raise TypeError(f"device input must be {want}, got {a.dtype}")
        if not a.is_contiguous():
            a = a.contiguous()
        return a, True
    arr = np.ascontiguousarray(a, dtype)
    if shape_tail:
        arr = arr.reshape((-1,) + shape_tail)
    return arr, False


def insert_batch(
    tree: Octree,
    xyz,
    rgba,
    state: UpdateState,
    collect_delta: bool = False,
    profile: bool = False,
) -> BatchDelta | None:
    """Run one full update cycle for a batch (update.py:252-393).

    ``xyz`` is (n, 3) float32 inside the tree bounds and ``rgba`` packed uint32
    (numpy arrays, copied H2D; or CUDA tensors already resident in HBM).  The
    whole batch is always consumed.
    """
    t0 = time.perf_counter()
    n_batch = len(rgba)
    if n_batch == 0:  # update.py:266-268
        return BatchDelta() if collect_delta else None
    if (n_batch <= _SMALL and not collect_delta and not profile and type(xyz) is np.ndarray
            and type(rgba) is np.ndarray):
        return _insert_small(tree, xyz, rgba, n_batch, state, t0)
    xyz_b, dev_x = _as_input(xyz, np.float32, (3,))
    rgba_b, dev_c = _as_input(rgba, np.uint32, ())
    if dev_x != dev_c:
        raise ValueError("xyz and rgba must both be host arrays or both be device tensors")
    # the C ABI copies / reads exactly 12 n + 4 n bytes: shapes must agree
    nx = xyz_b.numel() if dev_x else xyz_b.size
    nc = rgba_b.numel() if dev_c else rgba_b.size
    if nx != 3 * n_batch or nc != n_batch or (dev_x and tuple(xyz_b.shape) not in ((n_batch, 3), (3 * n_batch,))):
        raise ValueError(f"xyz must be ({n_batch}, 3) and rgba ({n_batch},); got {tuple(xyz_b.shape)} and "
                         f"{tuple(rgba_b.shape)}")
    flags = ((_lib.LOD_FLAG_DEVICE_INPUT if dev_x else 0) | (_lib.LOD_FLAG_PROFILE if profile else 0)
             | (_lib.LOD_FLAG_DELTA if collect_delta else 0))
    lim = _limits(tree, state, xyz_b if dev_x else None)
    if dev_x:
        flags |= _lib.LOD_FLAG_INPUT_STREAM
    bs = state._bstats
    rc = tree._L.lod_insert_batch(tree.handle, _lib.ptr(xyz_b), _lib.ptr(rgba_b), n_batch,
                                  ctypes.byref(lim), flags, ctypes.byref(bs))
    tree._invalidate()
    _lib.check(rc, "insert_batch")
    _account(state, bs, n_batch, profile)
    if bs.device_ms < 0:  # returned before its tail ran
        state._unsettled[id(tree)] = tree
    st = state._stats
    delta = _read_delta(tree) if collect_delta else None
    dt = time.perf_counter() - t0
    st.update_seconds += dt
    st.max_batch_ms = max(st.max_batch_ms, dt * 1e3)
    return delta


_SMALL = 256  # kSmallMaxBatch: host batches up to this size run as one kernel per cycle


def _insert_small(tree: Octree, xyz: np.ndarray, rgba: np.ndarray, n_batch: int, state: UpdateState,
                  t0: float) -> None:
    """insert_batch for a tiny host batch: the library runs the whole cycle as
    one kernel (lod_small.cuh) and, when no error is possible for the batch,
    returns as soon as it is queued (bs.iterations == -1); its counts reach
    ``state.stats`` when the state settles."""
    if xyz.dtype != np.float32 or not xyz.flags.c_contiguous:
        xyz = np.ascontiguousarray(xyz, np.float32)
    if rgba.dtype != np.uint32 or not rgba.flags.c_contiguous:
        rgba = np.ascontiguousarray(rgba, np.uint32)
    if xyz.size != 3 * n_batch or rgba.size != n_batch:
        raise ValueError(f"xyz must be ({n_batch}, 3) and rgba ({n_batch},); got {xyz.shape} and {rgba.shape}")
    lim = state._limits
    lim.backlog_capacity = state.config.backlog_capacity
    lim.spill_capacity = state.config.spill_capacity
    lim.input_stream = None
    bs = state._bstats
    rc = tree._L.lod_insert_batch(tree.handle, xyz.ctypes.data, rgba.ctypes.data, n_batch, ctypes.byref(lim), 0,
                                  ctypes.byref(bs))
    tree._gen += 1
    if tree._cache:
        tree._cache.clear()
    if tree._arena_edits:
        tree._arena_edits.clear()
    _lib.check(rc, "insert_batch")
    st = state._stats
    if bs.iterations < 0:  # queued: counts folded in when the state settles
        st.batches += 1
        st.points += n_batch
        st.launches += 1
        st.h2d_bytes += 16 * n_batch
        state._unsettled[id(tree)] = tree
    else:
        _account(state, bs, n_batch, False)
    dt = time.perf_counter() - t0
    st.update_seconds += dt
    if dt * 1e3 > st.max_batch_ms:
        st.max_batch_ms = dt * 1e3
    return None


def insert_records(tree: Octree, records, state: UpdateState, collect_delta: bool = False) -> BatchDelta | None:
    """insert_batch for a batch already packed as 16-byte records
    (f32 x, y, z | u32 rgba; store.py:14-16) -- e.g. the points routed to this
    rank by multigpu.route.  ``records`` is a CUDA tensor (n, 4) of 4-byte
    elements, or a numpy array of the same shape."""
    t0 = time.perf_counter()
    n_batch = int(records.shape[0])
    if n_batch == 0:
        return BatchDelta() if collect_delta else None
    if hasattr(records, "is_cuda") and records.is_cuda:
        if records.element_size() != 4 or records.dim() != 2 or records.shape[1] != 4:
            raise TypeError("records must be an (n, 4) tensor of 4-byte elements")
        rec, flags = records.contiguous(), _lib.LOD_FLAG_DEVICE_INPUT | _lib.LOD_FLAG_INPUT_STREAM
    else:
        rec = np.ascontiguousarray(records)
        if rec.ndim != 2 or rec.shape[1] != 4 or rec.dtype.itemsize != 4:
            raise TypeError("records must be an (n, 4) array of 4-byte elements")
        flags = 0
    flags |= _lib.LOD_FLAG_PACKED | (_lib.LOD_FLAG_DELTA if collect_delta else 0)
    lim = _limits(tree, state, rec if flags & _lib.LOD_FLAG_DEVICE_INPUT else None)
    bs = state._bstats
    rc = tree._L.lod_insert_batch(tree.handle, _lib.ptr(rec), None, n_batch, ctypes.byref(lim), flags, ctypes.byref(bs))
    tree._invalidate()
    _lib.check(rc, "insert_records")
    _account(state, bs, n_batch, profile=False)
    delta = _read_delta(tree) if collect_delta else None
    dt = time.perf_counter() - t0
    if bs.device_ms < 0:
        state._unsettled[id(tree)] = tree
    state._stats.update_seconds += dt
    state._stats.max_batch_ms = max(state._stats.max_batch_ms, dt * 1e3)
    return delta


def _limits(tree: Octree, state: UpdateState, dev_tensor):
    """LodLimits of one call.  Device inputs are ordered after the work queued
    so far on torch's current stream of their device (the copy, kernel or
    collective that produced them), without a host sync."""
    lim = state._limits
    lim.backlog_capacity = state.config.backlog_capacity
    lim.spill_capacity = state.config.spill_capacity
    lim.input_stream = None
    if dev_tensor is not None:
        import torch

        if dev_tensor.device.index != tree.device:
            raise ValueError(f"input on {dev_tensor.device}, tree on cuda:{tree.device}")
        lim.input_stream = torch.cuda.current_stream(dev_tensor.device).cuda_stream
    return lim


def _account(state: UpdateState, bs, n_batch: int, profile: bool) -> None:
    """UpdateStats bookkeeping of one cycle (update.py:382-392)."""
    st = state._stats
    n_v, n_s = int(bs.n_voxels), int(bs.n_spill)
    st.batches += 1
    st.points += n_batch
    state.backlog.high_water = max(state.backlog.high_water, n_v)
    state.spill.high_water = max(state.spill.high_water, n_s)
    st.backlog_high_water = state.backlog.high_water
    st.spill_high_water = state.spill.high_water
    st.voxels_created += n_v
    st.splits = int(bs.splits_total)
    st.nodes = int(bs.num_nodes)
    # device time: this call's, or (when it returned before its tail ran) the
    # previous early call's, reported now; wait_settled collects the last one
    for ms in (bs.device_ms, bs.device_ms_prev):
        if ms >= 0:
            st.device_seconds += float(ms) * 1e-3
    st.launches += int(bs.launches)
    st.h2d_bytes += int(bs.h2d_bytes)
    st.d2h_bytes += int(bs.d2h_bytes)
    state.last = bs.as_dict() if profile else None


def wait_settled(tree: Octree, state: UpdateState | None = None) -> float:
    """Block until the tree's updates have fully run on the device.

    insert_batch returns once the cycle's outcome is final (allocation done,
    errors raised); the sort + store + cleanup of its last pass may still run
    on the tree's stream, ahead of every later call on the tree, and a tiny
    batch's one-kernel cycle may still be queued.  Returns the device ms of
    the work that was outstanding (-1 if none) and, with ``state``, folds its
    counts and the wall wait into ``state.stats``."""
    if state is not None:
        state._unsettled[id(tree)] = tree
        before = state._stats.device_seconds
        state.settle()
        ms = (state._stats.device_seconds - before) * 1e3
        return ms if ms > 0 else -1.0
    out = _lib.LodSettleStats()
    rc = tree._L.lod_tree_settle(tree.handle, ctypes.byref(out))
    tree._invalidate()
    _lib.check(rc, "settle")
    return float(out.device_ms) if out.device_ms > 0 else -1.0


def _read_delta(tree: Octree) -> BatchDelta:
    """The cycle's BatchDelta, assembled on the device (k_delta_segs /
    k_delta_vox) and copied out once (lod_read_delta); the "create" events are
    each split's 8 children in octant order (update.py:240-245)."""
    info = _lib.LodDeltaInfo()
    _lib.check(tree._L.lod_delta_info(tree.handle, ctypes.byref(info)), "delta_info")
    ns, nvg, nv, npg = info.n_splits, info.n_voxel_groups, info.n_voxels, info.n_point_groups
    splits = np.empty(ns, np.int32)
    vnode, vstart, vcount = np.empty(nvg, np.int32), np.empty(nvg, np.int64), np.empty(nvg, np.int64)
    cells, cols = _lib.pinned_empty(nv, np.uint32), _lib.pinned_empty(nv, np.uint32)  # the bulk: DMA'd
    pnode, pstart, pcount = np.empty(npg, np.int32), np.empty(npg, np.int64), np.empty(npg, np.int64)
    p = _lib.ptr
    _lib.check(tree._L.lod_read_delta(tree.handle, p(splits), p(vnode), p(vstart), p(vcount), p(cells), p(cols),
                                      p(pnode), p(pstart), p(pcount)), "read_delta")
    d = BatchDelta()
    if ns:
        # every split appends its 8 children in split order (octree.py:249-261),
        # so the i-th split's children are n0 + 8 i + o; only the level column
        # is read back (not the whole node table)
        n1 = tree.num_nodes
        n0 = n1 - 8 * ns
        level = np.empty(n1, np.int32)
        _lib.check(tree._L.lod_read_nodes(tree.handle, n1, None, None, p(level), *([None] * 10)), "read levels")
        for i, nid in enumerate(splits.tolist()):
            d.structure.append(("split", nid))
            lv = int(level[nid]) + 1
            for o in range(8):
                d.structure.append(("create", n0 + 8 * i + o, nid, o, lv))
    d.voxels = [(int(a), cells[s:s + c], cols[s:s + c]) for a, s, c in zip(vnode.tolist(), vstart.tolist(),
                                                                        vcount.tolist())]
    d.points = list(zip(pnode.tolist(), pstart.tolist(), pcount.tolist()))
    return d


def _prefetch(tree: Octree, batch) -> bool:
    """Stage a queued host batch H2D on the tree's copy stream (the ingest
    feed, lod_prefetch_batch) when its arrays are used in place by
    insert_batch (C-contiguous float32 (n,3) / uint32); page-locked memory
    overlaps with the running update, anything else is left to the insert."""
    xyz, rgba = batch
    if not (isinstance(xyz, np.ndarray) and isinstance(rgba, np.ndarray)):
        return False
    if (xyz.dtype != np.float32 or rgba.dtype != np.uint32 or not xyz.flags.c_contiguous
            or not rgba.flags.c_contiguous or xyz.ndim != 2 or xyz.shape[1] != 3 or len(rgba) != len(xyz)
            or len(rgba) == 0):
        return False
    _lib.check(tree._L.lod_prefetch_batch(tree.handle, _lib.ptr(xyz), _lib.ptr(rgba), len(rgba)), "prefetch")
    return True


def run_frame_updates(tree, batches, state: UpdateState, on_delta=None) -> int:
    """Drain queued batches for one frame within the budget (update.py:396-417).

    The budget is checked between batches, as in the reference.  While batch
    k updates, the H2D copies of batches k+1 and k+2 run on the copy stream
    (pinned host batches), so the queue streams at the update rate or the
    PCIe rate, whichever is lower.  Staged copies of batches still queued at
    the end of a frame are kept for the next frame (the tree holds references
    to those arrays, so they stay alive): if the next call finds the same
    array objects at the head of the queue, their copies are used, otherwise
    every staged copy is dropped first.  As with any asynchronous copy, a
    queued batch must not be modified in place while it is queued."""
    state.clock.restart()
    processed = 0
    kept = getattr(tree, "_staged_heads", None)
    if kept:
        tree._staged_heads = None
        if not (len(batches) >= len(kept) and all(batches[i] is kept[i] for i in range(len(kept)))):
            tree._L.lod_prefetch_drain(tree.handle)
    staged = bool(kept)
    ok = False
    try:
        while batches and (processed == 0 or not state.clock.exceeded()):
            xyz, rgba = batches.popleft()
            # keep the next two queued batches copying (3 staging slots: the
            # one being consumed + two in flight)
            for ahead in range(min(2, len(batches))):
                staged = _prefetch(tree, batches[ahead]) or staged
            delta = insert_batch(tree, xyz, rgba, state, collect_delta=on_delta is not None)
            if on_delta is not None:
                on_delta(delta)
            processed += 1
        ok = True
    finally:
        if staged:
            if ok:  # the still-queued batches staged last keep their copies
                tree._staged_heads = [batches[i] for i in range(min(2, len(batches)))]
            else:  # an error ends the frame: the caller owns the queued arrays again
                tree._L.lod_prefetch_drain(tree.handle)
    if processed:
        st = state._stats  # no settle: the frame's last tail keeps running behind the caller
        st.frames += 1
        dt = state.clock.elapsed_ms()
        st.frame_ms_total += dt
        st.frame_ms_max = max(st.frame_ms_max, dt)
    return processed
