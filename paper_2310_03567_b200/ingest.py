"""Disk -> GPU ingest of SIM point files (reference: lodstream/io.py).

A SIM file is a flat array of 16-byte records ``f32 x, y, z, u8 r, g, b, a``
(io.py:38-40, 60-92) -- byte for byte the update path's record layout
(store.py:14-16; rgba packs as r | g << 8 | b << 16 | a << 24).  The
reference reads it with an O_DIRECT reader (io.py:218-290) on a thread that
feeds a queue of batches (BatchSource, io.py:340-413) into the frame loop.
Here ``SimSource`` is a native reader thread (csrc/lod_ingest.cu) reading
batches with O_DIRECT straight into page-locked slots, and ``stream_sim`` is
the disk -> insert -> render loop: batch k+1's DMA to HBM is staged
(lod_prefetch_records) while batch k updates, and no host code touches the
points.
"""
from __future__ import annotations

import ctypes
import os
import time

import numpy as np

from . import _lib

RECORD_BYTES = 16
SIM_DTYPE = np.dtype([("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("r", "u1"), ("g", "u1"), ("b", "u1"),
                      ("a", "u1")])


def write_sim(path, xyz: np.ndarray, rgba: np.ndarray) -> None:
    """Write records to a SIM file (io.py:60-72); ``rgba`` is packed uint32."""
    rec = np.empty((len(rgba), 4), np.uint32)
    rec[:, :3] = np.ascontiguousarray(xyz, np.float32).view(np.uint32)
    rec[:, 3] = np.ascontiguousarray(rgba, np.uint32)
    with open(path, "wb") as f:
        rec.tofile(f)


def read_sim(path) -> tuple[np.ndarray, np.ndarray]:
    """Whole SIM file as (xyz float32 (n, 3), rgba uint32) (io.py:75-84)."""
    size = os.path.getsize(path)
    if size == 0 or size % RECORD_BYTES:
        raise ValueError(f"{path}: {size} bytes is not a whole, non-empty number of records")
    rec = np.fromfile(path, np.uint32).reshape(-1, 4)
    return np.ascontiguousarray(rec[:, :3]).view(np.float32), np.ascontiguousarray(rec[:, 3])


class SimSource:
    """Batches of a SIM file in file order, read ahead by native reader
    threads (LOD_SIM_READERS, default 1; several reads in flight help striped
    volumes) with O_DIRECT into ``slots`` page-locked buffers.  ``next_batch``
    returns a packed (n, 4) uint32 record array (a view of its slot, valid
    until ``release``), or None at end of file."""

    def __init__(self, path, batch_size: int = 1_000_000, slots: int = 4) -> None:
        if (batch_size * RECORD_BYTES) % 4096:
            raise ValueError("batch_size * 16 must be a multiple of 4096 (O_DIRECT alignment)")
        self._L = _lib.load()
        h = ctypes.c_void_p()
        _lib.check(self._L.lod_sim_open(os.fsencode(str(path)), batch_size, slots, ctypes.byref(h)), f"open {path}")
        self._h = h
        self.batch_size = batch_size

    def next_batch(self) -> np.ndarray | None:
        p, n = ctypes.c_void_p(), ctypes.c_int64(0)
        _lib.check(self._L.lod_sim_next(self._h, ctypes.byref(p), ctypes.byref(n)), "sim read")
        if n.value == 0:
            return None
        buf = (ctypes.c_uint32 * (4 * n.value)).from_address(p.value)
        return np.frombuffer(buf, np.uint32).reshape(n.value, 4)

    def release(self, batch: np.ndarray) -> None:
        _lib.check(self._L.lod_sim_release(self._h, batch.ctypes.data), "sim release")

    def info(self) -> dict:
        i = _lib.LodSimInfo()
        _lib.check(self._L.lod_sim_info(self._h, ctypes.byref(i)), "sim info")
        return {"file_bytes": int(i.file_bytes), "bytes_read": int(i.bytes_read),
                "read_seconds": float(i.read_seconds), "o_direct": bool(i.direct), "pinned": bool(i.pinned)}

    def __iter__(self):
        while True:
            b = self.next_batch()
            if b is None:
                return
            yield b
            self.release(b)

    def close(self) -> None:
        if self._h:
            self._L.lod_sim_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def stream_sim(tree, path, state, batch_size: int = 1 << 20, camera=None, threshold: float = 128.0,
               render_every: int = 1, slots: int = 8) -> dict:
    """Disk -> insert -> render: every batch of the SIM file into the tree
    (insert_records), rendering ``camera`` into a device framebuffer every
    ``render_every`` batches (render.rasterize's device path: selection + splat,
    the paper's per-frame draw).  Returns the wall time from open to the
    settled tree and the reader's counters."""
    from .render import frustum_planes
    from .update import insert_records, wait_settled

    t0 = time.perf_counter()
    src = SimSource(path, batch_size, slots)
    L = tree._L
    fb = sel = planes = cam = None
    if camera is not None:
        import torch

        fb = torch.empty(camera.width * camera.height, dtype=torch.int64, device=f"cuda:{tree.device}")
        planes = np.ascontiguousarray(frustum_planes(camera), np.float64)
        cam = np.ascontiguousarray(camera.packed(), np.float64)
    batches = points = frames = drawn_total = 0
    cur = src.next_batch()
    while cur is not None:
        nxt = src.next_batch()
        if nxt is not None:  # its DMA runs while `cur` updates
            _lib.check(L.lod_prefetch_records(tree.handle, nxt.ctypes.data, len(nxt)), "prefetch")
        insert_records(tree, cur, state)
        src.release(cur)  # the insert returned: its copy has landed
        batches += 1
        points += len(cur)
        if camera is not None and batches % render_every == 0:
            if sel is None or len(sel) < tree.num_nodes:
                sel = np.empty(max(2 * tree.num_nodes, 1024), np.int32)
            n, drawn = ctypes.c_int64(0), ctypes.c_int64(0)
            fb.fill_(-1)
            _lib.check(L.lod_render(tree.handle, _lib.ptr(planes), _lib.ptr(cam), float(threshold), _lib.ptr(fb),
                                    camera.width, camera.height, _lib.LOD_FLAG_DEVICE_FB, _lib.ptr(sel), len(sel),
                                    ctypes.byref(n), ctypes.byref(drawn)), "render")
            frames += 1
            drawn_total += int(drawn.value)
        cur = nxt
    wait_settled(tree, state)
    dt = time.perf_counter() - t0
    info = src.info()
    src.close()
    return {"batches": batches, "points": points, "seconds": dt, "mpts_per_s": points / dt / 1e6,
            "gb_per_s": info["bytes_read"] / dt / 1e9, "frames": frames, "samples_drawn": drawn_total, **info}
