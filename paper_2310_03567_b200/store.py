"""Arena + chunk pool facades (reference: lodstream/store.py:34-166).

The storage of the B200 path lives in HBM: when an ``Octree`` is built over an
``Arena`` and a ``ChunkPool``, the library allocates one device arena of
``capacity`` bytes and the chunk tables next to it, and every allocation on
the update path (grid cuts, chunk acquisitions, LIFO reuse, releases) runs in
device kernels (csrc/lod_kernels.cuh: k_decide, k_execute, k_alloc_*).  The
Python objects then only mirror the device counters and tables on demand.

Before binding, the objects keep the reference's host bookkeeping so that the
standalone allocator API (``alloc``/``acquire``/``release``/``records``) behaves
exactly like the reference's (store.py:51-158); they hold no point data on the
update path.
"""
from __future__ import annotations

import threading

import numpy as np

from .errors import OutOfArena

RECORD_BYTES = 16
NO_CHUNK = -1


class Arena:
    """Monotone bump allocator (store.py:34-78); device-resident once bound."""

    def __init__(self, capacity: int) -> None:
        if capacity <= 0:
            raise ValueError("arena capacity must be positive")
        capacity = (capacity + 15) // 16 * 16
        self.capacity = capacity
        self._offset = 0
        self._host = None
        self._tree = None
        self._lock = threading.Lock()

    # -- binding -------------------------------------------------------------
    def _bind(self, tree) -> None:
        if self._tree is not None:
            raise ValueError("arena already backs another tree")
        if self._offset:
            raise ValueError("a device tree needs a fresh arena (offset 0)")
        self._tree = tree
        self._host = None

    @property
    def bound(self) -> bool:
        return self._tree is not None

    # -- allocator -------------------------------------------------------------
    def alloc(self, size: int, align: int = 16) -> int:
        """Reserve ``size`` bytes aligned to ``align`` (store.py:51-69)."""
        if size < 0:
            raise ValueError("negative allocation")
        if self._tree is not None:
            raise RuntimeError("this arena is owned by a device tree; allocation happens on the GPU")
        with self._lock:
            off = -self._offset % align + self._offset
            end = off + size
            if end > self.capacity:
                raise OutOfArena(
                    f"arena exhausted: need {end - self.capacity} bytes past capacity {self.capacity}"
                )
            self._offset = end
            return off

    @property
    def offset(self) -> int:
        if self._tree is not None:
            return int(self._tree._info().arena_offset)
        return self._offset

    @property
    def high_water(self) -> int:
        return self.offset

    # -- byte views ----------------------------------------------------------------
    @property
    def u8(self) -> np.ndarray:
        if self._tree is not None:
            return self._tree._arena_bytes(0, self.capacity)
        if self._host is None:
            self._host = np.zeros(self.capacity, np.uint8)
        return self._host

    @property
    def f32(self) -> np.ndarray:
        return self.u8.view(np.float32)

    @property
    def u32(self) -> np.ndarray:
        return self.u8.view(np.uint32)

    def bytes_at(self, off: int, size: int) -> np.ndarray:
        if self._tree is not None:
            return self._tree._arena_bytes(off, size)
        return self.u8[off: off + size]


class ChunkPool:
    """Fixed-capacity chunk table with LIFO reuse (store.py:81-166)."""

    def __init__(self, arena: Arena, capacity: int = 1000) -> None:
        if capacity <= 0:
            raise ValueError("chunk capacity must be positive")
        self.arena = arena
        self.capacity = capacity
        self.payload_bytes = capacity * RECORD_BYTES
        self._tree = None
        cap0 = 1024
        self._next = np.full(cap0, NO_CHUNK, dtype=np.int32)
        self._payload_off = np.zeros(cap0, dtype=np.int64)
        self._occupied = np.zeros(cap0, dtype=np.int32)
        self._allocated_total = 0
        self._released_total = 0
        self._free: list[int] = []
        self._lock = threading.Lock()

    def _bind(self, tree) -> None:
        if self._tree is not None:
            raise ValueError("pool already backs another tree")
        if self._allocated_total:
            raise ValueError("a device tree needs a fresh chunk pool")
        self._tree = tree

    # -- host bookkeeping (unbound pools only) -------------------------------------
    def _grow(self) -> None:
        cap = len(self._next) * 2
        self._next = np.concatenate([self._next, np.full(cap // 2, NO_CHUNK, np.int32)])
        self._payload_off = np.concatenate([self._payload_off, np.zeros(cap // 2, np.int64)])
        self._occupied = np.concatenate([self._occupied, np.zeros(cap // 2, np.int32)])

    def _unbound(self, what: str) -> None:
        if self._tree is not None:
            raise RuntimeError(f"{what}: this pool is owned by a device tree; chunks move on the GPU")

    def acquire(self) -> int:
        self._unbound("acquire")
        with self._lock:
            if self._free:
                cid = self._free.pop()
            else:
                cid = self._allocated_total
                if cid >= len(self._next):
                    self._grow()
                self._payload_off[cid] = self.arena.alloc(self.payload_bytes, RECORD_BYTES)
                self._allocated_total += 1
            self._next[cid] = NO_CHUNK
            self._occupied[cid] = 0
            return cid

    def release(self, head: int) -> int:
        self._unbound("release")
        n = 0
        with self._lock:
            cid = head
            while cid != NO_CHUNK:
                nxt = int(self._next[cid])
                self._occupied[cid] = 0
                self._next[cid] = NO_CHUNK
                self._free.append(cid)
                self._released_total += 1
                n += 1
                cid = nxt
        return n

    # -- mirrored state --------------------------------------------------------------
    @property
    def next(self) -> np.ndarray:
        return self._tree._pool_cols()["next"] if self._tree is not None else self._next

    @property
    def payload_off(self) -> np.ndarray:
        return self._tree._pool_cols()["payload_off"] if self._tree is not None else self._payload_off

    @property
    def occupied(self) -> np.ndarray:
        return self._tree._pool_cols()["occupied"] if self._tree is not None else self._occupied

    @property
    def allocated_total(self) -> int:
        return int(self._tree._info().allocated_total) if self._tree is not None else self._allocated_total

    @property
    def released_total(self) -> int:
        return int(self._tree._info().released_total) if self._tree is not None else self._released_total

    @property
    def free_count(self) -> int:
        return int(self._tree._info().free_count) if self._tree is not None else len(self._free)

    @property
    def free_list(self) -> np.ndarray:
        if self._tree is not None:
            return self._tree._pool_cols()["free_list"]
        return np.asarray(self._free, np.int32)

    @property
    def live_count(self) -> int:
        return self.allocated_total - self.free_count

    def records(self, cid: int) -> tuple[np.ndarray, np.ndarray]:
        """(xyz (capacity, 3) f32, rgba (capacity,) u32) of one payload (store.py:153-158).

        Bound pools return views of a host copy read from HBM, written back
        on the tree's next device call if edited; unbound pools return views.
        """
        off = int(self.payload_off[cid])
        if self._tree is not None:
            # a host copy of the payload; edits made through the returned
            # views are written back before the tree's next device call
            raw = self._tree._arena_bytes(off, self.payload_bytes)
            self._tree._arena_edits.append((off, raw, raw.copy()))
            f = raw.view(np.float32).reshape(self.capacity, 4)
            u = raw.view(np.uint32).reshape(self.capacity, 4)
            return f[:, :3], u[:, 3]
        f = self.arena.f32[off // 4: off // 4 + 4 * self.capacity].reshape(self.capacity, 4)
        u = self.arena.u32[off // 4: off // 4 + 4 * self.capacity].reshape(self.capacity, 4)
        return f[:, :3], u[:, 3]

    def check_ledger(self) -> None:
        """allocated_total == live + free (store.py:160-166)."""
        at, fc = self.allocated_total, self.free_count
        assert at == (at - fc) + fc and 0 <= fc <= at, (at, fc)
        if self._tree is not None:
            live = self._tree._live_chunks()
            assert at == live + fc, (at, live, fc)
