"""Octant-prefix partitioned insertion across GPUs.

One process per GPU (torch.distributed, NCCL).  Protocol per global batch
(the batch arrives striped: rank r holds global points [r*B, (r+1)*B)):

* **warm-up** -- until every node above the partition depth L is inner in the
  global tree, all stripes are gathered to rank 0 (in rank order = global
  order) and rank 0 inserts them into its tree: exactly the single-GPU run.
* **hand-off** -- rank 0 packs its tree (``lod_tree_pack``) and broadcasts it;
  every rank unpacks it, so all ranks share the same top and every prefix
  subtree starts from the single-GPU state.
* **partitioned** -- each rank computes the owner of its stripe's points from
  their depth-L octant prefix (exact float64 descent rule on the device) and
  buckets them stably by owner; the bucket scatter writes every 16-byte record
  straight into its owner's receive window over peer memory (``PeerRouter``:
  CUDA IPC windows, NVLink between GPUs; no send buffer, no NCCL all-to-all)
  behind the records of the lower source ranks, so each owner's window holds
  its points in global order, and the owner inserts them into its tree.  Below the top, each prefix
  subtree therefore evolves exactly as in the single-GPU run; top-node cells
  never straddle prefix boundaries (G a multiple of 2^(L-level)), so their
  claims stay rank-local (checked by the GPU tests on the merged trees).
* **render** -- every rank rasterizes its tree into its framebuffer window;
  ``PeerFramebuffers.composite`` min-reduces each rank's pixel slice across
  all windows and writes it back into every window (reduce-scatter and
  all-gather fused in one kernel over peer memory).  ``composite_min`` is the
  same composite as one ``all_reduce(MIN)`` for CPU tensors (gloo tests).

The peer-memory steps are ordered by host barriers (stream sync + barrier of
the process group) -- two per routed batch, two per composite -- never by
device-side spin waits, so ranks that share one GPU (the single-GPU test box:
``LOD_DIST_BACKEND=gloo``) cannot deadlock on each other's kernels.
"""
from __future__ import annotations

import os

import numpy as np

from . import _lib, partition

SENTINEL_U64 = np.uint64(0xFFFFFFFFFFFFFFFF)
INT64_MAX = np.iinfo(np.int64).max


def pack_tree(tree):
    """The tree's whole device state as a CUDA uint8 tensor (lod_tree_pack)."""
    import ctypes

    import torch

    nbytes = ctypes.c_uint64(0)
    _lib.check(tree._L.lod_tree_pack_size(tree.handle, ctypes.byref(nbytes)), "lod_tree_pack_size")
    buf = torch.empty(int(nbytes.value), dtype=torch.uint8, device=f"cuda:{tree.device}")
    _lib.check(tree._L.lod_tree_pack(tree.handle, _lib.ptr(buf), int(nbytes.value)), "lod_tree_pack")
    return buf


def unpack_tree(tree, buf) -> None:
    """Replace the tree's device state with a packed state (lod_tree_unpack)."""
    import torch

    torch.cuda.synchronize(buf.device)
    _lib.check(tree._L.lod_tree_unpack(tree.handle, _lib.ptr(buf), buf.numel()), "lod_tree_unpack")
    tree._invalidate()


def top_is_inner(tree, depth: int) -> bool:
    """All 8^0 + ... + 8^(depth-1) nodes above the partition depth are inner."""
    n = tree.num_nodes
    lvl, inner = tree.level[:n], tree.inner[:n]
    need = sum(8 ** k for k in range(depth))
    top = lvl < depth
    return int(top.sum()) == need and bool(inner[top].all())


def owners_device(xyz, plan: partition.Plan, bmin=(0.0, 0.0, 0.0), size: float = 1.0):
    """Owner rank of every point: exact f64 descent over the first plan.depth
    levels (_kernels.py:44-56), on the device."""
    import torch

    p = xyz.to(torch.float64)
    b = torch.tensor(bmin, dtype=torch.float64, device=p.device).expand_as(p).clone()
    s = float(size)
    key = torch.zeros(p.shape[0], dtype=torch.int64, device=p.device)
    for _ in range(plan.depth):
        h = s * 0.5
        up = p >= b + h
        b = torch.where(up, b + h, b)
        o = up[:, 0].long() | (up[:, 1].long() << 1) | (up[:, 2].long() << 2)
        key = key * 8 + o
        s = h
    owner = torch.as_tensor(plan.owner, device=p.device)
    return owner[key]


def bucket(xyz, rgba, plan: partition.Plan, world: int, bmin=(0.0, 0.0, 0.0), size: float = 1.0,
           positions: bool = False):
    """Stable bucketing of one stripe by owner rank into packed 16-byte records
    (CUDA tensors in; lod_route_bucket: owner prefix + per-tile counts, scans,
    warp-ordered stable scatter).  Returns (records (n, 4) int32, counts (world,)
    int64, starts (world,) int64), all on the device, plus with ``positions``
    every record's index in the stripe (int32)."""
    import torch

    dev = xyz.device
    n = int(rgba.shape[0])
    out = torch.empty((n, 4), dtype=torch.int32, device=dev)
    pos = torch.empty(n, dtype=torch.int32, device=dev) if positions else None
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    starts = torch.empty(world, dtype=torch.int64, device=dev)
    table = np.ascontiguousarray(plan.owner, np.int32)
    b = np.ascontiguousarray(bmin, np.float64)
    x = xyz.contiguous()
    c = rgba.contiguous()
    L = _lib.load()
    _lib.check(L.lod_route_bucket(dev.index, _lib.ptr(b), float(size), int(plan.depth), _lib.ptr(table), int(world),
                                  _lib.ptr(x), _lib.ptr(c), n, _lib.ptr(out), _lib.ptr(pos), _lib.ptr(counts),
                                  _lib.ptr(starts), torch.cuda.current_stream(dev).cuda_stream), "route_bucket")
    return (out, counts, starts, pos) if positions else (out, counts, starts)


def route(xyz, rgba, plan: partition.Plan, world: int, group=None, bmin=(0.0, 0.0, 0.0), size: float = 1.0,
          with_index: bool = False):
    """All-to-all routing of one stripe (global order) to the owners of its
    points; returns this rank's points as packed 16-byte records (n, 4) int32
    in global order (receivers concatenate by source rank), and with
    ``with_index`` each point's index in the global batch (int64; the order
    the replicated top nodes' voxels merge in).  ``bmin`` / ``size`` are the
    tree's root cube (``tree.bounds``): the octant prefix is computed against
    it, like ``partition.plan_owners`` must be.

    CUDA tensors are bucketed by the lod_route_bucket kernels; CPU tensors
    (the gloo test path) by the same rule in torch."""
    import torch
    import torch.distributed as dist

    if xyz.is_cuda:
        rec, send_counts, _, pos = bucket(xyz, rgba, plan, world, bmin, size, positions=True)
    else:
        own = owners_device(xyz, plan, bmin, size)
        order = torch.sort(own, stable=True).indices  # bucket by owner, keep order
        rec = torch.cat([xyz.contiguous().view(torch.int32), rgba.view(torch.int32).reshape(-1, 1)], dim=1)[order]
        pos = order.to(torch.int32)
        send_counts = torch.bincount(own, minlength=world).to(torch.int64)
    # every rank's stripe length -> the global index of a stripe position
    n_local = torch.tensor([int(rgba.shape[0])], dtype=torch.int64, device=send_counts.device)
    sizes = [torch.zeros_like(n_local) for _ in range(world)]
    dist.all_gather(sizes, n_local, group=group)
    stripe_off = np.concatenate([[0], np.cumsum([int(t.item()) for t in sizes])])[:-1]
    gloo_cuda = xyz.is_cuda and dist.get_backend(group) == "gloo"
    dev = xyz.device
    if gloo_cuda:  # gloo has no CUDA all-to-all: the exchange goes through host copies
        rec, send_counts, pos = rec.cpu(), send_counts.cpu(), pos.cpu()
    out, recv_counts = _all_to_all_records(rec, send_counts, group)
    if not with_index:
        return out.to(dev) if gloo_cuda else out
    got_pos, _ = _all_to_all_records(pos.reshape(-1, 1), send_counts, group)
    src = torch.repeat_interleave(torch.arange(world, device=got_pos.device), recv_counts.to(got_pos.device))
    gidx = torch.as_tensor(stripe_off, device=got_pos.device)[src] + got_pos.reshape(-1).to(torch.int64)
    if gloo_cuda:
        out, gidx = out.to(dev), gidx.to(dev)
    return out, gidx


def _all_to_all_records(rec, send_counts, group):
    import torch
    import torch.distributed as dist

    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    rc, sc = recv_counts.tolist(), send_counts.tolist()
    out = torch.empty((sum(rc),) + tuple(rec.shape[1:]), dtype=rec.dtype, device=rec.device)
    dist.all_to_all_single(out, rec.contiguous(), rc, sc, group=group)
    return out, recv_counts


def composite_min(fb_cells_dev, group=None):
    """Depth-min composite of packed u64 framebuffers (int64 CUDA tensor view)."""
    import torch
    import torch.distributed as dist

    x = fb_cells_dev
    sent = x == -1  # all-ones sentinel as int64
    x = torch.where(sent, torch.full_like(x, INT64_MAX), x)
    dist.all_reduce(x, op=dist.ReduceOp.MIN, group=group)
    return torch.where(x == INT64_MAX, torch.full_like(x, -1), x)


class _DeviceArray:
    """Zero-copy torch view of raw device memory (``__cuda_array_interface__``)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 2, "strides": None}


def _device_view(ptr: int, shape, dtype, device: int):
    import torch

    typestr = {torch.int32: "<i4", torch.int64: "<i8"}[dtype]
    return torch.as_tensor(_DeviceArray(ptr, shape, typestr), device=f"cuda:{device}")


class PeerUnavailable(RuntimeError):
    """Some rank cannot map another rank's window (no CUDA IPC / P2P path
    between the GPUs); raised on every rank together."""


class PeerWindows:
    """One IPC-shareable device allocation per rank, mapped by every rank
    (``lod_ipc_alloc`` / ``lod_ipc_open``: NVLink peer memory between GPUs).
    ``ptrs[r]`` is rank r's window as seen by this process.  Collective:
    every rank of the group constructs and closes it together."""

    def __init__(self, device: int, rank: int, world: int, nbytes: int, group=None):
        import ctypes

        import torch.distributed as dist

        self.device, self.rank, self.world, self.group, self.nbytes = device, rank, world, group, int(nbytes)
        L = self._L = _lib.load()
        own = ctypes.c_void_p()
        h = ctypes.create_string_buffer(_lib.LOD_IPC_HANDLE_BYTES)
        _lib.check(L.lod_ipc_alloc(device, self.nbytes, ctypes.byref(own), h), "lod_ipc_alloc")
        self.own = int(own.value)
        import torch

        handles = [None] * world
        uuid = str(torch.cuda.get_device_properties(device).uuid)
        dist.all_gather_object(handles, (bytes(h.raw), uuid), group=group)
        # ranks time-sliced on one device: the route's waits poll from the
        # host (a spinning wait kernel would hold the device for a time slice)
        self.shared_device = len({u for _, u in handles}) < world
        forced = os.environ.get("LOD_ROUTE_WAIT", "")  # "device" / "host": force a mode (tests)
        if forced in ("device", "host"):
            self.shared_device = forced == "host"
        handles = [hb for hb, _ in handles]
        self.ptrs = (ctypes.c_void_p * world)()
        self._opened = []
        err = ""
        for r in range(world):
            if r == rank:
                self.ptrs[r] = self.own
                continue
            p = ctypes.c_void_p()
            hb = ctypes.create_string_buffer(handles[r], _lib.LOD_IPC_HANDLE_BYTES)
            rc = L.lod_ipc_open(device, hb, ctypes.byref(p))
            if rc != _lib.LOD_OK:
                err = f"rank {rank} cannot map rank {r}'s window: {L.lod_strerror(rc).decode()}"
                break
            self.ptrs[r] = p.value
            self._opened.append(int(p.value))
        errs = [None] * world
        dist.all_gather_object(errs, err, group=group)  # every rank takes the same decision
        bad = [e for e in errs if e]
        if bad:
            for q in self._opened:
                L.lod_ipc_close(ctypes.c_void_p(q))
            dist.barrier(group=group)
            L.lod_device_free(ctypes.c_void_p(self.own))
            self.own, self._opened = None, []
            raise PeerUnavailable(bad[0])

    def close(self) -> None:
        import torch
        import torch.distributed as dist

        if self.own is None:
            return
        torch.cuda.synchronize(self.device)
        dist.barrier(group=self.group)  # nobody writes into a window that is about to go
        for p in self._opened:
            _lib.check(self._L.lod_ipc_close(p), "lod_ipc_close")
        dist.barrier(group=self.group)
        _lib.check(self._L.lod_device_free(self.own), "lod_device_free")
        self.own, self._opened = None, []


def _sync_barrier(device: int, group) -> None:
    import torch
    import torch.distributed as dist

    torch.cuda.current_stream(device).synchronize()
    dist.barrier(group=group)


class PeerRouter:
    """Routing of striped batches to the owners of their octant prefixes over
    peer memory (``lod_route_peers_begin`` / ``_finish``): the bucket sizes
    are exchanged through every window's count matrix, then the stable bucket
    scatter stores each record directly in its owner's window.  The ranks
    synchronise through sequence flags in the windows (system-scope release /
    acquire on the device, one mapped host word for the matrix) -- no process
    group barrier and no stream sync per batch.  Windows hold two halves of
    ``half_records`` records (batches alternate halves) and grow collectively
    -- every rank reads the same full count matrix, so all ranks take the
    same decision (the only step that uses the process group)."""

    def __init__(self, device: int, rank: int, world: int, plan: partition.Plan, half_records: int = 1 << 20,
                 group=None, bmin=(0.0, 0.0, 0.0), size: float = 1.0):
        self.device, self.rank, self.world, self.group, self.plan = device, rank, world, group, plan
        self.table = np.ascontiguousarray(plan.owner, np.int32)
        self.bmin, self.size = np.ascontiguousarray(bmin, np.float64), float(size)
        self.half_records = int(half_records)
        self.win = PeerWindows(device, rank, world, self._bytes(self.half_records), group)
        self.k = 0
        self.matrix = np.zeros((world, world), np.int64)
        self.extra = np.zeros(world, np.int64)

    @staticmethod
    def _bytes(half_records: int) -> int:
        # header | records half 0 | records half 1 | positions half 0 | positions half 1
        return _lib.LOD_WINDOW_HEADER_BYTES + 2 * 16 * half_records + 2 * 4 * half_records

    def _begin(self, x, n: int, stream: int, extra_dev) -> None:
        import ctypes

        _lib.check(self.win._L.lod_route_peers_begin(
            self.device, _lib.ptr(self.bmin), self.size, int(self.plan.depth), _lib.ptr(self.table), self.world,
            self.rank, _lib.ptr(x), n, self.win.ptrs, self.k & 1, self.k + 1,
            None if extra_dev is None else _lib.ptr(extra_dev), _lib.ptr(self.matrix), _lib.ptr(self.extra),
            int(self.win.shared_device), ctypes.c_void_p(stream)), "lod_route_peers_begin")

    def route(self, xyz, rgba, extra_dev=None):
        """This rank's stripe (CUDA tensors) in; this rank's points of the
        global batch out, as an (n, 4) int32 view of its window in global order
        (valid until the batch after next is routed; the current stream waits
        on the device until every source's records are in).  ``extra_dev``:
        an optional int64 CUDA scalar published with this rank's counts;
        afterwards ``self.extra[r]`` holds rank r's."""
        import ctypes

        import torch

        x, c = xyz.contiguous(), rgba.contiguous()
        n = int(c.shape[0])
        stream = torch.cuda.current_stream(self.device).cuda_stream
        self._begin(x, n, stream, extra_dev)
        need = int(self.matrix.sum(axis=0).max())
        if need > self.half_records:  # identical decision on every rank (collective re-allocation)
            self.win.close()
            self.half_records = max(need, 2 * self.half_records)
            self.win = PeerWindows(self.device, self.rank, self.world, self._bytes(self.half_records), self.group)
            self._begin(x, n, stream, extra_dev)  # fresh windows: the counts again
        half = self.k & 1
        _lib.check(self.win._L.lod_route_peers_finish(
            self.device, self.world, self.rank, _lib.ptr(x), _lib.ptr(c), n, self.win.ptrs, half,
            self.half_records, self.k + 1, int(self.win.shared_device), ctypes.c_void_p(stream)),
            "lod_route_peers_finish")
        self.k += 1
        mine = int(self.matrix[:, self.rank].sum())
        base = self.win.own + _lib.LOD_WINDOW_HEADER_BYTES + half * 16 * self.half_records
        pbase = self.win.own + _lib.LOD_WINDOW_HEADER_BYTES + 2 * 16 * self.half_records + half * 4 * self.half_records
        self.last_positions = _device_view(pbase, (mine,), torch.int32, self.device)
        return _device_view(base, (mine, 4), torch.int32, self.device)

    def global_index(self):
        """Global-batch index of every record of the last route(): the
        records from source s sit behind the lower sources' (column of the
        count matrix) and carry their position in s's stripe."""
        import torch

        col = self.matrix[:, self.rank]
        stripe_off = np.concatenate([[0], np.cumsum(self.matrix.sum(axis=1))])[:-1]
        dev = self.last_positions.device
        src = torch.repeat_interleave(torch.arange(self.world, device=dev), torch.as_tensor(col, device=dev),
                                      output_size=int(col.sum()))  # no device sync
        return torch.as_tensor(stripe_off, device=dev)[src] + self.last_positions.to(torch.int64)

    def close(self) -> None:
        self.win.close()


class PeerFramebuffers:
    """Per-rank framebuffer windows and the fused depth-min composite
    (``lod_composite_min_peers``)."""

    def __init__(self, device: int, rank: int, world: int, width: int, height: int, group=None):
        self.device, self.rank, self.world, self.group = device, rank, world, group
        self.width, self.height = int(width), int(height)
        self.npix = self.width * self.height
        self.win = PeerWindows(device, rank, world, 8 * self.npix, group)

    def render(self, tree, camera, plan: partition.Plan, threshold: float = 128.0) -> int:
        """Clear this rank's framebuffer and splat its share of the cut into
        it: the device selection (render.select_visible) restricted to the
        replicated top and the prefixes this rank owns (its copies of other
        prefixes are frozen at the hand-off), drawn by ``lod_rasterize`` into
        the window.  Returns the samples drawn."""
        import ctypes

        from . import render as R

        L = self.win._L
        _lib.check(L.lod_fb_fill(self.device, self.win.own, self.npix, int(SENTINEL_U64)), "fb fill")
        vis = np.asarray(owned_cut(tree, R.select_visible(tree, camera, threshold), plan, self.rank), np.int32)
        cam = np.ascontiguousarray(camera.packed(), np.float64)
        drawn = ctypes.c_int64(0)
        _lib.check(L.lod_rasterize(tree.handle, _lib.ptr(vis), len(vis), _lib.ptr(cam),
                                   ctypes.c_void_p(self.win.own), self.width, self.height, _lib.LOD_FLAG_DEVICE_FB,
                                   ctypes.byref(drawn)), "lod_rasterize")
        return int(drawn.value)

    def composite(self):
        """Depth-min of all ranks' framebuffers (collective); returns it as a
        host Framebuffer (every rank's window holds the same composite)."""
        import ctypes

        import torch

        from .render import Framebuffer

        _sync_barrier(self.device, self.group)
        stream = torch.cuda.current_stream(self.device).cuda_stream
        _lib.check(self.win._L.lod_composite_min_peers(self.device, self.world, self.rank, self.win.ptrs, self.npix,
                                                       ctypes.c_void_p(stream)), "lod_composite_min_peers")
        _sync_barrier(self.device, self.group)
        fb = Framebuffer(self.width, self.height)
        _lib.check(self.win._L.lod_memcpy_d2h(_lib.ptr(fb.cells), self.win.own, 8 * self.npix), "fb read")
        return fb

    def close(self) -> None:
        self.win.close()


def owned_cut(tree, selected, plan: partition.Plan, rank: int) -> list[int]:
    """The nodes of a selection this rank draws: the replicated top (level <
    plan.depth) and the nodes under the prefixes it owns."""
    par, octs, lvl = tree.parent, tree.octant, tree.level
    keep = []
    for nid in selected:
        if lvl[nid] < plan.depth:
            keep.append(nid)
            continue
        a = nid
        while lvl[a] > plan.depth:
            a = par[a]
        prefix, k = 0, 1
        while lvl[a] > 0:  # octants of the depth-`plan.depth` ancestor's path, deepest first
            prefix += int(octs[a]) * k
            k *= 8
            a = par[a]
        if int(plan.owner[prefix]) == rank:
            keep.append(nid)
    return keep


def last_top_voxels(tree, depth: int):
    """(node, cell, rgba, winner) of the voxels the tree's last insert created
    at nodes above the partition depth (level < depth), the winner as its
    batch position (lod_last_voxels; in no particular order)."""
    import ctypes

    L = tree._L
    n = ctypes.c_int64(0)
    _lib.check(L.lod_last_voxels(tree.handle, int(depth), 0, None, None, None, None, ctypes.byref(n)), "last_voxels")
    k = int(n.value)
    node, cell = np.empty(k, np.int32), np.empty(k, np.uint32)
    rgba, win = np.empty(k, np.uint32), np.empty(k, np.int64)
    if k:
        _lib.check(L.lod_last_voxels(tree.handle, int(depth), k, _lib.ptr(node), _lib.ptr(cell), _lib.ptr(rgba),
                                     _lib.ptr(win), ctypes.byref(n)), "last_voxels")
    assert (win >= 0).all(), "a spilled point claimed a replicated top-node cell"
    return node, cell, rgba, win


def merge_top_voxels(tree, own_nodes: np.ndarray, everyone) -> int:
    """Make this rank's copies of the replicated top nodes hold the
    single-tree voxel sequences ("all-gathered and merged by
    global index").  ``everyone`` lists every rank's (node, cell, rgba,
    global index) of the voxels its last cycle created at top nodes --
    top-node cells split along prefix boundaries, so each cell was claimed on
    exactly one rank and the winners are the single tree's; only their order
    in a node's sequence interleaves across ranks: ascending global index.
    ``own_nodes``: the node column of this rank's own items.  Each top node
    that got voxels anywhere is rewritten from the position its sequence had
    before the cycle (lod_merge_voxels).  Returns the voxels merged."""
    import ctypes

    node = np.concatenate([np.asarray(e[0], np.int32) for e in everyone])
    if not len(node):
        return 0
    cell = np.concatenate([np.asarray(e[1], np.uint32) for e in everyone])
    rgba = np.concatenate([np.asarray(e[2], np.uint32) for e in everyone])
    gidx = np.concatenate([np.asarray(e[3], np.int64) for e in everyone])
    order = np.lexsort((gidx, node))  # by node, then global index
    node, cell, rgba = node[order], np.ascontiguousarray(cell[order]), np.ascontiguousarray(rgba[order])
    gnode, first = np.unique(node, return_index=True)
    goff = np.append(first, len(node)).astype(np.int64)
    own = np.bincount(np.asarray(own_nodes, np.int64), minlength=int(gnode.max()) + 1)
    gstart = (tree.count[gnode] - own[gnode]).astype(np.int64)
    gnode = gnode.astype(np.int32)
    _lib.check(tree._L.lod_merge_voxels(tree.handle, len(gnode), _lib.ptr(gnode), _lib.ptr(gstart), _lib.ptr(goff),
                                        _lib.ptr(cell), _lib.ptr(rgba)), "merge_voxels")
    tree._invalidate()
    return len(node)


def check_plan(tree, plan: partition.Plan) -> None:
    """The partition invariants the protocol relies on: the plan covers every
    depth-L prefix, and no cell of a replicated top node straddles a prefix
    boundary (the split planes down to depth L coincide with cell faces iff
    grid_res is a multiple of 2^L), so top-node claims stay rank-local."""
    if len(plan.owner) != 8 ** plan.depth:
        raise ValueError(f"plan has {len(plan.owner)} owners for depth {plan.depth}")
    if tree.grid_res % (1 << plan.depth):
        raise ValueError(f"grid_res {tree.grid_res} is not a multiple of 2^{plan.depth}: top-node cells would "
                         "straddle prefix boundaries")


class PartitionedInserter:
    """Drives one rank of the warm-up / hand-off / partitioned protocol.
    Owners are computed against ``tree.bounds`` (the root cube); ``plan``
    must have been made with the same bounds (``partition.plan_owners(...,
    bmin=tree.bounds.min, size=tree.bounds.size)``)."""

    def __init__(self, tree, state, plan: partition.Plan, rank: int, world: int, group=None):
        check_plan(tree, plan)
        self.tree, self.state, self.plan = tree, state, plan
        self.rank, self.world, self.group = rank, world, group
        self.bmin = tuple(float(v) for v in tree.bounds.min)
        self.size = float(tree.bounds.size)
        self.partitioned = world == 1
        self.router = None  # PeerRouter, created at the first partitioned batch
        self.no_peers = ""  # why the peer route is unavailable (then: NCCL all-to-all)
        self.merged_top = 0  # top-node voxels merged across ranks so far
        self.flushes = 0  # top-voxel log merges (peer route)
        self.flush_at = int(os.environ.get("LOD_TOP_FLUSH_AT", 1 << 22))  # merge when some rank's log holds more
        # peer route: this rank's replicated-top voxels since the last merge,
        # on the device (node, cell, rgba, order key = batch << 40 | global index)
        self._log = None
        self._log_count = None  # int64 CUDA scalar: entries appended (published with the counts)
        self._log_used = 0  # its value as of the last route
        self._batch = 0

    def insert(self, xyz, rgba) -> int:
        """Insert this rank's stripe of one global batch; returns points inserted here.
        With the peer route, the voxels each rank creates at the replicated
        top nodes go to a device log and are merged across ranks when a log
        fills up or at ``flush`` (collective) -- not per batch.  Claims are
        unaffected (each top-node cell is claimed on exactly one rank), and a
        depth-min composite of the ranks' renders is the same either way;
        only a rank's own copy of a top node lacks the other ranks' voxels
        until the merge."""
        import ctypes

        import torch
        import torch.distributed as dist

        from .update import insert_batch, insert_records

        if self.partitioned:
            if self.world == 1:
                insert_batch(self.tree, xyz, rgba, self.state)
                return int(rgba.shape[0])
            if xyz.is_cuda and self.router is None and not self.no_peers:
                try:
                    self.router = PeerRouter(self.tree.device, self.rank, self.world, self.plan,
                                             half_records=2 * int(rgba.shape[0]), group=self.group,
                                             bmin=self.bmin, size=self.size)
                    self._log_count = torch.zeros(1, dtype=torch.int64, device=xyz.device)
                except PeerUnavailable as e:  # GPUs without a peer path: route with the collective
                    self.no_peers = str(e)
            if self.router is not None:
                # every rank's top-voxel log fill rides on the count exchange,
                # so all ranks take the same flush decision without a collective
                rec = self.router.route(xyz, rgba, extra_dev=self._log_count)
                self._log_used = int(self.router.extra[self.rank])
                if int(self.router.extra.max()) > self.flush_at:
                    self._flush_log(self._log_used)
                gidx = self.router.global_index()
                insert_records(self.tree, rec, self.state)
                nv = max(int(self.state._bstats.n_voxels), 0)  # bounds this batch's top voxels
                self._ensure_log(self._log_used + nv)
                stream = torch.cuda.current_stream(self.tree.device).cuda_stream
                lg = self._log
                _lib.check(self.tree._L.lod_last_voxels_log(
                    self.tree.handle, int(self.plan.depth), _lib.ptr(gidx), self._batch << 40, _lib.ptr(lg[0]),
                    _lib.ptr(lg[1]), _lib.ptr(lg[2]), _lib.ptr(lg[3]), int(lg[0].shape[0]), _lib.ptr(self._log_count),
                    ctypes.c_void_p(stream)), "last_voxels_log")
                self._batch += 1
                return int(rec.shape[0])
            rec, gidx = route(xyz, rgba, self.plan, self.world, self.group, self.bmin, self.size, with_index=True)
            insert_records(self.tree, rec, self.state)
            self._merge_top(gidx)
            return int(rec.shape[0])
        # warm-up: gather stripes to rank 0 (rank order = global order)
        n = torch.tensor([rgba.shape[0]], dtype=torch.int64, device=xyz.device)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        dist.all_gather(sizes, n, group=self.group)
        rec = torch.cat([xyz.contiguous().view(torch.int32), rgba.view(torch.int32).reshape(-1, 1)], dim=1)
        mx = int(max(s.item() for s in sizes))
        padded = torch.zeros((mx, 4), dtype=torch.int32, device=xyz.device)
        padded[: rec.shape[0]] = rec
        bufs = [torch.empty_like(padded) for _ in range(self.world)]
        dist.all_gather(bufs, padded, group=self.group)
        got = 0
        if self.rank == 0:
            allrec = torch.cat([b[: int(s.item())] for b, s in zip(bufs, sizes)])
            insert_records(self.tree, allrec, self.state)
            got = int(allrec.shape[0])
        flag = torch.tensor([1 if (self.rank == 0 and top_is_inner(self.tree, self.plan.depth)) else 0],
                            device=xyz.device)
        dist.broadcast(flag, 0, group=self.group)
        if int(flag.item()):
            self.hand_off()
        return got

    def _merge_top(self, gidx) -> None:
        """All-gather the top-node voxels of this batch with their winners'
        global indices and merge them into every rank's top nodes."""
        import torch
        import torch.distributed as dist

        node, cell, rgba, win = last_top_voxels(self.tree, self.plan.depth)
        g = gidx[torch.from_numpy(win).to(gidx.device)].cpu().numpy() if len(win) else np.empty(0, np.int64)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, (node, cell, rgba, g), group=self.group)
        self.merged_top += merge_top_voxels(self.tree, node, everyone)

    def _ensure_log(self, n: int) -> None:
        import torch

        cap = 0 if self._log is None else int(self._log[0].shape[0])
        if n <= cap:
            return
        new_cap = max(n, 2 * cap, 1 << 16)
        dev = self._log_count.device
        lg = (torch.empty(new_cap, dtype=torch.int32, device=dev), torch.empty(new_cap, dtype=torch.int32, device=dev),
              torch.empty(new_cap, dtype=torch.int32, device=dev), torch.empty(new_cap, dtype=torch.int64, device=dev))
        if self._log is not None and self._log_used:
            for a, b in zip(lg, self._log):
                a[: self._log_used].copy_(b[: self._log_used])
        self._log = lg

    def _flush_log(self, used: int) -> None:
        """Merge every rank's logged top voxels (collective: all ranks call
        it with their own entry count) and empty the logs."""
        import torch.distributed as dist

        if used:
            node = self._log[0][:used].cpu().numpy()
            cell = self._log[1][:used].cpu().numpy().view(np.uint32)
            rgba = self._log[2][:used].cpu().numpy().view(np.uint32)
            key = self._log[3][:used].cpu().numpy()
        else:
            node, cell, rgba = np.empty(0, np.int32), np.empty(0, np.uint32), np.empty(0, np.uint32)
            key = np.empty(0, np.int64)
        everyone = [None] * self.world
        dist.all_gather_object(everyone, (node, cell, rgba, key), group=self.group)
        self.merged_top += merge_top_voxels(self.tree, node, everyone)
        self._log_count.zero_()
        self._log_used = 0
        self.flushes += 1

    def flush(self) -> None:
        """Merge the replicated-top voxels logged since the last merge
        (collective; before reading a rank's top nodes as the single tree's)."""
        if self._log_count is not None:
            self._flush_log(int(self._log_count.item()))

    def close(self) -> None:
        """Merge what is pending and release the peer windows (collective)."""
        self.flush()
        if self.router is not None:
            self.router.close()
            self.router = None

    def hand_off(self) -> None:
        import torch
        import torch.distributed as dist

        if self.rank == 0:
            buf = pack_tree(self.tree)
            size = torch.tensor([buf.numel()], dtype=torch.int64, device=buf.device)
        else:
            size = torch.zeros(1, dtype=torch.int64, device=f"cuda:{self.tree.device}")
        dist.broadcast(size, 0, group=self.group)
        if self.rank != 0:
            buf = torch.empty(int(size.item()), dtype=torch.uint8, device=f"cuda:{self.tree.device}")
        dist.broadcast(buf, 0, group=self.group)
        if self.rank != 0:
            unpack_tree(self.tree, buf)
        self.partitioned = True
