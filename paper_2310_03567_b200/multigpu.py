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
  their depth-L octant prefix (exact float64 descent rule on the device),
  buckets them stably by owner, and one ``all_to_all_single`` routes 16-byte
  records to their owners; receivers concatenate by source rank, which is
  global order, and insert into their tree.  Below the top, each prefix
  subtree therefore evolves exactly as in the single-GPU run; top-node cells
  never straddle prefix boundaries (G a multiple of 2^(L-level)), so their
  claims stay rank-local (checked by the GPU tests on the merged trees).
* **render** -- every rank rasterizes its tree; framebuffers are combined with
  one ``all_reduce(MIN)`` (the all-ones sentinel is mapped to INT64_MAX for the
  signed reduction and back).
"""
from __future__ import annotations

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


def bucket(xyz, rgba, plan: partition.Plan, world: int, bmin=(0.0, 0.0, 0.0), size: float = 1.0):
    """Stable bucketing of one stripe by owner rank into packed 16-byte records
    (CUDA tensors in; lod_route_bucket: owner prefix + per-tile counts, scans,
    warp-ordered stable scatter).  Returns (records (n, 4) int32, counts (world,)
    int64, starts (world,) int64), all on the device."""
    import torch

    dev = xyz.device
    n = int(rgba.shape[0])
    out = torch.empty((n, 4), dtype=torch.int32, device=dev)
    counts = torch.empty(world, dtype=torch.int64, device=dev)
    starts = torch.empty(world, dtype=torch.int64, device=dev)
    table = np.ascontiguousarray(plan.owner, np.int32)
    b = np.ascontiguousarray(bmin, np.float64)
    x = xyz.contiguous()
    c = rgba.contiguous()
    L = _lib.load()
    _lib.check(L.lod_route_bucket(dev.index, _lib.ptr(b), float(size), int(plan.depth), _lib.ptr(table), int(world),
                                  _lib.ptr(x), _lib.ptr(c), n, _lib.ptr(out), _lib.ptr(counts), _lib.ptr(starts),
                                  torch.cuda.current_stream(dev).cuda_stream), "route_bucket")
    return out, counts, starts


def route(xyz, rgba, plan: partition.Plan, world: int, group=None):
    """All-to-all routing of one stripe (global order) to the owners of its
    points; returns this rank's points as packed 16-byte records (n, 4) int32
    in global order (receivers concatenate by source rank).

    CUDA tensors are bucketed by the lod_route_bucket kernels; CPU tensors
    (the gloo test path) by the same rule in torch."""
    import torch
    import torch.distributed as dist

    if xyz.is_cuda:
        rec, send_counts, _ = bucket(xyz, rgba, plan, world)
    else:
        own = owners_device(xyz, plan)
        order = torch.sort(own, stable=True).indices  # bucket by owner, keep order
        rec = torch.cat([xyz.contiguous().view(torch.int32), rgba.view(torch.int32).reshape(-1, 1)], dim=1)[order]
        send_counts = torch.bincount(own, minlength=world).to(torch.int64)
    if xyz.is_cuda and dist.get_backend(group) == "gloo":
        # gloo has no CUDA all-to-all: the exchange goes through host copies
        # (single-box validation of this path; NCCL moves device memory)
        out = _all_to_all_records(rec.cpu(), send_counts.cpu(), group)
        return out.to(xyz.device)
    return _all_to_all_records(rec, send_counts, group)


def _all_to_all_records(rec, send_counts, group):
    import torch
    import torch.distributed as dist

    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    rc, sc = recv_counts.tolist(), send_counts.tolist()
    out = torch.empty((sum(rc), 4), dtype=torch.int32, device=rec.device)
    dist.all_to_all_single(out, rec.contiguous(), rc, sc, group=group)
    return out


def composite_min(fb_cells_dev, group=None):
    """Depth-min composite of packed u64 framebuffers (int64 CUDA tensor view)."""
    import torch
    import torch.distributed as dist

    x = fb_cells_dev
    sent = x == -1  # all-ones sentinel as int64
    x = torch.where(sent, torch.full_like(x, INT64_MAX), x)
    dist.all_reduce(x, op=dist.ReduceOp.MIN, group=group)
    return torch.where(x == INT64_MAX, torch.full_like(x, -1), x)


class PartitionedInserter:
    """Drives one rank of the warm-up / hand-off / partitioned protocol."""

    def __init__(self, tree, state, plan: partition.Plan, rank: int, world: int, group=None):
        self.tree, self.state, self.plan = tree, state, plan
        self.rank, self.world, self.group = rank, world, group
        self.partitioned = world == 1

    def insert(self, xyz, rgba) -> int:
        """Insert this rank's stripe of one global batch; returns points inserted here."""
        import torch
        import torch.distributed as dist

        from .update import insert_batch, insert_records

        if self.partitioned:
            if self.world == 1:
                insert_batch(self.tree, xyz, rgba, self.state)
                return int(rgba.shape[0])
            rec = route(xyz, rgba, self.plan, self.world, self.group)
            insert_records(self.tree, rec, self.state)
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
