"""CPU tests of the multi-GPU host logic: octant-prefix keys, LPT ownership,
order-preserving per-rank routing, and a world_size-2 gloo exchange."""
import os

import numpy as np
import pytest

from paper_2310_03567_b200 import partition, synth


def _slow_prefix(p, depth, bmin=(0.0, 0.0, 0.0), size=1.0):
    """The reference's descent rule (_kernels.py:44-56), one point at a time."""
    bx, by, bz = (float(v) for v in bmin)
    s = float(size)
    key = 0
    x, y, z = (float(v) for v in p)
    for _ in range(depth):
        h = s * 0.5
        o = 0
        if x >= bx + h:
            o |= 1
            bx += h
        if y >= by + h:
            o |= 2
            by += h
        if z >= bz + h:
            o |= 4
            bz += h
        s = h
        key = key * 8 + o
    return key


def test_prefix_matches_reference_descent_rule():
    xyz, _ = synth.gen_surface(2000, 3)
    edgy = np.array([[0.5, 0.5, 0.5], [0.25, 0.75, 0.5], [0.0, 0.999, 0.125]], np.float32)
    pts = np.concatenate([xyz, edgy])
    for depth in (1, 2, 3):
        got = partition.prefix_of(pts, depth)
        want = [_slow_prefix(p, depth) for p in pts]
        assert got.tolist() == want


def test_prefix_offset_root():
    rng = np.random.default_rng(1)
    pts = (rng.random((500, 3)) * 6.5 + np.array([-3.0, 2.5, 10.0])).astype(np.float32)
    got = partition.prefix_of(pts, 2, (-3.0, 2.5, 10.0), 6.5)
    assert got.tolist() == [_slow_prefix(p, 2, (-3.0, 2.5, 10.0), 6.5) for p in pts]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_lpt_balance_on_terrain(world):
    sample = [synth.gen_surface(200_000, 10 + i) for i in range(2)]
    plan = partition.plan_owners(sample, world)
    assert plan.depth == (1 if world <= 4 else 2)
    assert set(np.unique(plan.owner[plan.owner >= 0])) <= set(range(world))
    # LPT over level-1 octants ~1.00 for 2/4, level-2 ~1.05 for 8
    assert partition.imbalance(plan) < (1.02 if world <= 4 else 1.10)


def test_take_partitions_and_keeps_order():
    xyz, rgba = synth.gen_surface(50_000, 5)
    rgba = np.arange(len(rgba), dtype=np.uint32)  # colour = global index
    plan = partition.plan_owners([(xyz, rgba)], 4)
    parts = [partition.take(plan, xyz, rgba, r) for r in range(4)]
    assert sum(len(c) for _, c in parts) == len(rgba)
    seen = np.concatenate([c for _, c in parts])
    assert np.array_equal(np.sort(seen), rgba)
    for x, c in parts:
        assert np.all(np.diff(c.astype(np.int64)) > 0)  # global order within a rank
        assert np.array_equal(x, xyz[c])


def _exchange_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    xyz, rgba = synth.gen_surface(20_000, 7)
    gidx = np.arange(len(rgba), dtype=np.int64)
    plan = partition.plan_owners([(xyz, rgba)], world)
    stripe = slice(rank * len(rgba) // world, (rank + 1) * len(rgba) // world)
    owners = plan.owner[partition.prefix_of(xyz[stripe], plan.depth)]
    order = np.argsort(owners, kind="stable")  # bucket by owner, keep global order
    send = torch.from_numpy(gidx[stripe][order].copy())
    counts = torch.from_numpy(np.bincount(owners, minlength=world).astype(np.int64))
    recv_counts = torch.empty_like(counts)
    dist.all_to_all_single(recv_counts, counts)
    recv = torch.empty(int(recv_counts.sum()), dtype=torch.int64)
    dist.all_to_all_single(recv, send, recv_counts.tolist(), counts.tolist())
    got = recv.numpy()
    want = gidx[plan.owner[partition.prefix_of(xyz, plan.depth)] == rank]
    out[rank] = bool(np.array_equal(got, want))
    dist.destroy_process_group()


def test_gloo_all_to_all_routing_preserves_global_order():
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    assert dict(out) == {0: True, 1: True}


OFFSET_ROOT = ((-3.0, 2.5, 10.0), 6.5)  # a cubified, non-unit, non-power-of-two root


def _route_worker(rank, world, port, out):
    """multigpu.route + composite_min with CPU tensors over gloo (the NCCL path's
    logic), for the unit cube and for an offset non-unit root (the owners must
    be computed against the tree's bounds, not the unit cube)."""
    import torch
    import torch.distributed as dist

    from paper_2310_03567_b200 import multigpu

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ok = True
    for bmin, size in (((0.0, 0.0, 0.0), 1.0), OFFSET_ROOT):
        xyz, _ = synth.gen_surface(12_000, 9)
        xyz = (xyz.astype(np.float64) * size + np.asarray(bmin)).astype(np.float32)
        rgba = np.arange(len(xyz), dtype=np.uint32)  # colour = global index
        plan = partition.plan_owners([(xyz, rgba)], world, bmin=bmin, size=size)
        assert len(np.unique(plan.owner[partition.prefix_of(xyz, plan.depth, bmin, size)])) == world
        n = len(rgba)
        st = slice(rank * n // world, (rank + 1) * n // world)
        rec = multigpu.route(torch.from_numpy(xyz[st].copy()), torch.from_numpy(rgba[st].view(np.int32).copy()),
                             plan, world, bmin=bmin, size=size).numpy()
        want_x, want_c = partition.take(plan, xyz, rgba, rank, bmin, size)
        ok = ok and np.array_equal(rec[:, :3].copy().view(np.float32), want_x) and np.array_equal(
            rec[:, 3].view(np.uint32), want_c)
    # framebuffer min-composite with the all-ones sentinel
    rng = np.random.default_rng(rank)
    fb = np.full(64, np.uint64(0xFFFFFFFFFFFFFFFF))
    hit = rng.choice(64, 20, replace=False)
    fb[hit] = rng.integers(0, 1 << 62, 20).astype(np.uint64)
    comp = multigpu.composite_min(torch.from_numpy(fb.view(np.int64).copy())).numpy().view(np.uint64)
    allfb = [torch.zeros(64, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(allfb, torch.from_numpy(fb.view(np.int64).copy()))
    want_fb = np.minimum.reduce([a.numpy().view(np.uint64) for a in allfb])
    out[rank] = bool(ok and np.array_equal(comp, want_fb))
    dist.destroy_process_group()


def test_gloo_route_and_composite():
    import multiprocessing as mp
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    out = ctx.Manager().dict()
    procs = [ctx.Process(target=_route_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs)
    assert dict(out) == {0: True, 1: True}


def test_owned_cut_keeps_top_and_owned_prefixes():
    """multigpu.owned_cut on a synthetic node table: a full tree to depth 3
    (ids in creation order, octant order); a node is kept iff it is above
    the partition depth or the owner of its depth-L octant prefix is the rank."""
    from types import SimpleNamespace

    from paper_2310_03567_b200 import multigpu

    parent, octant, level, paths = [-1], [0], [0], [()]
    frontier = [0]
    for _ in range(3):
        nxt = []
        for nid in frontier:
            for o in range(8):
                parent.append(nid)
                octant.append(o)
                level.append(level[nid] + 1)
                paths.append(paths[nid] + (o,))
                nxt.append(len(parent) - 1)
        frontier = nxt
    tree = SimpleNamespace(parent=np.array(parent, np.int32), octant=np.array(octant, np.uint8),
                           level=np.array(level, np.int32))
    rng = np.random.default_rng(4)
    for depth, world in ((1, 2), (2, 4), (2, 8)):
        plan = partition.Plan(depth=depth, owner=rng.integers(0, world, 8 ** depth).astype(np.int32),
                              load=np.zeros(world))
        sel = list(rng.permutation(len(parent)))
        kept = [set(multigpu.owned_cut(tree, sel, plan, r)) for r in range(world)]
        for nid in sel:
            p = paths[nid]
            if len(p) < depth:
                assert all(nid in k for k in kept)
                continue
            key = 0
            for o in p[:depth]:
                key = key * 8 + o
            owners = [r for r in range(world) if nid in kept[r]]
            assert owners == [int(plan.owner[key])], (nid, p)
        # order of the selection is preserved
        assert multigpu.owned_cut(tree, sel, plan, 0) == [n for n in sel if n in kept[0]]
