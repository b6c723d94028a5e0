"""The multi-GPU protocol on one GPU: N emulated ranks = N trees.

Warm-up batches go to rank 0 until the top is inner; its state is packed and
unpacked into the other ranks (lod_tree_pack/unpack); later batches are routed
by exact octant prefix.  Every prefix subtree of its owner must equal the
single-tree run path by path; top nodes must hold the common prefix plus
rank-disjoint new voxels whose union is the single-tree sequence; and the
min-composite of the ranks' renders must equal the single-tree render.
"""
import numpy as np
import pytest

from common import make_product

pytestmark = pytest.mark.gpu

P = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=512 << 20, chunk_capacity=256, grid_res=32,
         leaf_threshold=400, max_depth=14, backlog_capacity=10_000_000, spill_capacity=100_000_000)


def _paths(tree):
    from oracle.rebuild import tree_paths

    return tree_paths(tree.inner, tree.children)


def _samples(tree, nid):
    x, c = tree.gather_samples(nid)
    return np.concatenate([x.view(np.uint32), c.reshape(-1, 1)], axis=1)


@pytest.mark.parametrize("world", [2, 4])
def test_partitioned_ranks_match_single_tree(gpu, world):
    from paper_2310_03567_b200 import insert_batch, multigpu, partition, synth
    from paper_2310_03567_b200.render import Camera, Framebuffer, rasterize

    batches = [synth.gen_surface(40_000, 300 + i) for i in range(12)]
    plan = partition.plan_owners(batches[:2], world, depth=1)
    g, gs = make_product(P)
    ranks = [make_product(P) for _ in range(world)]
    handed_off = False
    pre = None
    for x, c in batches:
        insert_batch(g, x, c, gs)
        if not handed_off:
            insert_batch(ranks[0][0], x, c, ranks[0][1])
            if multigpu.top_is_inner(ranks[0][0], plan.depth):
                buf = multigpu.pack_tree(ranks[0][0])
                for r in range(1, world):
                    multigpu.unpack_tree(ranks[r][0], buf)
                handed_off = True
                pre = {p: _samples(ranks[0][0], nid) for p, nid in _paths(ranks[0][0]).items() if len(p) < plan.depth}
            continue
        for r in range(world):
            xr, cr = partition.take(plan, x, c, r)
            if len(cr):
                insert_batch(ranks[r][0], xr, cr, ranks[r][1])
    assert handed_off
    gp = _paths(g)
    rp = [_paths(t) for t, _ in ranks]
    # prefix subtrees: identical to the single tree, path by path
    for path, nid in gp.items():
        if len(path) < plan.depth:
            continue
        prefix = 0
        for o in path[: plan.depth]:
            prefix = prefix * 8 + o
        r = int(plan.owner[prefix])
        t = ranks[r][0]
        assert path in rp[r], path
        rid = rp[r][path]
        assert bool(t.inner[rid]) == bool(g.inner[nid]), path
        assert np.array_equal(_samples(t, rid), _samples(g, nid)), path
        if g.inner[nid]:
            assert np.array_equal(t.occupied_cells(rid), g.occupied_cells(nid)), path
    # top nodes: common prefix + rank-disjoint appended voxels
    for path, nid in gp.items():
        if len(path) >= plan.depth:
            continue
        want = _samples(g, nid)
        base = pre[path]
        assert np.array_equal(want[: len(base)], base), path
        rest = [_samples(t, rp[r][path])[len(base):] for r, (t, _) in enumerate(ranks)]
        cat = np.concatenate(rest)
        assert len(cat) == len(want) - len(base), path
        keys = lambda a: set(map(tuple, a.tolist()))
        assert keys(cat) == keys(want[len(base):]), path
        for a in range(world):
            for b in range(a + 1, world):
                assert not (keys(rest[a]) & keys(rest[b])), path
    # render: min-composite of per-rank renders (owned subtrees + top) == single tree
    cam = Camera((0.5, 0.45, -1.3), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=50.0, width=320, height=240)
    for thr in (-1.0, 64.0):
        want, _ = rasterize(g, cam, threshold=thr)
        comp = np.full(cam.width * cam.height, np.uint64(0xFFFFFFFFFFFFFFFF))
        for r, (t, _) in enumerate(ranks):
            from paper_2310_03567_b200.render import select_visible
            import ctypes

            inv = {nid: p for p, nid in rp[r].items()}
            keep = []
            for nid in select_visible(t, cam, thr):
                p = inv[nid]
                if len(p) < plan.depth:
                    keep.append(nid)
                    continue
                prefix = 0
                for o in p[: plan.depth]:
                    prefix = prefix * 8 + o
                if int(plan.owner[prefix]) == r:
                    keep.append(nid)
            fb = Framebuffer(cam.width, cam.height)
            from paper_2310_03567_b200 import _lib

            vis = np.asarray(keep, np.int32)
            cp = np.ascontiguousarray(cam.packed())
            drawn = ctypes.c_int64()
            _lib.check(t._L.lod_rasterize(t.handle, _lib.ptr(vis), len(vis), _lib.ptr(cp), _lib.ptr(fb.cells),
                                          fb.width, fb.height, 0, ctypes.byref(drawn)))
            comp = np.minimum(comp, fb.cells)
        assert np.array_equal(comp, want.cells), thr
