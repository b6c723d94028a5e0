"""The multi-GPU protocol on one GPU: N emulated ranks = N trees.

Warm-up batches go to rank 0 until the top is inner; its state is packed and
unpacked into the other ranks (lod_tree_pack/unpack); later batches are routed
by exact octant prefix, and after every batch the replicated top nodes'
new voxels are merged across ranks by their winners' global indices
(multigpu.merge_top_voxels).  The union must equal the single-tree run node
for node: every prefix subtree on its owner and every top node on every rank
(kind, sample sequence, bitgrid); and the min-composite of the ranks' renders
must equal the single-tree render.
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
    from paper_2310_03567_b200 import partition, synth
    from paper_2310_03567_b200.render import Camera, Framebuffer, rasterize

    from common import assert_union_equals_single, emulate_partitioned

    batches = [synth.gen_surface(40_000, 300 + i) for i in range(12)]
    plan = partition.plan_owners(batches[:2], world, depth=1)
    g, ranks, handed = emulate_partitioned(P, batches, plan)
    assert handed is not None and handed < len(batches) - 2
    # every node of the single tree, node for node: prefix subtrees on their
    # owner, the merged top nodes on every rank
    assert assert_union_equals_single(g, ranks, plan, label=f"x{world}") > 50
    rp = [_paths(t) for t, _ in ranks]
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
