"""Pin the oracle against the live reference at larger sizes (build container
only: /root/reference does not exist on the GPU box, where this skips)."""
import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


def _ref():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from lodstream import octree, store, synth, update

    return octree, store, synth, update


def _run_both(batches, **p):
    import oracle

    octree, store, synth, update = _ref()
    arena = store.Arena(p["arena_bytes"])
    tree = octree.Octree(octree.CubeBounds((0.0, 0.0, 0.0), 1.0), arena, store.ChunkPool(arena, p["chunk_capacity"]),
                         grid_res=p["grid_res"], leaf_threshold=p["leaf_threshold"], max_depth=p["max_depth"])
    st = update.UpdateState(update.UpdateConfig(backlog_capacity=64_000_000))
    o = oracle.OracleTree(grid_res=p["grid_res"], leaf_threshold=p["leaf_threshold"], max_depth=p["max_depth"],
                          chunk_capacity=p["chunk_capacity"], arena_bytes=p["arena_bytes"],
                          backlog_capacity=64_000_000)
    for x, c in batches:
        update.insert_batch(tree, x, c, st)
        o.insert_batch(x, c)
    s = o.state()
    n = tree.num_nodes
    assert s["num_nodes"] == n and s["allocated_total"] == tree.pool.allocated_total
    assert s["arena_offset"] == tree.arena.offset
    for k in ("parent", "level", "children", "inner", "count", "chunk_head", "chunk_count", "grid_off", "bmin"):
        assert np.array_equal(s[k], getattr(tree, k)[:n]), k
    assert np.array_equal(s["next"], tree.pool.next[: tree.pool.allocated_total])
    for nid in range(n):
        a = tree.gather_samples(nid)
        b = o.gather_samples(nid)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), nid
    return tree


def test_config1_one_million_uniform_matches_reference():
    _, _, synth, _ = _ref()
    tree = _run_both([synth.gen_uniform(1_000_000, 0)], grid_res=128, leaf_threshold=50_000, max_depth=20,
                     chunk_capacity=1000, arena_bytes=1 << 30)
    assert tree.num_nodes == 73


def test_terrain_prefix_matches_reference():
    _, _, synth, _ = _ref()
    _run_both([synth.gen_surface(500_000, 100 + i) for i in range(3)], grid_res=64, leaf_threshold=20_000,
              max_depth=20, chunk_capacity=500, arena_bytes=1 << 30)
