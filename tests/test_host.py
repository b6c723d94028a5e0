"""CPU tests of the host-side facade: geometry conventions, the standalone
allocator API, camera / frustum / screen-size math and the input generators.
Known answers are the reference suite's (pkg/tests/test_octree.py,
test_store.py, test_render.py)."""
import math
import os
import sys

import numpy as np
import pytest

from paper_2310_03567_b200 import Arena, ChunkPool, OutOfArena, synth
from paper_2310_03567_b200.octree import (CubeBounds, cell_coords, cell_of, cubify, octant_of, pack_rgba,
                                          voxel_center)
from paper_2310_03567_b200.render import Camera, Framebuffer, SENTINEL, frustum_intersects, frustum_planes, screen_size
from paper_2310_03567_b200.store import NO_CHUNK, RECORD_BYTES
from paper_2310_03567_b200.update import UpdateConfig, UpdateStats, chunks_needed

UNIT = CubeBounds((0.0, 0.0, 0.0), 1.0)


# -- geometry (test_octree.py:25-142) --------------------------------------------------------


def test_octant_routing_convention():
    assert octant_of((0.1, 0.1, 0.1), UNIT) == 0
    assert octant_of((0.8, 0.8, 0.8), UNIT) == 7
    assert octant_of((0.5, 0.1, 0.1), UNIT) == 1  # boundary goes up
    assert octant_of((0.1, 0.6, 0.1), UNIT) == 2
    assert octant_of((0.1, 0.1, 0.6), UNIT) == 4
    assert octant_of((0.6, 0.6, 0.1), UNIT) == 3


def test_children_tile_parent():
    b = CubeBounds((3.0, -2.0, 7.5), 4.0)
    for o in range(8):
        c = b.child(o)
        assert c.size == 2.0
        for axis in range(3):
            assert c.min[axis] == b.min[axis] + (2.0 if (o >> axis) & 1 else 0.0)


def test_cells_and_centres():
    assert cell_of((0.1, 0.1, 0.1), UNIT, 4) == 0
    assert cell_of((0.8, 0.8, 0.8), UNIT, 4) == 63
    assert cell_of((1.0, 1.0, 1.0), UNIT, 4) == 63
    assert cell_of((0.3, 0.1, 0.1), UNIT, 4) == 1
    assert cell_of((0.1, 0.3, 0.1), UNIT, 4) == 4
    assert cell_of((0.1, 0.1, 0.3), UNIT, 4) == 16
    assert voxel_center(0, UNIT, 4).tolist() == [0.125, 0.125, 0.125]
    assert voxel_center(63, UNIT, 4).tolist() == [0.875, 0.875, 0.875]
    assert voxel_center(0, CubeBounds((10.0, 10.0, 10.0), 8.0), 128).tolist() == [10.03125] * 3
    for cell in (0, 1, 8, 64, 511, 137):
        cx, cy, cz = cell_coords(cell, 8)
        assert (cz * 8 + cy) * 8 + cx == cell


def test_cubify_and_pack():
    b = cubify((0.0, 0.0, 0.0), (10.0, 4.0, 2.0))
    assert b.size == 10.0 and b.min == (0.0, -3.0, -4.0)
    b = cubify((5.0, 5.0, 5.0), (5.0, 5.0, 5.0))
    assert b.size == 1.0 and b.min == (4.5, 4.5, 4.5)
    assert pack_rgba(0xFF, 0, 0, 0xFF) == 0xFF0000FF
    assert pack_rgba(0x12, 0x34, 0x56, 0x78) == 0x78563412
    corners = UNIT.corners()
    assert corners.shape == (8, 3) and corners[7].tolist() == [1.0, 1.0, 1.0] and corners[5].tolist() == [1.0, 0.0, 1.0]


# -- standalone allocator API (test_store.py) -------------------------------------------------


def test_arena_alignment_and_errors():
    a = Arena(1024)
    assert a.alloc(16, 16) == 0 and a.offset == 16
    a.alloc(1, 16)
    assert a.alloc(16, 16) == 32
    b = Arena(1 << 20)
    b.alloc(256 * 1024, 64)
    assert b.offset == 262144
    c = Arena(64)
    c.alloc(48, 16)
    with pytest.raises(OutOfArena):
        c.alloc(32, 16)
    c.alloc(16, 16)
    with pytest.raises(ValueError):
        Arena(0)


def test_pool_lifo_reuse_and_ledger():
    arena = Arena(1 << 16)
    pool = ChunkPool(arena, 4)
    before = arena.offset
    cid = pool.acquire()
    assert arena.offset == before + 4 * RECORD_BYTES
    assert pool.allocated_total == 1 and pool.occupied[cid] == 0 and pool.next[cid] == NO_CHUNK
    ids = [cid] + [pool.acquire() for _ in range(2)]
    pool.next[ids[0]] = ids[1]
    pool.next[ids[1]] = ids[2]
    assert pool.release(ids[0]) == 3 and pool.free_count == 3
    assert pool.acquire() == ids[2]  # most recently released first
    assert pool.allocated_total == 3
    pool.check_ledger()
    f32, u32 = pool.records(ids[0])
    assert f32.shape == (4, 3) and u32.shape == (4,)


def test_chunks_needed_and_stats():
    assert chunks_needed(0, 1000) == 0
    assert chunks_needed(1000, 1000) == 1
    assert chunks_needed(1001, 1000) == 2
    s = UpdateStats(points=2_000_000, update_seconds=0.5)
    assert s.throughput_mps() == 4.0
    assert UpdateStats().throughput_mps() == 0.0
    assert UpdateConfig().backlog_capacity == 10_000_000


# -- camera / frustum (test_render.py:40-140) ----------------------------------------------------

FRONT = Camera(position=(0.5, 0.5, -1.0), target=(0.5, 0.5, 0.5), fov_deg=90.0, near=0.1, far=100.0,
               width=1000, height=1000)


def test_camera_projection_and_packing():
    sx, sy, d01 = FRONT.project((0.6, 0.7, 0.5))
    assert math.floor(sx) == 466 and math.floor(sy) == 433
    assert np.float32(d01) == np.float32(100.0 * 1.4 / (99.9 * 1.5))
    assert FRONT.project((0.5, 0.5, -0.95)) is None
    assert FRONT.project((0.5, 0.5, 200.0)) is None
    p = FRONT.packed()
    assert p.shape == (18,) and p.dtype == np.float64
    assert p[16] == 1000 and p[17] == 1000 and p[14] == 0.1 and p[15] == 100.0


def test_screen_size_and_frustum():
    assert screen_size(UNIT, FRONT) == pytest.approx(500.0, rel=1e-12)
    inside = Camera((0.5, 0.5, 0.5), (2.0, 0.5, 0.5), near=0.1, far=100.0)
    assert screen_size(UNIT, inside) == math.inf
    planes = frustum_planes(FRONT)
    assert frustum_intersects(UNIT, planes)
    assert not frustum_intersects(CubeBounds((0.0, 0.0, -30.0), 1.0), planes)
    assert not frustum_intersects(CubeBounds((40.0, 0.5, 0.0), 1.0), planes)
    assert frustum_intersects(CubeBounds((0.4, 0.4, -1.5), 1.0), planes)


def test_framebuffer_image():
    fb = Framebuffer(2, 1)
    fb.cells[0] = np.uint64(0x000000FF)
    img = fb.image(background=(1, 2, 3))
    assert img.tolist() == [[[255, 0, 0], [1, 2, 3]]]
    assert (Framebuffer(3, 2).cells == SENTINEL).all()


# -- generators -------------------------------------------------------------------------------------

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present (GPU box)")
def test_generators_match_reference():
    sys.path.insert(0, REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    from lodstream import synth as ref

    for name in ("gen_uniform", "gen_surface"):
        a = getattr(synth, name)(10_000, 42)
        b = getattr(ref, name)(10_000, 42)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_new_generators_shape_and_determinism():
    for gen in (synth.gen_mesh, synth.gen_skew):
        x1, c1 = gen(5000, 3)
        x2, c2 = gen(5000, 3)
        assert x1.dtype == np.float32 and x1.shape == (5000, 3) and c1.dtype == np.uint32
        assert np.array_equal(x1, x2) and np.array_equal(c1, c2)
        assert (x1 >= 0).all() and (x1 < 1).all()
    x, _ = synth.gen_skew(100_000, 1)
    inside = np.all((x >= np.array(synth.SKEW_CORNER, np.float32)) &
                    (x < np.array(synth.SKEW_CORNER, np.float32) + synth.SKEW_SIDE + 1e-6), axis=1)
    assert 0.89 < inside.mean() < 0.91
