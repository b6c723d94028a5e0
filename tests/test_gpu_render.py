"""GPU rasterizer parity: brute force and LOD splats vs the reference fixtures."""
import math

import numpy as np
import pytest

from common import dense_fb, load_raster, make_product

pytestmark = pytest.mark.gpu

FRONT = dict(position=(0.5, 0.5, -1.0), target=(0.5, 0.5, 0.5), fov_deg=90.0, near=0.1, far=100.0,
             width=1000, height=1000)


def _cam_from_packed(packed, kw):
    from paper_2310_03567_b200.render import Camera

    cam = Camera(**kw)
    assert np.array_equal(cam.packed(), packed)
    return cam


def test_brute_force_matches_reference(gpu):
    from paper_2310_03567_b200.render import brute_force_render

    import sys
    sys.path.insert(0, __file__.rsplit("/", 1)[0] + "/golden")
    from make_golden import RASTER_CAMS

    r = load_raster()
    for ci, kw in enumerate(RASTER_CAMS):
        cam = _cam_from_packed(r[f"cam{ci}"], kw)
        fb = brute_force_render(r["xyz"], r["rgba"], cam)
        assert np.array_equal(fb.cells, dense_fb(r[f"brute{ci}_idx"], r[f"brute{ci}_val"], cam.width * cam.height))


def test_lod_raster_matches_reference(gpu):
    from paper_2310_03567_b200 import insert_batch
    from paper_2310_03567_b200.render import rasterize

    import sys
    sys.path.insert(0, __file__.rsplit("/", 1)[0] + "/golden")
    from make_golden import RASTER_CAMS

    r = load_raster()
    tree, state = make_product(dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=64 << 20, chunk_capacity=1000,
                                    grid_res=16, leaf_threshold=64, max_depth=12, backlog_capacity=10_000_000,
                                    spill_capacity=100_000_000))
    insert_batch(tree, r["xyz"], r["rgba"], state)
    for ci, kw in enumerate(RASTER_CAMS):
        cam = _cam_from_packed(r[f"cam{ci}"], kw)
        for thr in (-1, 128, 20):
            key = f"lod{ci}_{thr}"
            fb, rep = rasterize(tree, cam, threshold=float(thr))
            assert rep.selected == r[key + "_sel"].tolist(), key
            assert rep.samples_drawn == int(r[key + "_samples"][0]), key
            assert np.array_equal(fb.cells, dense_fb(r[key + "_idx"], r[key + "_val"], cam.width * cam.height)), key


def test_single_point_lands_on_computed_pixel(gpu):
    """test_render.py:43-59 worked by hand: pixel (466, 433), exact depth bits."""
    from paper_2310_03567_b200.render import SENTINEL, Camera, brute_force_render

    fb = brute_force_render(np.array([[0.6, 0.7, 0.5]], np.float32), np.array([0xAABBCCDD], np.uint32),
                            Camera(**FRONT))
    hit = np.flatnonzero(fb.cells != SENTINEL)
    assert hit.tolist() == [433 * 1000 + 466]
    assert fb.cells[hit[0]] & np.uint64(0xFFFFFFFF) == 0xAABBCCDD
    depth = 100.0 * (1.5 - 0.1) / ((100.0 - 0.1) * 1.5)
    assert fb.cells[hit[0]] >> np.uint64(32) == np.float32(depth).view(np.uint32)


def test_closer_wins_and_ties_break_to_lower_colour(gpu):
    from paper_2310_03567_b200.render import Camera, brute_force_render

    cam = Camera(**FRONT)
    p = np.array([[0.5, 0.5, 0.7], [0.5, 0.5, 0.2]], np.float32)
    c = np.array([111, 222], np.uint32)
    fb = brute_force_render(p, c, cam)
    assert fb.grid()[500, 500] & np.uint64(0xFFFFFFFF) == 222
    fb2 = brute_force_render(p[::-1].copy(), c[::-1].copy(), cam)
    assert np.array_equal(fb.cells, fb2.cells)
    tie = brute_force_render(np.array([[0.5, 0.5, 0.4]] * 2, np.float32), np.array([9, 5], np.uint32), cam)
    assert tie.grid()[500, 500] & np.uint64(0xFFFFFFFF) == 5


def test_empty_input_leaves_background(gpu):
    from paper_2310_03567_b200.render import SENTINEL, Camera, brute_force_render

    fb = brute_force_render(np.empty((0, 3), np.float32), np.empty(0, np.uint32), Camera(**FRONT))
    assert (fb.cells == SENTINEL).all()


def test_full_refinement_equals_brute_force_many_scenes(gpu):
    """criterion 6 (test_acceptance.py:222-252), scaled: LOD at threshold -1 == brute force == oracle."""
    import oracle
    from oracle import rebuild
    from paper_2310_03567_b200 import insert_batch
    from paper_2310_03567_b200.render import Camera, brute_force_render, rasterize

    rng = np.random.default_rng(6)
    for scene in range(8):
        n = int(rng.integers(100, 20_001))
        r2 = np.random.default_rng(6000 + scene)
        xyz = r2.random((n, 3)).astype(np.float32)
        rgba = r2.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
        d, theta, phi = rng.uniform(1.1, 2.5), rng.uniform(0, 2 * math.pi), rng.uniform(-0.9, 0.9)
        pos = (0.5 + d * math.cos(phi) * math.cos(theta), 0.5 + d * math.sin(phi),
               0.5 + d * math.cos(phi) * math.sin(theta))
        cam = Camera(position=pos, target=(0.5, 0.5, 0.5), fov_deg=float(rng.uniform(50, 90)), near=0.05, far=50.0,
                     width=256, height=256)
        fb = brute_force_render(xyz, rgba, cam)
        assert np.array_equal(fb.cells, rebuild.ref_render(xyz, rgba, cam.packed(), 256, 256))
        tree, state = make_product(dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=128 << 20, chunk_capacity=1000,
                                        grid_res=8, leaf_threshold=400, max_depth=12,
                                        backlog_capacity=10_000_000, spill_capacity=100_000_000))
        insert_batch(tree, xyz, rgba, state)
        lod, rep = rasterize(tree, cam, threshold=-1.0)
        assert all(not tree.inner[nid] for nid in rep.selected)
        assert np.array_equal(lod.cells, fb.cells)
        ofb = np.full(256 * 256, np.uint64(0xFFFFFFFFFFFFFFFF))
        oracle.rasterize_points(xyz, rgba, cam.packed(), ofb)
        assert np.array_equal(ofb, fb.cells)


def _cols(tree):
    return {k: getattr(tree, k) for k in ("inner", "count", "children", "bmin", "level")}


def _random_cameras(rng, k):
    from paper_2310_03567_b200.render import Camera

    cams = []
    for _ in range(k):
        target = rng.uniform(0.2, 0.8, 3)
        d = rng.normal(size=3)
        d /= np.linalg.norm(d)
        pos = target + d * rng.uniform(0.15, 2.5)
        cams.append(Camera(tuple(pos), tuple(target), fov_deg=float(rng.uniform(40, 100)), near=0.01,
                           far=float(rng.uniform(2.0, 50.0)), width=int(rng.integers(200, 1400)),
                           height=int(rng.integers(150, 1000))))
    return cams


def test_device_selection_matches_host_restatement(gpu):
    """select_visible on the GPU vs the reference's stack walk (oracle/select.py)
    on a terrain tree, 24 random cameras x 4 thresholds; a differing node must be
    a float-order tie (decision margin < 1e-9), which none of these cameras hit."""
    from oracle import select as osel
    from paper_2310_03567_b200 import insert_batch, synth
    from paper_2310_03567_b200.render import rasterize, select_visible

    import oracle

    params = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=1 << 30, chunk_capacity=500, grid_res=32,
                  leaf_threshold=2000, max_depth=14, backlog_capacity=10_000_000, spill_capacity=100_000_000)
    tree, state = make_product(params)
    ot = oracle.OracleTree(grid_res=32, leaf_threshold=2000, max_depth=14, chunk_capacity=500, arena_bytes=1 << 30)
    for i in range(4):
        xyz, rgba = synth.gen_surface(100_000, 50 + i)
        insert_batch(tree, xyz, rgba, state)
        ot.insert_batch(xyz, rgba)
    cols = _cols(tree)
    rng = np.random.default_rng(7)
    for cam in _random_cameras(rng, 24):
        for thr in (-1.0, 32.0, 128.0, 700.0):
            want = osel.select_visible(cols, 1.0, cam, thr)
            got = select_visible(tree, cam, thr)
            if got != want:
                diff = sorted(set(got) ^ set(want))
                m = osel.decision_margins(cols, 1.0, cam, thr, diff)
                assert all(min(v) < 1e-9 for v in m.values()), (thr, m)
                continue
            fb, rep = rasterize(tree, cam, threshold=thr)
            assert rep.selected == want
            from paper_2310_03567_b200.render import Framebuffer

            ofb = Framebuffer(cam.width, cam.height)
            assert rep.samples_drawn == ot.rasterize_nodes(want, cam.packed(), ofb.cells)
            assert np.array_equal(fb.cells, ofb.cells)


def test_empty_tree_selects_nothing(gpu):
    from paper_2310_03567_b200.render import Camera, rasterize, select_visible

    tree, _ = make_product(dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=1 << 20, chunk_capacity=10,
                                grid_res=4, leaf_threshold=10, max_depth=4, backlog_capacity=10, spill_capacity=10))
    cam = Camera(**FRONT)
    assert select_visible(tree, cam) == []
    fb, rep = rasterize(tree, cam)
    assert rep.selected == [] and rep.samples_drawn == 0


def test_render_onto_existing_framebuffer_and_pinned_targets(gpu):
    """A fresh target (pinned, device-filled: LOD_FLAG_FB_CLEAR) and a caller's
    framebuffer splatted on top of its contents agree: drawing onto existing
    cells is their depth-min with a fresh render; pooled targets are reused
    without leaking old contents."""
    import gc

    from paper_2310_03567_b200 import insert_batch, synth
    from paper_2310_03567_b200.render import Camera, Framebuffer, brute_force_render, rasterize, rasterize_nodes

    P = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=256 << 20, chunk_capacity=256, grid_res=32,
             leaf_threshold=2000, max_depth=12, backlog_capacity=10_000_000, spill_capacity=100_000_000)
    tree, state = make_product(P)
    for i in range(3):
        insert_batch(tree, *synth.gen_surface(30_000, 70 + i), state)
    cam = Camera((0.5, 0.4, -1.5), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=100.0, width=320, height=240)
    xa, ca = synth.gen_uniform(20_000, 5)
    a = brute_force_render(xa, ca, cam).cells.copy()
    fresh, rep = rasterize(tree, cam, threshold=64.0)
    want = np.minimum(a, fresh.cells)
    host = Framebuffer(cam.width, cam.height)
    host.cells[:] = a
    got, rep2 = rasterize(tree, cam, threshold=64.0, fb=host)
    assert got is host and np.array_equal(host.cells, want)
    assert rep2.samples_drawn == rep.samples_drawn
    nodes_fb, _ = rasterize_nodes(tree, rep.selected, cam)
    assert np.array_equal(nodes_fb.cells, fresh.cells)
    # pooled pinned targets: a recycled buffer starts from the sentinel again
    ref = fresh.cells.copy()
    del fresh, nodes_fb
    gc.collect()
    for _ in range(3):
        again, _ = rasterize(tree, cam, threshold=64.0)
        assert np.array_equal(again.cells, ref)
    empty = Camera((0.5, 0.5, 3.0), (0.5, 0.5, 10.0), fov_deg=30.0, near=0.05, far=1.0, width=320, height=240)
    blank, rep3 = rasterize(tree, empty, threshold=64.0)
    assert rep3.samples_drawn == 0 and bool((blank.cells == np.uint64(0xFFFFFFFFFFFFFFFF)).all())
