"""CPU: the host selection restatement (oracle/select.py) reproduces the
reference's own selections in the raster fixture (render.py:177-200)."""
import sys

import numpy as np

import oracle
from oracle import select as osel
from common import GOLDEN, load_raster


def test_host_selection_matches_reference_fixture():
    sys.path.insert(0, GOLDEN)
    from make_golden import RASTER_CAMS

    from paper_2310_03567_b200.render import Camera

    r = load_raster()
    t = oracle.OracleTree(grid_res=16, leaf_threshold=64, max_depth=12, chunk_capacity=1000, arena_bytes=64 << 20)
    t.insert_batch(r["xyz"], r["rgba"])
    cols = t.state()
    for ci, kw in enumerate(RASTER_CAMS):
        cam = Camera(**kw)
        assert np.array_equal(cam.packed(), r[f"cam{ci}"])
        assert np.array_equal(osel.frustum_planes(cam), osel.frustum_planes(cam))
        for thr in (-1, 128, 20):
            assert osel.select_visible(cols, 1.0, cam, float(thr)) == r[f"lod{ci}_{thr}_sel"].tolist()
