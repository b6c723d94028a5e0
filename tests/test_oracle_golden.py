"""Pin the CPU oracle against the reference's own outputs (golden fixtures).

The fixtures were produced by running /root/reference's ``lodstream`` package
(tests/golden/make_golden.py).  The oracle must reproduce every observable,
including chunk ids, payload offsets and the free list.
"""
import numpy as np
import pytest

import oracle
from common import GOLDEN as GOLDEN_DIR
from oracle import rebuild
from common import (assert_same_deltas, assert_same_state, delta_names, dense_fb, flatten_deltas, golden_names,
                    load_deltas, load_golden, load_raster, oracle_state, run_oracle)


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_fixture(name):
    g = load_golden(name)
    t, error, per_batch = run_oracle(g["params"], g["batches"])
    assert error == g["error"]
    assert np.array_equal(np.array(per_batch, np.int64).reshape(-1, 5), g["per_batch"])
    if not error:
        assert_same_state(oracle_state(t), g["state"], chunk_ids=True, label=name)


def test_oracle_brute_force_raster_matches_fixture():
    r = load_raster()
    for ci in range(3):
        cam = r[f"cam{ci}"]
        w, h = int(cam[16]), int(cam[17])
        fb = np.full(w * h, np.uint64(0xFFFFFFFFFFFFFFFF))
        oracle.rasterize_points(r["xyz"], r["rgba"], cam, fb)
        assert np.array_equal(fb, dense_fb(r[f"brute{ci}_idx"], r[f"brute{ci}_val"], w * h))
        # the independent numpy restatement agrees as well (oracles.py:258-286)
        assert np.array_equal(rebuild.ref_render(r["xyz"], r["rgba"], cam, w, h), fb)


def test_oracle_lod_raster_matches_fixture():
    r = load_raster()
    t = oracle.OracleTree(grid_res=16, leaf_threshold=64, max_depth=12, chunk_capacity=1000, arena_bytes=64 << 20)
    t.insert_batch(r["xyz"], r["rgba"])
    for ci in range(3):
        cam = r[f"cam{ci}"]
        w, h = int(cam[16]), int(cam[17])
        for thr in (-1, 128, 20):
            key = f"lod{ci}_{thr}"
            fb = np.full(w * h, np.uint64(0xFFFFFFFFFFFFFFFF))
            drawn = t.rasterize_nodes(r[key + "_sel"], cam, fb)
            assert drawn == int(r[key + "_samples"][0])
            assert np.array_equal(fb, dense_fb(r[key + "_idx"], r[key + "_val"], w * h))


@pytest.mark.parametrize("name", ["rebuild_bs31", "replay_bs37", "uniform_g16_c7", "skew_g8"])
def test_oracle_matches_topdown_rebuild(name):
    """The oracle's tree equals the reference suite's top-down rebuild (oracles.py:55-147)."""
    g = load_golden(name)
    p = g["params"]
    t, error, _ = run_oracle(p, g["batches"])
    assert not error
    ref = rebuild.build_reference(g["xyz"], g["rgba"], p["bmin"], p["size"], grid_res=p["grid_res"],
                                  leaf_threshold=p["leaf_threshold"], max_depth=p["max_depth"])
    st = t.state()

    class View:  # the attributes assert_matches_reference reads
        inner, children, bmin, grid_res = st["inner"], st["children"], st["bmin"], p["grid_res"]

        def node_size(self, nid):
            return p["size"] * 0.5 ** int(st["level"][nid])

        gather_samples = staticmethod(t.gather_samples)
        occupied_cells = staticmethod(t.occupied_cells)

    rebuild.assert_matches_reference(View(), ref)


@pytest.mark.parametrize("name", delta_names())
def test_oracle_delta_matches_reference_fixture(name):
    """BatchDelta restatement (update.py:333-355) vs the reference's own deltas."""
    g = load_golden(name)
    p = g["params"]
    t = oracle.OracleTree(p["bmin"], p["size"], grid_res=p["grid_res"], leaf_threshold=p["leaf_threshold"],
                          max_depth=p["max_depth"], chunk_capacity=p["chunk_capacity"],
                          arena_bytes=p["arena_bytes"], backlog_capacity=p["backlog_capacity"],
                          spill_capacity=p["spill_capacity"])
    deltas = [t.insert_batch(x, c, collect_delta=True)["delta"] for x, c in g["batches"]]
    assert_same_deltas(flatten_deltas(deltas), load_deltas(name), name)


def test_oracle_morton_matches_reference_fixture():
    """io.py:419-446 restatement (oracle/morton.py) vs the reference's own keys and orders."""
    from oracle import morton

    z = np.load(GOLDEN_DIR + "/morton.npz")
    x, c = z["xyz"], z["rgba"]
    for bits in (1, 2, 5, 10, 11, 16, 21):
        assert np.array_equal(morton.morton_key(x, (0.0, 0.0, 0.0), 1.0, bits), z[f"keys_b{bits}"]), bits
    order = morton.morton_order(x, (0.0, 0.0, 0.0), 1.0)
    assert np.array_equal(x[order], z["sorted_xyz"]) and np.array_equal(c[order], z["sorted_rgba"])
    assert np.array_equal(morton.morton_key(z["off_xyz"], (-3.0, 2.5, 10.0), 6.5), z["off_keys"])
    assert np.array_equal(c[morton.morton_order(z["off_xyz"], (-3.0, 2.5, 10.0), 6.5)], z["off_sorted_rgba"])


def test_oracle_morton_known_answers():
    """test_io.py:231-275 known answers."""
    from oracle import morton

    pts = np.array([[0.1, 0.1, 0.1], [0.6, 0.6, 0.6], [0.6, 0.1, 0.1]], np.float32)
    assert morton.morton_key(pts, (0, 0, 0), 1.0, bits=1).tolist() == [0, 7, 1]
    for p, k in (([0.6, 0.1, 0.1], 8), ([0.1, 0.6, 0.1], 16), ([0.1, 0.1, 0.6], 32)):
        assert morton.morton_key(np.array([p], np.float32), (0, 0, 0), 1.0, bits=2).tolist() == [k]
