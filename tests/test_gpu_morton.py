"""GPU parity of the device Morton order (lod_morton_sort) -- reference
lodstream/io.py:419-446, pinned to the reference's own keys/orders
(tests/golden/morton.npz) and its known answers (test_io.py:231-275); at 4M
points through size-independent properties (keys == oracle keys, sortedness,
stability, multiset)."""
import numpy as np
import pytest

from common import GOLDEN

pytestmark = pytest.mark.gpu


def test_keys_and_order_match_reference_fixture(gpu):
    from paper_2310_03567_b200 import CubeBounds
    from paper_2310_03567_b200.morton import morton_key, morton_sort

    z = np.load(GOLDEN + "/morton.npz")
    x, c = z["xyz"], z["rgba"]
    unit = CubeBounds((0.0, 0.0, 0.0), 1.0)
    for bits in (1, 2, 5, 10, 11, 16, 21):
        assert np.array_equal(morton_key(x, unit, bits=bits), z[f"keys_b{bits}"]), bits
    sx, sr = morton_sort(x, c, unit)
    assert np.array_equal(sx, z["sorted_xyz"]) and np.array_equal(sr, z["sorted_rgba"])
    off = CubeBounds((-3.0, 2.5, 10.0), 6.5)
    assert np.array_equal(morton_key(z["off_xyz"], off), z["off_keys"])
    assert np.array_equal(morton_sort(z["off_xyz"], c, off)[1], z["off_sorted_rgba"])


def test_known_answers(gpu):
    from paper_2310_03567_b200 import CubeBounds
    from paper_2310_03567_b200.morton import morton_key, morton_sort

    unit = CubeBounds((0.0, 0.0, 0.0), 1.0)
    pts = np.array([[0.1, 0.1, 0.1], [0.6, 0.6, 0.6], [0.6, 0.1, 0.1]], np.float32)
    assert morton_key(pts, unit, bits=1).tolist() == [0, 7, 1]
    for p, k in (([0.6, 0.1, 0.1], 8), ([0.1, 0.6, 0.1], 16), ([0.1, 0.1, 0.6], 32)):
        assert morton_key(np.array([p], np.float32), unit, bits=2).tolist() == [k]
    xyz = np.array([[0.8, 0.8, 0.8], [0.2, 0.2, 0.2], [0.1, 0.1, 0.1]], np.float32)
    assert morton_sort(xyz, np.array([3, 2, 1], np.uint32), unit)[1].tolist() == [1, 2, 3]
    e = morton_sort(np.empty((0, 3), np.float32), np.empty(0, np.uint32), unit)
    assert e[0].shape == (0, 3) and e[1].shape == (0,)


def test_four_million_points_properties(gpu):
    from oracle import morton as om
    from paper_2310_03567_b200 import CubeBounds, synth
    from paper_2310_03567_b200.morton import morton_key, morton_sort

    unit = CubeBounds((0.0, 0.0, 0.0), 1.0)
    xs, cs = zip(*(synth.gen_surface(1_000_000, 70 + i) for i in range(4)))
    x, c = np.concatenate(xs), np.concatenate(cs)
    c = np.arange(len(c), dtype=np.uint32)  # payload = input index: stability is checkable
    keys = morton_key(x, unit)
    assert np.array_equal(keys, om.morton_key(x, (0.0, 0.0, 0.0), 1.0))
    sx, sr = morton_sort(x, c, unit)
    assert np.array_equal(sr, om.morton_order(x, (0.0, 0.0, 0.0), 1.0).astype(np.uint32))
    assert np.array_equal(sx, x[sr])
    k2 = keys[sr]
    assert (k2[1:] >= k2[:-1]).all()
    same = k2[1:] == k2[:-1]
    assert (sr[1:][same] > sr[:-1][same]).all()  # stable
