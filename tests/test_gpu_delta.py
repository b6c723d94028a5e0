"""GPU parity of insert_batch(collect_delta=True) -- the BatchDelta the
streaming service consumes (update.py:183-194, 333-355; service.py:228-243).

Checked against the reference's own deltas (tests/golden/deltas.npz, made by
running lodstream), against the oracle's restatement on larger streams, and by
a size-independent property: replaying the deltas into a client-side mirror
(the service's ClientMirror contract, service.py:450-485) reproduces the tree.
"""
from collections import deque

import numpy as np
import pytest

from common import (assert_same_deltas, delta_names, flatten_deltas, load_deltas, load_golden, make_product)
from test_gpu_parity import _cloud, _params

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", delta_names())
def test_delta_matches_reference_fixture(gpu, name):
    from paper_2310_03567_b200 import insert_batch

    g = load_golden(name)
    tree, state = make_product(g["params"])
    deltas = [insert_batch(tree, x, c, state, collect_delta=True) for x, c in g["batches"]]
    assert_same_deltas(flatten_deltas(deltas), load_deltas(name), name)


DELTA_CASES = [
    ("surface_bs1000", 60_000, 3, "surface", 1000, _params(grid_res=16, leaf_threshold=100, chunk_capacity=64)),
    ("skew_bs7000", 70_000, 4, "skew", 7000, _params(grid_res=32, leaf_threshold=200, max_depth=16, chunk_capacity=100)),
    ("mesh_bs25000", 100_000, 5, "mesh", 25_000, _params(grid_res=64, leaf_threshold=1000, chunk_capacity=250)),
]


@pytest.mark.parametrize("label,n,seed,kind,bs,params", DELTA_CASES, ids=[c[0] for c in DELTA_CASES])
def test_delta_matches_oracle(gpu, label, n, seed, kind, bs, params):
    import oracle
    from paper_2310_03567_b200 import insert_batch

    xyz, rgba = _cloud(n, seed, kind)
    batches = [(xyz[i:i + bs], rgba[i:i + bs]) for i in range(0, n, bs)]
    p = params
    ot = oracle.OracleTree(p["bmin"], p["size"], grid_res=p["grid_res"], leaf_threshold=p["leaf_threshold"],
                           max_depth=p["max_depth"], chunk_capacity=p["chunk_capacity"],
                           arena_bytes=p["arena_bytes"], backlog_capacity=p["backlog_capacity"],
                           spill_capacity=p["spill_capacity"])
    want = [ot.insert_batch(x, c, collect_delta=True)["delta"] for x, c in batches]
    tree, state = make_product(params)
    got = [insert_batch(tree, x, c, state, collect_delta=True) for x, c in batches]
    assert_same_deltas(flatten_deltas(got), flatten_deltas(want), label)


class Mirror:
    """Client-side replay of deltas (the service's ClientMirror contract)."""

    def __init__(self):
        self.nodes = {0: dict(parent=-1, octant=0, level=0, inner=False)}
        self.points = {0: []}
        self.voxels = {}

    def apply(self, tree, d):
        for ev in d.structure:
            if ev[0] == "split":
                nid = ev[1]
                self.nodes[nid]["inner"] = True
                self.points[nid] = []
                self.voxels.setdefault(nid, ([], []))
            else:
                _, kid, parent, octant, level = ev
                assert kid not in self.nodes
                self.nodes[kid] = dict(parent=parent, octant=octant, level=level, inner=False)
                self.points[kid] = []
        for nid, cells, cols in d.voxels:
            assert self.nodes[nid]["inner"]
            self.voxels[nid][0].append(cells)
            self.voxels[nid][1].append(cols)
        for nid, start, count in d.points:
            assert len(self.points[nid]) == start
            xyz, rgba = tree.gather_samples(nid, start)
            assert len(rgba) == count
            self.points[nid].extend(zip(map(tuple, xyz.tolist()), rgba.tolist()))


def test_delta_replay_reproduces_terrain_tree(gpu):
    """Config 2 shape at paper parameters: 3 x 1M terrain batches through
    run_frame_updates(on_delta=...); the mirror equals the settled tree."""
    from paper_2310_03567_b200 import run_frame_updates, synth

    params = _params(arena_bytes=2 << 30, grid_res=128, leaf_threshold=50_000, max_depth=20, chunk_capacity=1000)
    tree, state = make_product(params)
    state.clock.budget_ms = 1e9  # all three batches in one frame
    m = Mirror()
    q = deque(synth.gen_surface(1_000_000, 300 + i) for i in range(3))
    got = []
    n = run_frame_updates(tree, q, state, on_delta=lambda d: (got.append(d), m.apply(tree, d)))
    assert n == 3 and len(got) == 3
    nn = tree.num_nodes
    assert sorted(m.nodes) == list(range(nn))
    for nid in range(nn):
        nd = m.nodes[nid]
        assert nd["parent"] == tree.parent[nid] and nd["octant"] == tree.octant[nid]
        assert nd["level"] == tree.level[nid] and nd["inner"] == bool(tree.inner[nid])
        xyz, rgba = tree.gather_samples(nid)
        if tree.inner[nid]:
            cells = np.concatenate(m.voxels[nid][0]) if m.voxels[nid][0] else np.empty(0, np.uint32)
            cols = np.concatenate(m.voxels[nid][1]) if m.voxels[nid][1] else np.empty(0, np.uint32)
            assert np.array_equal(np.sort(cells.astype(np.int64)), tree.occupied_cells(nid))
            assert np.array_equal(cols, rgba)  # voxel sequence = claim order
        else:
            assert [c for _, c in m.points[nid]] == rgba.tolist()
            assert np.array_equal(np.array([p for p, _ in m.points[nid]], np.float32).reshape(-1, 3), xyz)


def test_empty_batch_delta(gpu):
    from paper_2310_03567_b200 import BatchDelta, insert_batch

    tree, state = make_product(_params())
    d = insert_batch(tree, np.empty((0, 3), np.float32), np.empty(0, np.uint32), state, collect_delta=True)
    assert d == BatchDelta()
