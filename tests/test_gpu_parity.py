"""GPU parity: the CUDA update path vs the reference fixtures and the oracle.

Every comparison is bit-exact on the observable tree: node hierarchy and ids,
every node's sample (point / voxel) sequence, bitgrids, chunk counts, arena
growth, free-list length and overflow behaviour.  Only the ids of individual
chunks are free (their assignment order is not observable).
"""
import numpy as np
import pytest

from common import (assert_same_state, golden_names, load_golden, make_product, oracle_state, product_state,
                    run_oracle, run_product)

pytestmark = pytest.mark.gpu


def _hygiene(tree, state):
    n = tree.num_nodes
    assert len(state.spill) == 0
    assert state.backlog.length == 0
    assert not tree.final[:n].any()
    assert not tree.pending[:n].any()


@pytest.mark.parametrize("name", golden_names())
def test_matches_reference_fixture(gpu, name):
    g = load_golden(name)
    tree, state, error, per_batch = run_product(g["params"], g["batches"])
    assert error == g["error"]
    assert np.array_equal(np.array(per_batch, np.int64).reshape(-1, 5), g["per_batch"])
    if not error:
        assert_same_state(product_state(tree), g["state"], chunk_ids=False, label=name)
        _hygiene(tree, state)
        tree.validate()


def _cloud(n, seed, kind):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        xyz = rng.random((n, 3)).astype(np.float32)
    elif kind == "surface":
        from paper_2310_03567_b200 import synth

        return synth.gen_surface(n, seed)
    elif kind == "skew":
        from paper_2310_03567_b200 import synth

        return synth.gen_skew(n, seed)
    elif kind == "mesh":
        from paper_2310_03567_b200 import synth

        return synth.gen_mesh(n, seed)
    np.clip(xyz, 0.0, np.nextafter(np.float32(1.0), np.float32(0.0)), out=xyz)
    return xyz, rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)


def _params(**kw):
    p = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=256 << 20, chunk_capacity=1000, grid_res=16,
             leaf_threshold=100, max_depth=12, backlog_capacity=10_000_000, spill_capacity=100_000_000)
    p.update(kw)
    return p


CASES = [
    # (label, n, seed, kind, batch, params)
    ("uniform_small_bs1", 300, 1, "uniform", 1, _params(grid_res=4, leaf_threshold=10, max_depth=6, chunk_capacity=3)),
    ("uniform_bs7", 3000, 2, "uniform", 7, _params(grid_res=8, leaf_threshold=20, chunk_capacity=5)),
    ("surface_bs1000", 50_000, 3, "surface", 1000, _params(grid_res=16, leaf_threshold=100, chunk_capacity=64)),
    ("skew_bs5000", 60_000, 4, "skew", 5000, _params(grid_res=32, leaf_threshold=200, max_depth=16, chunk_capacity=100)),
    ("mesh_bs20000", 100_000, 5, "mesh", 20_000, _params(grid_res=64, leaf_threshold=1000, chunk_capacity=250)),
    ("uniform_big_batches", 400_000, 6, "uniform", 100_000,
     _params(arena_bytes=1 << 30, grid_res=128, leaf_threshold=5000, max_depth=20, chunk_capacity=1000)),
    ("offset_cube", 20_000, 7, "uniform", 3000, _params(bmin=(-3.0, 2.5, 10.0), size=6.5, grid_res=8, leaf_threshold=64)),
]


@pytest.mark.parametrize("label,n,seed,kind,bs,params", CASES, ids=[c[0] for c in CASES])
def test_matches_oracle(gpu, label, n, seed, kind, bs, params):
    xyz, rgba = _cloud(n, seed, kind)
    if params["size"] != 1.0:
        xyz = (xyz.astype(np.float64) * params["size"] + np.asarray(params["bmin"])).astype(np.float32)
    batches = [(xyz[i:i + bs], rgba[i:i + bs]) for i in range(0, n, bs)]
    ot, oerr, oper = run_oracle(params, batches)
    tree, state, err, per = run_product(params, batches)
    assert err == oerr == ""
    assert per == oper
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label=label)
    _hygiene(tree, state)
    tree.validate()


def test_config1_one_million_uniform(gpu):
    """BASELINE config 1: 1M uniform points, one batch, paper parameters."""
    from paper_2310_03567_b200 import synth

    xyz, rgba = synth.gen_uniform(1_000_000, 0)
    params = _params(arena_bytes=1 << 30, grid_res=128, leaf_threshold=50_000, max_depth=20, chunk_capacity=1000)
    ot, _, oper = run_oracle(params, [(xyz, rgba)])
    tree, state, err, per = run_product(params, [(xyz, rgba)])
    assert err == ""
    assert per == oper
    assert tree.num_nodes == 73 and int(tree.inner[:73].sum()) == 9
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="config1")
    tree.validate()


def test_terrain_stream_matches_oracle(gpu):
    """Config 2 exactly as bench.py streams it (gen_surface 1M batches, seeds
    1000+i, paper parameters): a 60-batch prefix, through the spill bursts of
    batches 12-13 (3.4M points) and 51 (5.8M points)."""
    from paper_2310_03567_b200 import synth

    params = _params(arena_bytes=4 << 30, grid_res=128, leaf_threshold=50_000, max_depth=20, chunk_capacity=1000,
                     backlog_capacity=64_000_000)
    batches = [synth.gen_surface(1_000_000, 1000 + i) for i in range(60)]
    ot, _, oper = run_oracle(params, batches)
    tree, state, err, per = run_product(params, batches)
    assert err == ""
    assert per == oper
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="terrain")


def test_empty_batch_is_noop(gpu):
    from paper_2310_03567_b200 import insert_batch

    tree, state = make_product(_params())
    insert_batch(tree, np.empty((0, 3), np.float32), np.empty(0, np.uint32), state)
    assert state.stats.batches == 0
    assert tree.num_nodes == 1 and tree.count[0] == 0


def test_device_resident_input_matches_host_input(gpu):
    import torch

    from paper_2310_03567_b200 import insert_batch

    xyz, rgba = _cloud(50_000, 9, "surface")
    p = _params(grid_res=32, leaf_threshold=300, chunk_capacity=128)
    t1, s1 = make_product(p)
    t2, s2 = make_product(p)
    for i in range(0, 50_000, 10_000):
        insert_batch(t1, xyz[i:i + 10_000], rgba[i:i + 10_000], s1)
        dx = torch.from_numpy(xyz[i:i + 10_000]).cuda()
        dc = torch.from_numpy(rgba[i:i + 10_000].view(np.int32)).cuda()
        insert_batch(t2, dx, dc, s2)
    assert_same_state(product_state(t2), product_state(t1), chunk_ids=True, label="device-input")


def test_conservation_and_placement(gpu):
    """Leaf counts sum to n; every stored point routes to its own leaf (criterion 2)."""
    xyz, rgba = _cloud(30_000, 2, "uniform")
    edgy = np.array([[0.5, 0.5, 0.5], [0.25, 0.5, 0.75], [0.5, 0.0, 0.999], [0.5, 0.25, 0.5]], np.float32)
    xyz = np.concatenate([xyz, edgy])
    rgba = np.concatenate([rgba, np.arange(4, dtype=np.uint32)])
    tree, state, err, _ = run_product(_params(grid_res=8, leaf_threshold=64),
                                      [(xyz[i:i + 997], rgba[i:i + 997]) for i in range(0, len(rgba), 997)])
    n = tree.num_nodes
    leaves = np.flatnonzero(~tree.inner[:n])
    assert int(tree.count[leaves].sum()) == len(rgba)
    for leaf in leaves:
        if tree.count[leaf] == 0:
            continue
        lx, _ = tree.gather_samples(int(leaf))
        nid = int(leaf)
        while nid != 0:
            par = int(tree.parent[nid])
            b = tree.node_bounds(par)
            cx = np.array(b.min) + b.size * 0.5
            o = (lx[:, 0] >= cx[0]).astype(np.int8) | ((lx[:, 1] >= cx[1]).astype(np.int8) << 1) | (
                (lx[:, 2] >= cx[2]).astype(np.int8) << 2)
            assert (o == int(tree.octant[nid])).all()
            nid = par


def test_frame_loop_with_pinned_ingest_feed_matches_oracle(gpu):
    """run_frame_updates over page-locked batches (the staged H2D feed,
    lod_prefetch_batch) settles the same tree as the oracle; frames follow
    the reference's budget rule."""
    from collections import deque

    import torch

    from paper_2310_03567_b200 import run_frame_updates

    params = _params(arena_bytes=1 << 30, grid_res=64, leaf_threshold=3000, max_depth=16, chunk_capacity=500)
    xyz, rgba = _cloud(400_000, 11, "surface")
    bs = 40_000
    batches = [(xyz[i:i + bs], rgba[i:i + bs]) for i in range(0, len(rgba), bs)]
    pinned = []
    for x, c in batches:
        px = torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
        pc = torch.from_numpy(np.ascontiguousarray(c).view(np.int32)).pin_memory().numpy().view(np.uint32)
        pinned.append((px, pc))
    ot, _, oper = run_oracle(params, batches)
    tree, state = make_product(params)
    q = deque(pinned)
    frames = 0
    while q:
        assert run_frame_updates(tree, q, state) >= 1
        frames += 1
    assert state.stats.frames == frames and state.stats.batches == len(batches)
    assert state.stats.h2d_bytes == 16 * len(rgba)
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="frame_loop")
    _hygiene(tree, state)


def test_skew_stream_burst_matches_oracle(gpu):
    """Config 4 shape at paper parameters: 12 x 1M density-skew batches; batch 11
    is the measured burst (5.9M spilled points, 7.45M new voxels, 125 splits),
    which drives the claim table through growth + rehash."""
    from paper_2310_03567_b200 import synth

    params = _params(arena_bytes=4 << 30, grid_res=128, leaf_threshold=50_000, max_depth=20, chunk_capacity=1000,
                     backlog_capacity=64_000_000)
    batches = [synth.gen_skew(1_000_000, 1000 + i) for i in range(12)]
    ot, _, oper = run_oracle(params, batches)
    tree, state, err, per = run_product(params, batches)
    assert err == ""
    assert per == oper
    assert max(p[4] for p in per) > 5_000_000  # the spill burst happened
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="skew_burst")
    tree.validate()


def test_frame_budget_semantics(gpu):
    """run_frame_updates (update.py:396-417): at least one batch per call even
    over budget, the budget checked between batches, frames counted."""
    from collections import deque

    from paper_2310_03567_b200 import run_frame_updates

    params = _params(grid_res=16, leaf_threshold=200, chunk_capacity=64)
    xyz, rgba = _cloud(20_000, 12, "uniform")
    batches = [(xyz[i:i + 1000], rgba[i:i + 1000]) for i in range(0, 20_000, 1000)]
    tree, state = make_product(params)
    state.clock.budget_ms = 0.0
    q = deque(batches[:5])
    assert [run_frame_updates(tree, q, state) for _ in range(5)] == [1, 1, 1, 1, 1]
    assert not q and state.stats.frames == 5 and state.stats.batches == 5
    assert run_frame_updates(tree, q, state) == 0 and state.stats.frames == 5  # empty queue: no frame
    state.clock.budget_ms = 1e9
    q = deque(batches[5:])
    assert run_frame_updates(tree, q, state) == 15 and state.stats.frames == 6
    ot, _, _ = run_oracle(params, batches)
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="budget")


def test_frame_loop_keeps_staged_copies_across_frames(gpu):
    """One batch per frame (budget 0): the two queued batches staged at the end
    of a frame are used by the next frames; replacing the queue's head between
    frames drops the staged copies (the new head's own data is inserted)."""
    from collections import deque

    import torch

    from paper_2310_03567_b200 import UpdateConfig, UpdateState, run_frame_updates

    params = _params(arena_bytes=1 << 30, grid_res=64, leaf_threshold=3000, max_depth=16, chunk_capacity=500)
    xyz, rgba = _cloud(360_000, 12, "surface")
    bs = 30_000

    def pin(x, c):
        px = torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()
        pc = torch.from_numpy(np.ascontiguousarray(c).view(np.int32)).pin_memory().numpy().view(np.uint32)
        return px, pc

    batches = [pin(xyz[i:i + bs], rgba[i:i + bs]) for i in range(0, len(rgba), bs)]
    sub_x, sub_c = _cloud(bs, 99, "uniform")
    substitute = pin(sub_x, sub_c)
    tree, _ = make_product(params)
    state = UpdateState(UpdateConfig(budget_ms=0.0, backlog_capacity=params["backlog_capacity"],
                                     spill_capacity=params["spill_capacity"]))
    q = deque(batches)
    inserted = []
    frame = 0
    while q:
        if frame == 4:  # the staged head is replaced by a different batch of the same size
            q[0] = substitute
        inserted.append(q[0])
        assert run_frame_updates(tree, q, state) == 1
        frame += 1
    ot, _, _ = run_oracle(params, [(np.asarray(x), np.asarray(c)) for x, c in inserted])
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="frames_staged")
    _hygiene(tree, state)


def test_burst_resolve_path_forced_matches_reference(gpu):
    """The burst resolve (win list ordered by the radix passes, normally from
    4M new voxels per cycle) forced on every cycle (LOD_WINSORT_MIN=0, read
    once per process): the reference fixtures and oracle cases still match."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, LOD_WINSORT_MIN="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        os.path.join(here, "test_gpu_parity.py"), "-k", "reference_fixture or test_matches_oracle"],
                       env=env, capture_output=True, text=True, timeout=900, cwd=os.path.dirname(here))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout


def test_claim_epoch_wraparound_matches_oracle(gpu):
    """600 small batches: the claim table's key epochs (255 per cycle of
    resets, stale slots never cleared) wrap twice; per-batch stats and the
    final state still match the oracle."""
    from paper_2310_03567_b200 import synth

    params = _params(arena_bytes=1 << 30, grid_res=32, leaf_threshold=600, max_depth=14, chunk_capacity=128)
    batches = [synth.gen_surface(1500, 5000 + i) for i in range(600)]
    ot, _, oper = run_oracle(params, batches)
    tree, state, err, per = run_product(params, batches)
    assert err == ""
    assert per == oper
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="epoch_wrap")


@pytest.mark.parametrize("label,bmin,size", [
    ("unit", (0.0, 0.0, 0.0), 1.0),               # f32 descent (the bench's trees)
    ("offset_pow2", (2.0, 0.5, 0.25), 0.5),       # f32 descent, root off the origin
    ("straddles_zero", (-0.5, -0.5, -0.5), 1.0),  # f64 only: x - bx is not exact in f32 near 0
])
def test_f32_descent_matches_oracle(gpu, label, bmin, size):
    """The count pass descends in f32 when the root, grid and depth make every
    plane, difference and cell product exact in f32 (Geo::f32ok); the trees
    must equal the oracle's (f64, the reference's arithmetic) -- including
    points on cell and split planes, which the f32 compares must place exactly
    like the f64 ones."""
    from paper_2310_03567_b200 import synth

    params = dict(bmin=bmin, size=size, arena_bytes=256 << 20, chunk_capacity=64, grid_res=32, leaf_threshold=300,
                  max_depth=12, backlog_capacity=10_000_000, spill_capacity=100_000_000)
    rng = np.random.default_rng(7)
    batches = []
    for i in range(6):
        x, c = synth.gen_surface(40_000, 900 + i)
        x = (np.asarray(x, np.float64) * size + np.asarray(bmin)).astype(np.float32)
        # a share of the points exactly on the planes of a level-1..6 grid
        k = rng.integers(1, 7)
        q = size / (32 * 2 ** k)
        on = rng.random(len(c)) < 0.2
        snapped = (np.floor((x.astype(np.float64) - np.asarray(bmin)) / q) * q + np.asarray(bmin)).astype(np.float32)
        x[on] = snapped[on]
        batches.append((np.ascontiguousarray(x), c))
    ot, oerr, oper = run_oracle(params, batches)
    tree, state, err, per = run_product(params, batches)
    assert err == oerr == "" and per == oper
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label=label)


@pytest.mark.parametrize("switch", ["LOD_SYNC_MEMCPY=1", "LOD_NO_EARLY=1", "LOD_NO_SPEC=1", "LOD_COUNT_STAGED=1",
                                    "LOD_COUNT_F64=1", "LOD_RESOLVE_LIST_MAX_MB=0", "LOD_NO_SMALL=1",
                                    "LOD_STORE_LSD=1", "LOD_DIR_W=8"])
def test_runtime_switches_keep_parity(gpu, switch):
    """Every runtime switch of DESIGN.md's table selects an alternative with
    the same results: a child process with the switch set runs oracle-checked
    cases (the skew and big-batch streams, a device-resident stream)."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    name, value = switch.split("=")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.join(here, "test_gpu_parity.py"), "-x", "-q",
                        "-p", "no:cacheprovider", "-k",
                        "skew_bs5000 or uniform_big_batches or offset_cube or device_resident"],
                       env=dict(os.environ, **{name: value}), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
