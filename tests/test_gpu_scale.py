"""Bit-exact parity at BASELINE scale (the configs bench.py and DESIGN quote).

* config 2: the full 100 x 1M-point terrain stream exactly as bench.py
  generates it (gen_surface, seeds 1000+i), paper parameters (G=128,
  T=50,000, C=1,000, depth 20), every batch's UpdateStats and the settled tree
  vs the oracle, plus the render at the bench camera vs the oracle's splat;
* config 4: the density-skew stream through its split waves of > 20M spilled
  points (claim-table growth, rehash, burst resolve and 16-bit-histogram
  fallbacks all trigger there);
* config 3: the mesh stream, insert + rasterize per frame at the bench
  camera, every frame's framebuffer vs the oracle's splat of the same
  selection, and the tree at the end;
* config 5: the partition protocol at paper parameters on a 24M-point
  terrain prefix, 2/4/8 ranks emulated on one GPU, top-node voxels merged by
  global index: the union equals the single-tree run node for node.

The oracle (oracle/lod_oracle.c, a 1-thread C restatement pinned to the
reference's own outputs) runs live; these tests take minutes.
"""
import numpy as np
import pytest

from common import assert_same_state, make_product, oracle_state, product_state, run_oracle

pytestmark = pytest.mark.gpu

PAPER = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=8 << 30, chunk_capacity=1000, grid_res=128,
             leaf_threshold=50_000, max_depth=20, backlog_capacity=64_000_000, spill_capacity=100_000_000)
BENCH_CAM = dict(position=(0.5, 0.5, -1.5), target=(0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=100.0, width=1024,
                 height=768)


def _stream(kind, count, seed0=1000):
    import sys

    sys.path.insert(0, __file__.rsplit("/", 2)[0])
    from bench import gen_batches

    return gen_batches(kind, count, seed0)


def _run_stream(params, batches, frames=None):
    """Oracle and product over the same batches, batch by batch; returns
    (oracle tree, product tree, product state, per-batch stats of both)."""
    from paper_2310_03567_b200 import insert_batch

    import oracle

    ot = oracle.OracleTree(params["bmin"], params["size"], grid_res=params["grid_res"],
                           leaf_threshold=params["leaf_threshold"], max_depth=params["max_depth"],
                           chunk_capacity=params["chunk_capacity"], arena_bytes=params["arena_bytes"],
                           backlog_capacity=params["backlog_capacity"], spill_capacity=params["spill_capacity"])
    tree, state = make_product(params)
    o_per, p_per = [], []
    for i, (x, c) in enumerate(batches):
        s = ot.insert_batch(x, c)
        o_per.append((s["n_voxels"], s["n_spill"], s["n_splits"]))
        insert_batch(tree, x, c, state)
        b = state._bstats
        p_per.append((int(b.n_voxels), int(b.n_spill), int(b.n_splits)))
        if frames is not None:
            frames(i, ot, tree)
    return ot, tree, state, o_per, p_per


def _render_vs_oracle(ot, tree, threshold=128.0):
    from paper_2310_03567_b200.render import Camera, Framebuffer, rasterize

    cam = Camera(**BENCH_CAM)
    fb, rep = rasterize(tree, cam, threshold=threshold)
    ofb = Framebuffer(cam.width, cam.height)
    drawn = ot.rasterize_nodes(rep.selected, cam.packed(), ofb.cells)
    assert drawn == rep.samples_drawn
    assert np.array_equal(fb.cells, ofb.cells)
    return rep


def test_config2_full_terrain_stream(gpu):
    batches = _stream("surface", 100)
    ot, tree, state, o_per, p_per = _run_stream(PAPER, batches)
    assert p_per == o_per
    st = state.stats
    assert st.voxels_created == ot.voxels_created and st.points == 100_000_000
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="config2_100M")
    rep = _render_vs_oracle(ot, tree)
    assert rep.samples_drawn > 1_000_000
    print(f"config 2: {tree.num_nodes} nodes, max spill {max(s for _, s, _ in p_per)}, "
          f"max new voxels {max(v for v, _, _ in p_per)}, render {rep.samples_drawn} samples")


def test_config4_skew_split_waves(gpu):
    batches = _stream("skew", 100)
    ot, tree, state, o_per, p_per = _run_stream(PAPER, batches)
    assert p_per == o_per
    spills = [s for _, s, _ in p_per]
    print("config 4 spill per batch (M):", [round(s / 1e6, 1) for s in spills])
    assert max(spills) > 20_000_000, "the stream must reach a split wave of > 20M spilled points"
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="config4_skew")
    tree.validate()


def test_config3_mesh_frames(gpu):
    """Insert + render per frame (config 3's loop) on a 20M-point mesh prefix."""
    frames = []

    def each_frame(i, ot, tree):
        rep = _render_vs_oracle(ot, tree)
        frames.append(rep.samples_drawn)

    batches = _stream("mesh", 20)
    ot, tree, state, o_per, p_per = _run_stream(PAPER, batches, frames=each_frame)
    assert p_per == o_per
    assert len(frames) == 20 and min(frames) > 0
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="config3_mesh")


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config5_partition_protocol_paper_params(gpu, world):
    """The warm-up / hand-off / partitioned protocol at paper parameters: the
    single-tree run vs `world` emulated rank trees fed by exact octant-prefix
    routing (plan over depth 1 for 2/4 ranks, depth 2 for 8), the top nodes'
    voxels merged across ranks by global index after every batch: the union
    equals the single tree node for node."""
    from paper_2310_03567_b200 import partition

    from common import assert_union_equals_single, emulate_partitioned

    params = dict(PAPER, arena_bytes=6 << 30)
    batches = _stream("surface", 24, seed0=5000)
    plan = partition.plan_owners(batches[:2], world)
    g, ranks, handed = emulate_partitioned(params, batches, plan)
    assert handed is not None and handed < 20
    checked = assert_union_equals_single(g, ranks, plan, label=f"config5 x{world}")
    assert checked > 100
    print(f"config 5 x{world}: {checked} (node, rank) copies equal, single tree {g.num_nodes} nodes, "
          f"hand-off after batch {handed}")


def test_node_ids_past_2_24(gpu):
    """Claim keys pack {epoch:8, node:56-cbits, cell:cbits}: with G = 2 the
    node field takes 53 bits and ids run to the reference's int32 range.  A
    tree of > 2^24 nodes (T = 0: every touched leaf splits down to depth 9;
    1.5M uniform points, ~22M nodes) against the oracle: node columns, counters, every
    grid byte and the sample sequences of 2000 random nodes."""
    import oracle
    from paper_2310_03567_b200 import insert_batch, synth

    params = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=1 << 30, chunk_capacity=1, grid_res=2,
                  leaf_threshold=0, max_depth=9, backlog_capacity=100_000_000, spill_capacity=100_000_000)
    xyz, rgba = synth.gen_uniform(1_500_000, 24)
    batches = [(xyz[i:i + 500_000], rgba[i:i + 500_000]) for i in range(0, 1_500_000, 500_000)]
    ot = oracle.OracleTree(params["bmin"], params["size"], grid_res=2, leaf_threshold=0, max_depth=9,
                           chunk_capacity=1, arena_bytes=params["arena_bytes"],
                           backlog_capacity=params["backlog_capacity"], spill_capacity=params["spill_capacity"])
    tree, state = make_product(params)
    for x, c in batches:
        ot.insert_batch(x, c)
        insert_batch(tree, x, c, state)
    want = ot.state()
    n = want["num_nodes"]
    assert n > (1 << 24), n
    assert tree.num_nodes == n
    for k in ("splits_total", "max_level", "allocated_total", "free_count", "arena_offset"):
        got = {"arena_offset": tree.arena.offset, "allocated_total": tree.pool.allocated_total,
               "free_count": tree.pool.free_count}.get(k, getattr(tree, k, None))
        assert int(got) == int(want[k]), k
    for k in ("parent", "level", "inner", "children", "count", "chunk_count", "grid_off"):
        assert np.array_equal(getattr(tree, k)[:n], want[k]), k
    assert np.array_equal(tree.bmin[:n].view(np.uint64), want["bmin"].view(np.uint64))
    inner = np.flatnonzero(want["inner"])
    v = ot._view()
    o_arena = np.ctypeslib.as_array(ctypes_u8(v.arena), shape=(int(v.arena_offset),))
    p_arena = tree._arena_bytes(0, int(v.arena_offset))
    offs = want["grid_off"][inner]
    assert np.array_equal(p_arena[offs], o_arena[offs])  # G = 2: one byte per grid
    rng = np.random.default_rng(0)
    for nid in rng.choice(n, 2000, replace=False):
        gx, gc = tree.gather_samples(int(nid))
        ox, oc = ot.gather_samples(int(nid))
        assert np.array_equal(gx, ox) and np.array_equal(gc, oc), nid


def ctypes_u8(addr):
    import ctypes

    return ctypes.cast(addr, ctypes.POINTER(ctypes.c_uint8))
