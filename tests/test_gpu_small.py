"""The small-batch path (lod_small.cuh: one kernel per cycle for host batches
of <= 256 points, queued without a host wait when no error is possible)
against the oracle: C1's parameters (test_acceptance.py:81-101: G=16, T=100,
C=1000, depth 12) at batch sizes 1 and 7, small and pipeline batches
interleaved on one tree, tiny chunks, the depth cap, T = 0, an offset root,
the three fatal errors at the reference's batch, and the UpdateStats totals
folded in by the settle."""
import zlib

import numpy as np
import pytest

from common import assert_same_state, make_product, oracle_state, product_state, run_oracle, run_product

pytestmark = pytest.mark.gpu


def _params(**kw):
    p = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=256 << 20, chunk_capacity=1000, grid_res=16,
             leaf_threshold=100, max_depth=12, backlog_capacity=10_000_000, spill_capacity=100_000_000)
    p.update(kw)
    return p


def _cloud(n, seed, kind="uniform"):
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        xyz = rng.random((n, 3)).astype(np.float32)
    else:
        xy = rng.random((n, 2))
        z = 0.5 + 0.2 * np.sin(6.0 * xy[:, 0]) * np.cos(5.0 * xy[:, 1])
        xyz = np.column_stack([xy[:, 0], xy[:, 1], z]).astype(np.float32)
    np.clip(xyz, 0.0, np.nextafter(np.float32(1.0), np.float32(0.0)), out=xyz)
    return xyz, rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)


def _split(xyz, rgba, sizes):
    out, i, k = [], 0, 0
    while i < len(rgba):
        b = sizes[k % len(sizes)]
        out.append((xyz[i:i + b], rgba[i:i + b]))
        i += b
        k += 1
    return out


CASES = [
    # label, n, kind, batch sizes (cycled), params
    ("c1_uniform_bs1", 6000, "uniform", [1], _params()),
    ("c1_surface_bs7", 30_000, "surface", [7], _params()),
    ("mixed_sizes", 60_000, "surface", [1, 7, 256, 257, 1000, 3, 40], _params()),
    ("tiny_chunks", 5000, "uniform", [1, 2, 5], _params(grid_res=4, leaf_threshold=10, max_depth=6, chunk_capacity=3)),
    ("depth_cap", 3000, "surface", [7], _params(leaf_threshold=4, max_depth=3, chunk_capacity=2)),
    ("threshold_zero", 400, "uniform", [1, 3], _params(leaf_threshold=0, max_depth=5, chunk_capacity=4)),
    ("grid128_t1000", 40_000, "surface", [256, 100], _params(grid_res=128, leaf_threshold=1000, max_depth=20)),
]


@pytest.mark.parametrize("label,n,kind,sizes,params", CASES, ids=[c[0] for c in CASES])
def test_small_batches_match_oracle(gpu, label, n, kind, sizes, params):
    xyz, rgba = _cloud(n, zlib.crc32(label.encode()) & 0xFFFF, kind)
    batches = _split(xyz, rgba, sizes)
    ot, oerr, oper = run_oracle(params, batches)
    tree, state, err, per = run_product(params, batches)  # reads state.stats after every batch
    assert err == oerr == ""
    assert per == oper
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label=label)
    tree.validate()


def test_offset_root_small_batches(gpu):
    params = _params(bmin=(-3.0, 2.5, 10.0), size=6.5, grid_res=8, leaf_threshold=20)
    xyz, rgba = _cloud(8000, 5)
    xyz = (xyz.astype(np.float64) * 6.5 + np.array([-3.0, 2.5, 10.0])).astype(np.float32)
    batches = _split(xyz, rgba, [1, 7, 13])
    ot, _, oper = run_oracle(params, batches)
    tree, state, err, per = run_product(params, batches)
    assert err == "" and per == oper
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="offset_small")


def test_queued_cycles_fold_into_stats(gpu):
    """A stream of tiny batches without reading the stats in between: every
    cycle is queued, and the first read of state.stats folds them in."""
    from paper_2310_03567_b200 import insert_batch

    params = _params()
    xyz, rgba = _cloud(20_000, 77, "surface")
    batches = _split(xyz, rgba, [1, 7])
    ot, _, oper = run_oracle(params, batches)
    tree, state = make_product(params)
    for x, c in batches:
        insert_batch(tree, x, c, state)
    assert state._unsettled  # cycles were queued without a host wait
    st = state.stats
    assert not state._unsettled
    assert st.batches == len(batches) and st.points == len(rgba)
    want_v, want_s, want_n, want_hb, want_hs = oper[-1]
    assert (st.voxels_created, st.splits, st.nodes, st.backlog_high_water, st.spill_high_water) == (
        want_v, want_s, want_n, want_hb, want_hs)
    assert st.update_seconds > 0 and st.device_seconds > 0
    assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="queued")


@pytest.mark.parametrize("which", ["backlog", "spill", "arena"])
def test_small_batch_errors_match_oracle(gpu, which):
    """The fatal errors on the small path (run synchronously when the worst
    case could overflow) at the same batch as the reference."""
    kw = {"backlog": dict(backlog_capacity=40), "spill": dict(spill_capacity=50, leaf_threshold=60),
          "arena": dict(arena_bytes=150_000, chunk_capacity=200)}[which]
    params = _params(**kw)
    xyz, rgba = _cloud(6000, 11)
    batches = _split(xyz, rgba, [7, 1, 30])
    ot, oerr, oper = run_oracle(params, batches)
    tree, state, err, per = run_product(params, batches)
    assert oerr != ""
    assert err == oerr
    assert per == oper


def test_small_path_equals_pipeline(gpu):
    """The same stream through the small path and through the pipeline
    (LOD_NO_SMALL=1 in a child process): identical trees, chunk ids aside."""
    import json
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    code = f"""
import sys, json, numpy as np
sys.path.insert(0, {os.path.dirname(here)!r}); sys.path.insert(0, {here!r})
from common import run_product, product_state
from test_gpu_small import _cloud, _split, _params
xyz, rgba = _cloud(9000, 3, "surface")
tree, state, err, per = run_product(_params(), _split(xyz, rgba, [1, 7, 64]))
st = product_state(tree)
np.savez(sys.argv[1], **{{k: np.asarray(v) for k, v in st.items()}})
print(json.dumps(per[-1]))
"""
    outs = []
    for env_extra, name in (({}, "small"), ({"LOD_NO_SMALL": "1"}, "pipe")):
        path = os.path.join("/tmp", f"small_vs_pipe_{name}_{os.getpid()}.npz")
        r = subprocess.run([sys.executable, "-c", code, path], env=dict(os.environ, **env_extra), capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        z = np.load(path)
        outs.append(({k: z[k] for k in z.files}, json.loads(r.stdout.strip().splitlines()[-1])))
        os.remove(path)
    (a, pa), (b, pb) = outs
    assert pa == pb
    assert_same_state(a, b, chunk_ids=False, label="small_vs_pipeline")


def test_directory_overflow_rebuild(gpu):
    """Small cycles size the chunk directory softly; a relocation that finds
    no room flags the control block and the host rebuilds every directory
    from the chains at its next sync.  LOD_DIR_FORCE_OVERFLOW=1 (child
    process) makes every small-cycle relocation fail: the tree, the
    directory (validate walks it against the lists) and a render through it
    must still equal the oracle's."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    code = f"""
import sys, numpy as np
sys.path.insert(0, {os.path.dirname(here)!r}); sys.path.insert(0, {here!r})
from common import run_oracle, run_product, product_state, oracle_state, assert_same_state
from test_gpu_small import _cloud, _split, _params
from paper_2310_03567_b200 import insert_batch
from paper_2310_03567_b200.render import Camera, Framebuffer, rasterize
params = _params(grid_res=8, leaf_threshold=30, chunk_capacity=4)
xyz, rgba = _cloud(12000, 9, "surface")
batches = _split(xyz, rgba, [1, 7, 300, 5])
ot, oerr, oper = run_oracle(params, batches)
tree, state, err, per = run_product(params, batches)
assert err == oerr == "" and per == oper
assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label="dir_overflow")
tree.validate()
# queued cycles only, then a render (the rebuild runs at the render's sync)
more = _split(*_cloud(3000, 10, "surface"), [1, 3])
for x, c in more:
    insert_batch(tree, x, c, state)
    ot.insert_batch(x, c)
cam = Camera((0.5, 0.45, -1.3), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=50.0, width=256, height=192)
fb, rep = rasterize(tree, cam, threshold=-1.0)
ofb = Framebuffer(cam.width, cam.height)
assert ot.rasterize_nodes(rep.selected, cam.packed(), ofb.cells) == rep.samples_drawn
assert np.array_equal(fb.cells, ofb.cells)
tree.validate()
print("ok")
"""
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, LOD_DIR_FORCE_OVERFLOW="1", LOD_DEBUG="1"),
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "chunk directory overflow: rebuilding" in r.stderr
