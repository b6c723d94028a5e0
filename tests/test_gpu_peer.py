"""The fused peer-memory multi-GPU path (multigpu.PeerRouter /
PeerFramebuffers: CUDA IPC windows, bucket scatter straight into the owners'
windows, depth-min composite over peer memory) run for real: N processes under
torchrun sharing the test box's GPU, ordered over gloo (tests/peer_worker.py).
Every owned prefix subtree must equal the single-tree run path by path
(samples and grid cells), every rank's copy of every top node must equal the
single tree's (the voxels merged by global index), and every rank's
composite must equal the single-tree render."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from common import make_product

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
P = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=512 << 20, chunk_capacity=256, grid_res=32,
         leaf_threshold=400, max_depth=14, backlog_capacity=10_000_000, spill_capacity=100_000_000)


@pytest.mark.parametrize("world,depth,wait", [(2, 1, "host"), (4, 2, "host"), (2, 1, "device")])
def test_peer_route_and_composite_match_single_tree(gpu, tmp_path, world, depth, wait):
    """wait: how the ranks wait on the window flags -- "device" (spinning
    wait kernels: the multi-GPU mode) or "host" (polled from the host: the
    mode ranks sharing one GPU select, as here)."""
    from oracle.rebuild import tree_paths
    from paper_2310_03567_b200 import insert_batch, synth
    from paper_2310_03567_b200.render import Camera, rasterize

    n_batches, stripe = 12, 40_000 // world
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, LOD_POOL_RESERVE_MIB="256", LOD_ROUTE_WAIT=wait)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(HERE, "peer_worker.py"),
           str(tmp_path), str(n_batches), str(stripe), str(depth)]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]

    g, gs = make_product(P)
    for i in range(n_batches):
        x, c = synth.gen_surface(world * stripe, 300 + i)
        insert_batch(g, x, c, gs)
    gp = tree_paths(g.inner, g.children)
    ranks = [dict(np.load(os.path.join(tmp_path, f"rank{k}.npz"))) for k in range(world)]
    owned = {}
    for k, d in enumerate(ranks):
        for key in d:
            if key.startswith("p_"):
                assert key not in owned, key  # prefixes are disjoint across ranks
                owned[key] = k
    deep = [p for p in gp if len(p) >= depth]
    assert len(owned) == len(deep)
    for path in deep:
        key = "".join(map(str, path))
        d = ranks[owned["p_" + key]]
        xs, cs = g.gather_samples(gp[path])
        assert np.array_equal(d["p_" + key], np.concatenate([xs.view(np.uint32), cs.reshape(-1, 1)], axis=1)), path
        if g.inner[gp[path]]:
            assert np.array_equal(d["g_" + key], g.occupied_cells(gp[path])), path
    # the replicated top nodes: every rank's copy is the single-tree sequence
    top = [p for p in gp if len(p) < depth]
    for path in top:
        key = "".join(map(str, path))
        xs, cs = g.gather_samples(gp[path])
        want = np.concatenate([xs.view(np.uint32), cs.reshape(-1, 1)], axis=1)
        for k, d in enumerate(ranks):
            got = d["t_" + key]
            diff = np.flatnonzero((got != want).any(axis=1))[:5] if got.shape == want.shape else None
            assert np.array_equal(got, want), (path, k, got.shape, want.shape, diff)
            assert np.array_equal(d["tg_" + key], g.occupied_cells(gp[path])), (path, k)
    cam = Camera((0.5, 0.45, -1.3), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=50.0, width=320, height=240)
    for thr, name in ((-1.0, "comp_all"), (64.0, "comp_64")):
        want, _ = rasterize(g, cam, threshold=thr)
        for d in ranks:
            assert np.array_equal(d[name], want.cells), (thr, name)
