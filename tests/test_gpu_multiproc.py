"""bench.py's multi-process path (torchrun, one process per rank) on the test
box: ranks share the GPU and exchange over gloo (LOD_DIST_BACKEND=gloo), so
warm-up on rank 0, the packed-tree broadcast, the routing kernels + all-to-all,
the partitioned inserts and the max-over-ranks timing all run for real."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_two_ranks_over_gloo(gpu, tmp_path):
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, LOD_DIST_BACKEND="gloo", LOD_POOL_RESERVE_MIB="512")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--arena-gib", "2"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints the line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["batch_points"] == 1_000_000 and "GLOO" in d["notes"]["parallelism"]
    assert d["notes"]["global_batch"].startswith("2 x 1M")
