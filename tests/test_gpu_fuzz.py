"""Randomised parity: 120 seeded configurations (grid 2..64, thresholds, chunk
capacities, depth caps, batch sizes 1..5000, all point generators, offset
non-power-of-two roots, duplicate-heavy inputs, small arena / backlog /
spill capacities that trip the fatal errors) through the GPU path and the
oracle, compared bit-exactly (every node column except chunk ids, every
record sequence, every bitgrid, pool counters, per-batch stats) -- the
reference suite's hypothesis property (test_update.py:396-412) as a fixed,
reproducible sample."""
import numpy as np
import pytest

from common import assert_same_state, oracle_state, product_state, run_oracle, run_product

pytestmark = pytest.mark.gpu


def _case(seed):
    from paper_2310_03567_b200 import synth

    rng = np.random.default_rng(seed)
    g = int(rng.choice([2, 4, 6, 8, 16, 32, 64]))
    params = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=256 << 20,
                  chunk_capacity=int(rng.choice([1, 2, 3, 7, 16, 100, 1000])), grid_res=g,
                  leaf_threshold=int(rng.choice([1, 2, 5, 20, 64, 300])), max_depth=int(rng.integers(1, 14)),
                  backlog_capacity=10_000_000, spill_capacity=100_000_000)
    n = int(rng.integers(1, 6000))
    kind = rng.choice(["uniform", "surface", "skew", "mesh", "dups"])
    if kind == "dups":  # few distinct positions, many repeats
        base = rng.random((max(1, n // 50), 3)).astype(np.float32)
        xyz = base[rng.integers(0, len(base), n)]
        rgba = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    elif kind == "mesh":
        xyz, rgba = synth.gen_mesh(n, seed, synth.mesh_scene(16, seed))
    else:
        xyz, rgba = synth.GENERATORS[str(kind)](n, seed)
    if rng.random() < 0.3:  # offset, non-power-of-two root
        lo = rng.uniform(-5, 5, 3)
        size = float(rng.uniform(0.3, 9.0))
        params["bmin"], params["size"] = tuple(float(v) for v in lo), size
        xyz = (xyz.astype(np.float64) * size + lo).astype(np.float32)
    r = rng.random()
    if r < 0.08:  # fatal paths: the first overflow must hit at the same batch with the same type
        params["arena_bytes"] = int(rng.integers(2_000, 400_000))
    elif r < 0.14:
        params["backlog_capacity"] = int(rng.integers(1, 60))
    bs = int(rng.choice([1, 3, 17, 128, 999, 5000]))
    if 0.14 <= r < 0.20:  # leaves fill over several batches, then split past the spill cap
        params["spill_capacity"] = int(rng.integers(1, 100))
        params["leaf_threshold"], params["max_depth"], bs = 64, max(params["max_depth"], 3), 17
    batches = [(xyz[i:i + bs], rgba[i:i + bs]) for i in range(0, n, bs)][:300]
    return params, batches


@pytest.mark.parametrize("seed", range(120))
def test_random_configuration_matches_oracle(gpu, seed):
    params, batches = _case(1000 + seed)
    ot, oerr, oper = run_oracle(params, batches)
    tree, state, err, per = run_product(params, batches)
    assert err == oerr
    assert per == oper
    if not err:
        assert_same_state(product_state(tree), oracle_state(ot), chunk_ids=False, label=f"fuzz{seed}")
