"""GPU parity of the routing kernels (lod_route_bucket, multigpu.bucket): every
stripe bucketed by owner rank with the reference's float64 descent rule,
stable (global order kept inside a bucket), packed as 16-byte records -- checked
against the numpy restatement (partition.take) for 2/4/8/64 ranks, boundary
points on the split planes, an offset non-unit root, an empty stripe; and the
packed-record insert (insert_records) against insert_batch."""
import numpy as np
import pytest

from common import assert_same_state, make_product, product_state

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world,depth", [(2, 1), (4, 1), (8, 2), (64, 2)])
def test_bucket_matches_partition_take(gpu, world, depth):
    import torch

    from paper_2310_03567_b200 import multigpu, partition, synth

    xyz, _ = synth.gen_surface(300_000, 21)
    edge = np.array([[0.5, 0.5, 0.5], [0.25, 0.75, 0.5], [0.0, 0.999, 0.125], [0.75, 0.25, 0.25]], np.float32)
    xyz = np.concatenate([xyz, edge])
    rgba = np.arange(len(xyz), dtype=np.uint32)  # colour = input index
    plan = partition.plan_owners([(xyz, rgba)], world, depth=depth)
    rec, counts, starts = multigpu.bucket(torch.from_numpy(xyz).cuda(), torch.from_numpy(rgba.view(np.int32)).cuda(),
                                          plan, world)
    rec, counts, starts = rec.cpu().numpy(), counts.cpu().numpy(), starts.cpu().numpy()
    assert counts.sum() == len(xyz) and np.array_equal(starts, np.concatenate([[0], np.cumsum(counts)[:-1]]))
    for r in range(world):
        want_x, want_c = partition.take(plan, xyz, rgba, r)
        part = rec[starts[r]:starts[r] + counts[r]]
        assert np.array_equal(part[:, 3].view(np.uint32), want_c), r
        assert np.array_equal(part[:, :3].copy().view(np.float32), want_x), r


def test_bucket_offset_root_and_empty(gpu):
    import torch

    from paper_2310_03567_b200 import multigpu, partition

    rng = np.random.default_rng(3)
    lo, size = (-3.0, 2.5, 10.0), 6.5
    xyz = (rng.random((50_000, 3)) * size + np.array(lo)).astype(np.float32)
    rgba = np.arange(len(xyz), dtype=np.uint32)
    plan = partition.plan_owners([(xyz, rgba)], 4, bmin=lo, size=size)
    rec, counts, starts = multigpu.bucket(torch.from_numpy(xyz).cuda(), torch.from_numpy(rgba.view(np.int32)).cuda(),
                                          plan, 4, bmin=lo, size=size)
    rec, counts, starts = rec.cpu().numpy(), counts.cpu().numpy(), starts.cpu().numpy()
    for r in range(4):
        _, want_c = partition.take(plan, xyz, rgba, r, bmin=lo, size=size)
        assert np.array_equal(rec[starts[r]:starts[r] + counts[r], 3].view(np.uint32), want_c)
    e, ec, es = multigpu.bucket(torch.empty((0, 3), device="cuda"), torch.empty(0, dtype=torch.int32, device="cuda"),
                                plan, 4)
    assert e.shape == (0, 4) and ec.cpu().tolist() == [0, 0, 0, 0]


def test_insert_records_matches_insert_batch(gpu):
    import torch

    from paper_2310_03567_b200 import insert_batch, synth
    from paper_2310_03567_b200.update import insert_records

    params = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=1 << 30, chunk_capacity=500, grid_res=32,
                  leaf_threshold=2000, max_depth=14, backlog_capacity=10_000_000, spill_capacity=100_000_000)
    a, sa = make_product(params)
    b, sb = make_product(params)
    c, sc = make_product(params)
    for i in range(5):
        x, col = synth.gen_surface(80_000, 40 + i)
        insert_batch(a, x, col, sa)
        rec = np.concatenate([x.view(np.int32), col.view(np.int32).reshape(-1, 1)], axis=1)
        insert_records(b, torch.from_numpy(rec).cuda(), sb)  # device records
        insert_records(c, rec, sc)  # host records
    want = product_state(a)
    assert_same_state(product_state(b), want, chunk_ids=True, label="records_dev")
    assert_same_state(product_state(c), want, chunk_ids=True, label="records_host")
