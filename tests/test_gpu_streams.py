"""Device inputs produced asynchronously on the caller's stream: insert_batch /
insert_records must read a batch only once the copy that writes it has run
(LodLimits.input_stream + LOD_FLAG_INPUT_STREAM, an event wait on the tree's
stream, no host sync).  The copy is queued behind a ~20 ms spin on a side
stream, over a buffer holding a different valid batch; the tree must match
one built from the same batches with synchronised inputs."""
import numpy as np
import pytest

from common import assert_same_state, make_product, product_state

pytestmark = pytest.mark.gpu

PARAMS = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=1 << 30, chunk_capacity=500, grid_res=32,
              leaf_threshold=2000, max_depth=14, backlog_capacity=10_000_000, spill_capacity=100_000_000)


@pytest.mark.parametrize("packed", [False, True])
def test_inputs_ordered_after_producer_stream(gpu, packed):
    import torch

    from paper_2310_03567_b200 import insert_batch, synth
    from paper_2310_03567_b200.update import insert_records

    want_t, want_s = make_product(PARAMS)
    got_t, got_s = make_product(PARAMS)
    decoy_x, decoy_c = synth.gen_uniform(60_000, 999)
    side = torch.cuda.Stream()
    for i in range(4):
        x, c = synth.gen_surface(60_000, 70 + i)
        rec = np.concatenate([x.view(np.int32), c.view(np.int32).reshape(-1, 1)], axis=1)
        if packed:
            insert_records(want_t, torch.from_numpy(rec).cuda(), want_s)
        else:
            insert_batch(want_t, torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda(), want_s)
        # buffers hold the decoy batch (synchronised), the real one lands late
        dx = torch.from_numpy(decoy_x).cuda()
        dc = torch.from_numpy(decoy_c.view(np.int32)).cuda()
        drec = torch.cat([dx.view(torch.int32), dc.reshape(-1, 1)], dim=1).contiguous()
        hx = torch.from_numpy(x).pin_memory()
        hc = torch.from_numpy(c.view(np.int32)).pin_memory()
        hrec = torch.from_numpy(rec).pin_memory()
        torch.cuda.synchronize()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            torch.cuda._sleep(40_000_000)  # ~20 ms of spinning ahead of the copy
            if packed:
                drec.copy_(hrec, non_blocking=True)
                insert_records(got_t, drec, got_s)
            else:
                dx.copy_(hx, non_blocking=True)
                dc.copy_(hc, non_blocking=True)
                insert_batch(got_t, dx, dc, got_s)
        torch.cuda.synchronize()
    assert_same_state(product_state(got_t), product_state(want_t), chunk_ids=True,
                      label="packed" if packed else "xyz+rgba")


def test_input_on_other_device_rejected(gpu):
    import torch

    from paper_2310_03567_b200 import insert_batch, synth

    if torch.cuda.device_count() < 2:
        pytest.skip("one device")
    t, s = make_product(PARAMS)
    x, c = synth.gen_uniform(1000, 1)
    with pytest.raises(ValueError):
        insert_batch(t, torch.from_numpy(x).to("cuda:1"), torch.from_numpy(c.view(np.int32)).to("cuda:1"), s)


@pytest.mark.parametrize("packed", [False, True])
def test_inputs_reused_right_after_insert(gpu, packed):
    """insert returns before the last pass's store has re-read the batch: the
    caller's stream is made to wait, so overwriting the input at once is safe."""
    import torch

    from paper_2310_03567_b200 import insert_batch, synth
    from paper_2310_03567_b200.update import insert_records

    want_t, want_s = make_product(PARAMS)
    got_t, got_s = make_product(PARAMS)
    for i in range(4):
        x, c = synth.gen_surface(60_000, 90 + i)
        rec = np.concatenate([x.view(np.int32), c.view(np.int32).reshape(-1, 1)], axis=1)
        insert_batch(want_t, x, c, want_s)
        if packed:
            drec = torch.from_numpy(rec).cuda()
            insert_records(got_t, drec, got_s)
            drec.fill_(0x7FC00000)  # NaN coordinates
        else:
            dx, dc = torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()
            insert_batch(got_t, dx, dc, got_s)
            dx.fill_(float("nan"))
            dc.fill_(0)
    torch.cuda.synchronize()
    assert_same_state(product_state(got_t), product_state(want_t), chunk_ids=True,
                      label="packed" if packed else "xyz+rgba")


def test_device_time_reported_after_early_return(gpu):
    """Early-returning calls report device_ms = -1; the next call (device_ms_prev)
    or wait_settled reports it, and UpdateStats.device_seconds gets every batch."""
    from paper_2310_03567_b200 import insert_batch, synth, wait_settled

    t, s = make_product(PARAMS)
    got = []
    for i in range(5):
        x, c = synth.gen_surface(60_000, 110 + i)
        insert_batch(t, x, c, s)
        b = s._bstats
        got.append((float(b.device_ms), float(b.device_ms_prev)))
    last = wait_settled(t, s)
    assert all(d < 0 for d, _ in got)  # host input, no delta / profile: every call returned early
    assert got[0][1] < 0 and all(p > 0 for _, p in got[1:])
    assert last > 0 and wait_settled(t, s) < 0  # nothing outstanding the second time
    total = sum(p for _, p in got[1:]) + last
    assert s.stats.device_seconds == pytest.approx(total * 1e-3, rel=1e-4)
    # profile / delta calls are synchronous: their own time, and the pending one
    x, c = synth.gen_surface(60_000, 120)
    insert_batch(t, x, c, s)
    insert_batch(t, *synth.gen_surface(60_000, 121), s, profile=True)
    assert s._bstats.device_ms > 0 and s._bstats.device_ms_prev > 0
    assert wait_settled(t, s) < 0
