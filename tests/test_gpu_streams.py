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
