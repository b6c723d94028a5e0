"""Cost of the multi-GPU routing's local part (owner prefix + stable bucketing) on one GPU."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2310_03567_b200 import multigpu, partition, synth

    x, c = synth.gen_surface(1_000_000, 5)
    plan = partition.plan_owners([(x, c)], 8)
    xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()
    for _ in range(3):
        own = multigpu.owners_device(xd, plan)
        order = torch.sort(own, stable=True).indices
        rec = torch.cat([xd.view(torch.int32), cd.reshape(-1, 1)], dim=1)[order]
        cnt = torch.bincount(own, minlength=8)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        own = multigpu.owners_device(xd, plan)
        order = torch.sort(own, stable=True).indices
        rec = torch.cat([xd.view(torch.int32), cd.reshape(-1, 1)], dim=1)[order]
        cnt = torch.bincount(own, minlength=8).tolist()
    torch.cuda.synchronize()
    print(f"route local part (owners + stable bucket + pack + counts): {(time.perf_counter() - t0) / 20 * 1e3:.3f} ms per 1M stripe")


if __name__ == "__main__":
    main()


def fused():
    import torch

    from paper_2310_03567_b200 import multigpu, partition, synth

    x, c = synth.gen_surface(1_000_000, 5)
    plan = partition.plan_owners([(x, c)], 8)
    xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()
    for _ in range(3):
        rec, cnt, st = multigpu.bucket(xd, cd, plan, 8)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        rec, cnt, st = multigpu.bucket(xd, cd, plan, 8)
    e1.record()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        rec, cnt, st = multigpu.bucket(xd, cd, plan, 8)
        cnt.tolist()
    print(f"lod_route_bucket: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us device per 1M stripe; "
          f"{(time.perf_counter() - t0) / 20 * 1e3:.3f} ms wall incl. the counts read-back")


fused()
