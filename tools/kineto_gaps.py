"""Device timeline of steady-state batches from CUPTI (torch.profiler): every
kernel / memcpy on the GPU with start and duration, and the idle gaps between
them, to see how much of a batch is launch / host-round-trip latency.

    python tools/kineto_gaps.py [--warm 20] [--batches 4] [--e2e]

--e2e: pinned host batches through the frame loop (run_frame_updates, the
bench's e2e path) instead of device-resident insert_batch calls.
"""
import argparse
import json
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    from bench import gen_batches, new_tree
    import collections

    from paper_2310_03567_b200 import insert_batch, run_frame_updates, wait_settled

    ap = argparse.ArgumentParser()
    ap.add_argument("--warm", type=int, default=20)
    ap.add_argument("--batches", type=int, default=4)
    ap.add_argument("--e2e", action="store_true")
    a = ap.parse_args()
    bs = gen_batches("surface", a.warm + a.batches)
    if a.e2e:
        src = []
        for x, c in bs:
            src.append((torch.from_numpy(x).pin_memory().numpy(),
                        torch.from_numpy(c.view(np.int32)).pin_memory().numpy().view(np.uint32)))
    else:
        src = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in bs]
    tree, state = new_tree(0, 16 << 30)

    def feed(lo, hi):
        if a.e2e:
            q = collections.deque(src[lo:hi])
            while q:
                run_frame_updates(tree, q, state)
        else:
            for i in range(lo, hi):
                insert_batch(tree, *src[i], state)

    feed(0, a.warm)
    wait_settled(tree, state)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        feed(a.warm, a.warm + a.batches)
        wait_settled(tree, state)
        torch.cuda.synchronize()
    path = os.path.join(tempfile.mkdtemp(), "trace.json")
    prof.export_chrome_trace(path)
    ev = json.load(open(path))["traceEvents"]
    ks = [e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset") and "dur" in e]
    ks.sort(key=lambda e: e["ts"])
    t0 = ks[0]["ts"]
    busy = 0.0
    end = t0
    gaps = []
    for e in ks:
        gap = e["ts"] - end
        if gap > 0:
            gaps.append((gap, e["name"][:28]))
        busy += max(0.0, e["ts"] + e["dur"] - max(e["ts"], end))
        end = max(end, e["ts"] + e["dur"])
        print(f"{e['ts'] - t0:9.1f} {e['dur']:7.1f} gap {max(gap, 0):6.1f}  {e['name'][:60]}")
    span = end - t0
    print(f"span {span:.1f} us over {a.batches} batches ({span / a.batches:.1f} us/batch), busy {busy:.1f} us "
          f"({100 * busy / span:.1f}%), idle {span - busy:.1f} us")
    gaps.sort(reverse=True)
    print("largest gaps (us, next kernel):", [(round(g, 1), n) for g, n in gaps[:12]])


if __name__ == "__main__":
    main()
