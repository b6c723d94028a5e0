"""Host time around each insert in the e2e frame loop (pinned host batches
through run_frame_updates): the call's own wall time and the host time
between calls, next to the device time per cycle -- with an early return
the host has until the previous cycle's tail ends to queue the next one."""
import collections
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2310_03567_b200.update as U
    from bench import gen_batches, new_tree

    bs = gen_batches("surface", 45)
    pin = [(torch.from_numpy(x).pin_memory().numpy(), torch.from_numpy(c.view(np.int32)).pin_memory().numpy().view(np.uint32))
           for x, c in bs]
    tree, state = new_tree(0, 16 << 30)
    marks = []
    orig = U.insert_batch

    devlog = []

    def timed(*a, **k):
        t0 = time.perf_counter()
        r = orig(*a, **k)
        marks.append((t0, time.perf_counter()))
        b = a[3]._bstats if len(a) > 3 else None
        if b is not None:
            devlog.append((round(float(b.device_ms), 3), round(float(b.device_ms_prev), 3)))
        return r

    U.insert_batch = timed
    q = collections.deque(pin[:25])
    while q:
        U.run_frame_updates(tree, q, state)
    U.wait_settled(tree, state)
    marks.clear()
    devlog.clear()
    q = collections.deque(pin[25:])
    t0 = time.perf_counter()
    while q:
        U.run_frame_updates(tree, q, state)
    dev = U.wait_settled(tree, state)
    wall = time.perf_counter() - t0
    calls = [(b - a) * 1e6 for a, b in marks]
    gaps = [(marks[i + 1][0] - marks[i][1]) * 1e6 for i in range(len(marks) - 1)]
    devms = list(devlog)
    # the same batches device-resident, same tree history, for comparison
    tree2, state2 = new_tree(0, 16 << 30)
    dv = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in bs]
    for i in range(25):
        orig(tree2, *dv[i], state2)
    U.wait_settled(tree2, state2)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    for i in range(25, 45):
        orig(tree2, *dv[i], state2)
    U.wait_settled(tree2, state2)
    torch.cuda.synchronize()
    wall2 = time.perf_counter() - t1
    if os.environ.get("HB_VERBOSE"):
        print("calls_us", [round(c) for c in calls])
        print("gaps_us", [round(g) for g in gaps])
        print("device_ms", devms)
    print(json.dumps({"device_resident_wall_ms_per_batch": round(wall2 / 20 * 1e3, 3)}))
    print(json.dumps({"batches": len(marks), "wall_ms_per_batch": round(wall / len(marks) * 1e3, 3),
                      "call_us_median": round(float(np.median(calls)), 1), "between_calls_us_median":
                      round(float(np.median(gaps)), 1), "between_calls_us_max": round(max(gaps), 1)}))


if __name__ == "__main__":
    main()
