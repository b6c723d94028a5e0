"""Host overhead per insert_batch: wall time of the call vs its device time."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import gen_batches, new_tree
    from paper_2310_03567_b200 import insert_batch, run_frame_updates
    from paper_2310_03567_b200 import _lib
    import ctypes

    batches = gen_batches("surface", 40)
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in batches]
    tree, state = new_tree(0, 8 << 30)
    for i in range(10):
        insert_batch(tree, *dev[i], state)
    walls, devs = [], []
    for i in range(10, 40):
        t0 = time.perf_counter()
        insert_batch(tree, *dev[i], state)
        walls.append((time.perf_counter() - t0) * 1e3)
        devs.append(state._bstats.device_ms)
    print("python insert_batch: wall %.3f ms, device %.3f ms, host-only %.3f ms (medians)" % (
        np.median(walls), np.median(devs), np.median(np.array(walls) - np.array(devs))))
    # raw C call with the same arguments
    tree2, state2 = new_tree(0, 8 << 30)
    lim = state2._limits
    lim.backlog_capacity, lim.spill_capacity = state2.config.backlog_capacity, state2.config.spill_capacity
    bs = _lib.LodBatchStats()
    walls = []
    for i in range(40):
        x, c = dev[i]
        t0 = time.perf_counter()
        tree2._L.lod_insert_batch(tree2.handle, _lib.ptr(x), _lib.ptr(c), c.numel(), ctypes.byref(lim),
                                  _lib.LOD_FLAG_DEVICE_INPUT, ctypes.byref(bs))
        if i >= 10:
            walls.append(((time.perf_counter() - t0) * 1e3, bs.device_ms))
    w = np.array(walls)
    print("C lod_insert_batch: wall %.3f ms, device %.3f ms, host-only %.3f ms" % (
        np.median(w[:, 0]), np.median(w[:, 1]), np.median(w[:, 0] - w[:, 1])))


if __name__ == "__main__":
    main()
