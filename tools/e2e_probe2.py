"""Per-batch device time and wall time in the frame loop vs device-resident."""
import collections
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import gen_batches, new_tree
    from paper_2310_03567_b200 import insert_batch, update

    nb = 40
    batches = gen_batches("surface", nb)
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in batches]
    pin = []
    for x, c in batches:
        px = torch.from_numpy(x).pin_memory()
        pc = torch.from_numpy(c.view(np.int32)).pin_memory()
        pin.append((px.numpy(), pc.numpy().view(np.uint32)))
    for kind in ("device", "staged"):
        tree, state = new_tree(0, 8 << 30)
        for i in range(5):
            insert_batch(tree, *dev[i], state)
        torch.cuda.synchronize()
        devms, walls, pre = [], [], []
        src = dev if kind == "device" else pin
        for i in range(5, nb):
            t0 = time.perf_counter()
            if kind == "staged" and i + 1 < nb:
                update._prefetch(tree, pin[i + 1])
            t1 = time.perf_counter()
            insert_batch(tree, *src[i], state)
            t2 = time.perf_counter()
            pre.append((t1 - t0) * 1e3)
            walls.append((t2 - t1) * 1e3)
            devms.append(state._bstats.device_ms)
        print(f"{kind}: prefetch call {np.median(pre):.3f} ms, insert wall {np.median(walls):.3f} ms, "
              f"device {np.median(devms):.3f} ms, sum wall {sum(walls) + sum(pre):.1f} ms")
        tree.close()


if __name__ == "__main__":
    main()
