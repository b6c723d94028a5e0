"""Is the first DMA from freshly pinned pages slower?  The e2e frame loop over
the same pinned batches twice (two fresh trees) in one process."""
import collections
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import gen_batches, new_tree
    from paper_2310_03567_b200 import insert_batch, run_frame_updates, wait_settled

    nb = 100
    batches = gen_batches("surface", nb)
    pin = []
    for x, c in batches:
        px = torch.from_numpy(x).pin_memory()
        pc = torch.from_numpy(c.view(np.int32)).pin_memory()
        pin.append((px.numpy(), pc.numpy().view(np.uint32)))
    for rep in range(3):
        tree, state = new_tree(0, 8 << 30)
        for i in range(5):
            insert_batch(tree, *pin[i], state)
        wait_settled(tree, state)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q = collections.deque(pin[5:])
        while q:
            run_frame_updates(tree, q, state)
        wait_settled(tree, state)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"rep {rep}: {95 / dt:.1f} Mpts/s e2e (wall)", flush=True)
        tree.close()


if __name__ == "__main__":
    main()
