"""LOD_DEBUG=2 python tools/feed_probe.py: frame loop over pinned batches, with the staged-copy state per insert."""
import collections
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import gen_batches, new_tree
    from paper_2310_03567_b200 import insert_batch, run_frame_updates

    batches = gen_batches("surface", 30)
    pin = []
    for x, c in batches:
        pin.append((torch.from_numpy(x).pin_memory().numpy(),
                    torch.from_numpy(c.view(np.int32)).pin_memory().numpy().view(np.uint32)))
    tree, state = new_tree(0, 8 << 30)
    for i in range(5):
        insert_batch(tree, *pin[i], state)
    q = collections.deque(pin[5:])
    state.clock.budget_ms = 1e9
    run_frame_updates(tree, q, state)


if __name__ == "__main__":
    main()
