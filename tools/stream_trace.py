"""Per-batch trace of a config stream (device-resident inputs):

    LOD_DEBUG=1 python tools/stream_trace.py --config terrain --batches 100
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import CONFIGS, gen_batches, new_tree
    from paper_2310_03567_b200 import insert_batch, wait_settled

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="terrain")
    ap.add_argument("--batches", type=int, default=100)
    ap.add_argument("--repeat", type=int, default=1)
    a = ap.parse_args()
    batches = gen_batches(CONFIGS[a.config][0], a.batches)
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in batches]
    for rep in range(a.repeat):
        tree, state = new_tree(0, 16 << 30)
        tot = 0.0
        for i in range(a.batches):
            insert_batch(tree, *dev[i], state)
            b = state._bstats
            ms = b.device_ms if b.device_ms >= 0 else wait_settled(tree)  # serialised: time each batch
            tot += ms
            print(f"rep {rep} batch {i:3d} ms {ms:7.3f} n_s {b.n_spill:8d} n_v {b.n_voxels:8d} "
                  f"iters {b.iterations} splits {b.n_splits:3d} nodes {b.num_nodes:6d} launches {b.launches}",
                  flush=True)
        print(f"rep {rep} total {tot:.1f} ms -> {a.batches * 1e3 / tot:.1f} Mpts/s", flush=True)
        tree.close()


if __name__ == "__main__":
    main()
