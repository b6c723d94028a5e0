"""Per-batch phase times (profile mode CUDA events) of a config stream."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import CONFIGS, gen_batches, new_tree
    from paper_2310_03567_b200 import insert_batch

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="terrain")
    ap.add_argument("--batches", type=int, default=20)
    a = ap.parse_args()
    batches = gen_batches(CONFIGS[a.config][0], a.batches)
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in batches]
    tree, state = new_tree(0, 16 << 30)
    for i in range(a.batches):
        insert_batch(tree, *dev[i], state, profile=True)
        b = state.last
        ph = " ".join(f"{k}={v * 1e3:6.1f}" for k, v in b["phase_ms"].items())
        print(f"batch {i:3d} n_s {b['n_spill']:8d} n_v {b['n_voxels']:8d} it {b['iterations']} | {ph}", flush=True)


if __name__ == "__main__":
    main()
