"""Phase times (profile mode) at points along a long terrain stream."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import new_tree
    from paper_2310_03567_b200 import insert_batch, synth

    n_b = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    tree, state = new_tree(0, 32 << 30)
    for i in range(n_b):
        x, c = synth.gen_surface(1_000_000, 1000 + i)
        xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()
        prof = i % 50 == 49 or i >= n_b - 3
        insert_batch(tree, xd, cd, state, profile=prof)
        if prof:
            b = state.last
            ph = " ".join(f"{k}={v * 1e3:6.1f}" for k, v in b["phase_ms"].items())
            print(f"batch {i:4d} nodes {b['num_nodes']:6d} chunks {b['allocated_total']:8d} n_s {b['n_spill']:7d} "
                  f"n_v {b['n_voxels']:8d} | {ph}", flush=True)


if __name__ == "__main__":
    main()
