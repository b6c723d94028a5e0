"""Per-frame split of config 3's loop (insert a 1M batch + rasterize at the
bench camera) on a fresh tree: wall ms of the insert and of the render."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import gen_batches, new_tree
    from paper_2310_03567_b200 import insert_batch
    from paper_2310_03567_b200.render import Camera, rasterize

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 25
    bs = gen_batches("surface", n)
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in bs]
    cam = Camera((0.5, 0.5, -1.5), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=100.0, width=1024, height=768)
    tree, state = new_tree(0, 16 << 30)
    for i in range(n):
        t0 = time.perf_counter()
        insert_batch(tree, *dev[i], state)
        t1 = time.perf_counter()
        _, rep = rasterize(tree, cam)
        t2 = time.perf_counter()
        print(f"frame {i:3d} insert {1e3 * (t1 - t0):7.3f} ms render {1e3 * (t2 - t1):7.3f} ms "
              f"samples {rep.samples_drawn}", flush=True)
    tree.close()


if __name__ == "__main__":
    main()
