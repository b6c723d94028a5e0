"""Insert W warm-up terrain batches, then one batch inside cudaProfilerStart/Stop.

    ncu --profile-from-start off --set full -o gpurun_out/prof python tools/profile_run.py --warmup 10
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import PARAMS, gen_batches, new_tree
    from paper_2310_03567_b200 import insert_batch

    ap = argparse.ArgumentParser()
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="surface")
    ap.add_argument("--profiled", type=int, default=1)
    ap.add_argument("--arena-gib", type=float, default=8.0)
    a = ap.parse_args()
    batches = gen_batches(a.config, a.warmup + a.profiled)  # bench.py's stream: seeds 1000+i
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in batches]
    tree, state = new_tree(0, int(a.arena_gib * (1 << 30)))
    for i in range(a.warmup):
        insert_batch(tree, *dev[i], state)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for i in range(a.warmup, a.warmup + a.profiled):
        insert_batch(tree, *dev[i], state)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled batches:", a.profiled, "nodes", tree.num_nodes, PARAMS)


if __name__ == "__main__":
    main()
