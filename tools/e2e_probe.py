"""Where the end-to-end time goes: device-resident inserts vs pinned host inserts
(serial H2D) vs the frame loop with the ingest feed (staged H2D)."""
import collections
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import gen_batches, new_tree
    from paper_2310_03567_b200 import insert_batch, run_frame_updates

    nb = 60
    batches = gen_batches("surface", nb)
    dev = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in batches]
    pin = []
    for x, c in batches:
        px = torch.from_numpy(x).pin_memory()
        pc = torch.from_numpy(c.view(np.int32)).pin_memory()
        pin.append((px.numpy(), pc.numpy().view(np.uint32)))

    def run(kind, budget=10.0):
        tree, state = new_tree(0, 8 << 30)
        for i in range(5):
            insert_batch(tree, *dev[i], state)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if kind == "device":
            for i in range(5, nb):
                insert_batch(tree, *dev[i], state)
        elif kind == "pinned":
            for i in range(5, nb):
                insert_batch(tree, *pin[i], state)
        else:
            state.clock.budget_ms = budget
            q = collections.deque(pin[5:])
            while q:
                run_frame_updates(tree, q, state)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        tree.close()
        return (nb - 5) / dt / 1e3 * 1e3, state.stats.frames

    for kind, b in (("device", 0), ("pinned", 0), ("frames", 10.0), ("frames", 1e9)):
        v, f = run(kind, b)
        print(f"{kind:8s} budget {b:8.0f} ms: {v:8.1f} Mpts/s wall  frames {f}")


if __name__ == "__main__":
    main()


def h2d_bandwidth():
    import torch

    x = torch.empty(16 << 20, dtype=torch.uint8).pin_memory()
    y = torch.empty(16 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        y.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        y.copy_(x, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"pinned H2D: {20 * 16 * 2**20 / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")


h2d_bandwidth()
