"""Build the bench's terrain tree (W batches, bench.py's stream) and render the
bench camera once inside cudaProfilerStart/Stop (device framebuffer):

    ncu --profile-from-start off --set full -o gpurun_out/render python tools/render_profile.py --warmup 25
"""
import argparse
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import gen_batches, new_tree
    from paper_2310_03567_b200 import _lib, insert_batch
    from paper_2310_03567_b200.render import Camera, frustum_planes

    ap = argparse.ArgumentParser()
    ap.add_argument("--warmup", type=int, default=25)
    ap.add_argument("--config", default="surface")
    a = ap.parse_args()
    tree, state = new_tree(0, 8 << 30)
    for x, c in gen_batches(a.config, a.warmup):
        insert_batch(tree, x, c, state)
    cam = Camera((0.5, 0.5, -1.5), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=100.0, width=1024, height=768)
    planes = np.ascontiguousarray(frustum_planes(cam), np.float64)
    cpk = np.ascontiguousarray(cam.packed(), np.float64)
    fb = torch.full((cam.width * cam.height,), -1, dtype=torch.int64, device="cuda:0")
    sel = np.empty(tree.num_nodes, np.int32)
    n, drawn = ctypes.c_int64(0), ctypes.c_int64(0)

    def render():
        _lib.check(tree._L.lod_render(tree.handle, _lib.ptr(planes), _lib.ptr(cpk), 128.0, _lib.ptr(fb), cam.width,
                                      cam.height, _lib.LOD_FLAG_DEVICE_FB, _lib.ptr(sel), len(sel), ctypes.byref(n),
                                      ctypes.byref(drawn)), "render")

    render()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    render()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"render: {n.value} nodes, {drawn.value} samples, tree {tree.num_nodes} nodes")


if __name__ == "__main__":
    main()
