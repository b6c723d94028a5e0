"""Long single-GPU stream (config 2/3 scale): N x 1M batches into one tree,
device time per batch from the library's CUDA events; batches are generated on
the host one at a time (not timed).

    python tools/long_stream.py --config terrain --batches 1000 --arena-gib 64
    python tools/long_stream.py --config mesh --batches 1000 --frames   # config 3: insert + render per frame

--frames: after every insert the bench camera is rendered (selection + splat
into a device framebuffer, lod_render) and each frame's wall time (insert +
render, the render's sync settles the insert) is reported as well.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from bench import CONFIGS, new_tree
    from paper_2310_03567_b200 import insert_batch, wait_settled, synth

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="terrain")
    ap.add_argument("--batches", type=int, default=1000)
    ap.add_argument("--arena-gib", type=float, default=64)
    ap.add_argument("--window", type=int, default=100)
    ap.add_argument("--frames", action="store_true")
    a = ap.parse_args()
    kind = CONFIGS[a.config][0]
    gen = synth.GENERATORS[kind]
    scene = synth.mesh_scene() if kind == "mesh" else None
    tree, state = new_tree(0, int(a.arena_gib * (1 << 30)))
    dev_ms, out, frame_ms = [], [], []
    frame = FrameRenderer(tree) if a.frames else None
    t0 = time.time()
    for i in range(a.batches):
        x, c = gen(1_000_000, 1000 + i, scene) if scene is not None else gen(1_000_000, 1000 + i)
        xd, cd = torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()
        torch.cuda.synchronize()
        f0 = time.perf_counter()
        insert_batch(tree, xd, cd, state)
        if frame is not None:
            frame.render(int(state._bstats.num_nodes))
            frame_ms.append((time.perf_counter() - f0) * 1e3)
        b = state._bstats
        if b.device_ms_prev >= 0 and dev_ms and dev_ms[-1] < 0:  # early-returned call, timed now
            dev_ms[-1] = float(b.device_ms_prev)
        dev_ms.append(float(b.device_ms))
        if (i + 1) % a.window == 0:
            if dev_ms[-1] < 0:
                dev_ms[-1] = wait_settled(tree)
            w = dev_ms[-a.window:]
            row = dict(batches=i + 1, window_mpts_s=round(a.window * 1e3 / sum(w), 1),
                       window_p50_ms=round(float(np.median(w)), 3), window_max_ms=round(max(w), 3),
                       nodes=int(state._bstats.num_nodes), arena_gb=round(state._bstats.arena_offset / 1e9, 2),
                       wall_s=round(time.time() - t0, 1))
            if frame_ms:
                fw = frame_ms[-a.window:]
                row.update(frame_p50_ms=round(float(np.median(fw)), 3), frame_max_ms=round(max(fw), 3),
                           frame_mpts_s=round(a.window * 1e3 / sum(fw), 1), frame_samples=frame.samples)
            out.append(row)
            print(json.dumps(row), flush=True)
    total = dict(config=a.config, batches=a.batches, points=a.batches * 1_000_000,
                 device_mpts_s=round(a.batches * 1e3 / sum(dev_ms), 1), nodes=int(state._bstats.num_nodes),
                 arena_gb=round(state._bstats.arena_offset / 1e9, 2), voxels=state.stats.voxels_created)
    total["chunks"] = tree.pool.allocated_total
    if frame_ms:
        total["frames"] = dict(count=len(frame_ms), mpts_s=round(len(frame_ms) * 1e3 / sum(frame_ms), 1),
                               p50_ms=round(float(np.median(frame_ms)), 3),
                               p99_ms=round(float(np.percentile(frame_ms, 99)), 3), max_ms=round(max(frame_ms), 3),
                               note="wall per frame: insert_batch (device-resident 1M batch) + lod_render of the "
                                    "bench camera into a device framebuffer (its sync settles the insert)")
    total["render"] = render_rows(tree)
    print(json.dumps(total), flush=True)


class FrameRenderer:
    """The bench camera (cli.py:325-328, threshold 128) rendered into a device
    framebuffer through lod_render, once per frame."""

    def __init__(self, tree):
        import torch

        from paper_2310_03567_b200.render import Camera, frustum_planes

        self.tree = tree
        cam = Camera((0.5, 0.5, -1.5), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=100.0, width=1024, height=768)
        self.cam = cam
        self.planes = np.ascontiguousarray(frustum_planes(cam), np.float64)
        self.cpk = np.ascontiguousarray(cam.packed(), np.float64)
        self.fb = torch.empty(cam.width * cam.height, dtype=torch.int64, device="cuda")
        self.samples = 0

    def render(self, num_nodes: int) -> None:
        import ctypes

        from paper_2310_03567_b200 import _lib

        sel = np.empty(max(num_nodes, 1), np.int32)  # the insert's final node count (no extra sync)
        n, drawn = ctypes.c_int64(0), ctypes.c_int64(0)
        _lib.check(self.tree._L.lod_render(self.tree.handle, _lib.ptr(self.planes), _lib.ptr(self.cpk), 128.0,
                                           _lib.ptr(self.fb), self.cam.width, self.cam.height,
                                           _lib.LOD_FLAG_DEVICE_FB | _lib.LOD_FLAG_FB_CLEAR, _lib.ptr(sel), len(sel),
                                           ctypes.byref(n), ctypes.byref(drawn)), "render")
        self.samples = int(drawn.value)


def render_rows(tree) -> dict:
    """render.rasterize's device path (selection + work-list splat, device
    framebuffer) on the settled tree, best of 5 wall: the bench overview camera
    (cli.py:325-328) and a close-up, both at threshold 128 -- next to the CPU
    reference's 12 + 66 ms (overview, 2.4M samples) and 62 + 257 ms (close-up,
    6.6M samples) on a 10M-point terrain tree."""
    import ctypes

    import torch

    from paper_2310_03567_b200 import _lib
    from paper_2310_03567_b200.render import Camera, frustum_planes

    out = {}
    for name, cam in (("overview_1024x768", Camera((0.5, 0.5, -1.5), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05,
                                                     far=100.0, width=1024, height=768)),
                      ("closeup_1920x1080", Camera((0.45, 0.2, 0.85), (0.5, 0.5, 0.45), fov_deg=60.0, near=0.01,
                                                     far=100.0, width=1920, height=1080))):
        planes = np.ascontiguousarray(frustum_planes(cam), np.float64)
        cpk = np.ascontiguousarray(cam.packed(), np.float64)
        fb = torch.empty(cam.width * cam.height, dtype=torch.int64, device="cuda")
        sel = np.empty(tree.num_nodes, np.int32)
        n, drawn = ctypes.c_int64(0), ctypes.c_int64(0)
        best = 1e9
        for _ in range(6):
            fb.fill_(-1)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _lib.check(tree._L.lod_render(tree.handle, _lib.ptr(planes), _lib.ptr(cpk), 128.0, _lib.ptr(fb), cam.width,
                                          cam.height, _lib.LOD_FLAG_DEVICE_FB, _lib.ptr(sel), len(sel),
                                          ctypes.byref(n), ctypes.byref(drawn)), "render")
            best = min(best, time.perf_counter() - t0)
        out[name] = dict(ms=round(best * 1e3, 3), nodes=int(n.value), samples=int(drawn.value),
                         msamples_per_s=round(drawn.value / best / 1e6, 1))
    return out


if __name__ == "__main__":
    main()
