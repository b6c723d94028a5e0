"""Benchmark: incremental LOD insertion throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config terrain] [--impl ours|reference]

A *step* is one ``insert_batch`` of one synthetic 1M-point batch (the paper's
update-only unit).  Default workload = BASELINE config 2: a
gen_surface terrain streamed in 1M-point batches into one tree (unit root,
T=50,000, C=1,000, G=128, max depth 20); W + K batches = the stream prefix.

* ``value``: Mpts/s = K * 1M / (device time of the K timed steps), inputs
  already resident in HBM (CUDA tensors), timed with CUDA events bracketed by
  barrier + synchronize, max over ranks.
* ``e2e``: the same metric through the public API a user streams with: the
  reference's frame loop (``run_frame_updates`` over a queue of host batches
  in pinned memory, 10 ms budget, cli._build) -- every batch's H2D copy (the
  ingest feed stages batch k+1 while batch k updates) + update + control-block
  read-backs inside the timed region.
* ``roofline``: the dominant phase of the update (per-phase CUDA events on the
  tree stream in a profiled replay), algorithmic bytes / time vs measured HBM.
* ``cpu_baseline``: the reference's own implementation (``lodstream``,
  numba, single-threaded by design) on a bounded prefix of the same stream --
  the unmodified package staged by ``__graft_entry__.build()`` under
  tests/ref_suite/_ref, which travels with the working tree; where it is not
  staged, the C oracle (a 1-thread port of the same sequential path, slower
  than numba on terrain: tools/ref_vs_port.py).
* ``--impl reference``: the same implementation on the same steps.

Multi-GPU (torchrun, N > 1): points are partitioned by octant prefix across
ranks (paper_2310_03567_b200/partition.py); each rank runs its own subtree
stream; ``value`` = all ranks' points / max-over-ranks time ("scaling": "weak").
"""
from __future__ import annotations

import argparse
import collections
import dataclasses
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "M points/s inserted into LOD (ms per 1M-pt batch) at 1/2/4/8 B200 vs CPU ref"
BATCH = 1_000_000
PARAMS = dict(grid_res=128, leaf_threshold=50_000, max_depth=20, chunk_capacity=1000)
CONFIGS = {
    # name: (generator, description)
    "terrain": ("surface", "config 2: 100M-point 2.5D LIDAR terrain (height field + noise), 1M batches"),
    "uniform": ("uniform", "config 1 shape: uniform points in the unit cube, 1M batches"),
    "skew": ("skew", "config 4: density skew, 90% of points in a 1e-4-volume cube, 1M batches"),
    "mesh": ("mesh", "config 3: photogrammetry-style surface samples on random triangles, 1M batches"),
}


def rank_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _gen_one(args):
    from paper_2310_03567_b200 import synth

    kind, seed = args
    if kind == "mesh":
        return synth.gen_mesh(BATCH, seed, synth.mesh_scene())
    return synth.GENERATORS[kind](BATCH, seed)


def gen_batches(kind: str, count: int, seed0: int = 1000):
    """Batches seed0 .. seed0+count-1 of the stream (deterministic per seed);
    generated on a process pool when there are many (the full 100-batch
    stream in a few seconds)."""
    jobs = [(kind, seed0 + i) for i in range(count)]
    if count <= 8:
        return [_gen_one(j) for j in jobs]
    import concurrent.futures as cf
    import multiprocessing as mp

    workers = max(1, min(16, (os.cpu_count() or 2) - 1))
    with cf.ProcessPoolExecutor(workers, mp_context=mp.get_context("fork")) as ex:
        return list(ex.map(_gen_one, jobs, chunksize=2))


FULL_STREAM = 100  # BASELINE config 2: 100 x 1M-point batches
BATCH_SIM = 1 << 20  # SIM feed batch (16 MiB, O_DIRECT-aligned)


def bench_config(args) -> dict:
    """The `config` both arms print (identical dicts: the driver compares them)."""
    w, k = args.warmup, args.steps
    return {"workload": f"{CONFIGS[args.config][1]}; timed: stream batches {w}..{w + k - 1} ({k} x 1M points) "
                        f"after {w} untimed warm-up batches (the tree holds {w + k}M points at the end)",
            "batch_points": BATCH, "tree": PARAMS, "timed_batches": [w, w + k],
            "l2": "inputs larger than L2: every step inserts a distinct 16 MB batch"}


def morton_sorted(xyz, rgba, bits: int = 10):
    """z-order a batch (unit cube) -- for the --presort locality experiment."""
    q = np.clip((xyz * (1 << bits)).astype(np.int64), 0, (1 << bits) - 1)
    key = np.zeros(len(q), np.int64)
    for b in range(bits):
        for a in range(3):
            key |= ((q[:, a] >> b) & 1) << (3 * b + a)
    o = np.argsort(key, kind="stable")
    return np.ascontiguousarray(xyz[o]), np.ascontiguousarray(rgba[o])


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.QUERY}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak_hbm() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def new_tree(device: int, arena_bytes: int):
    from paper_2310_03567_b200 import Arena, ChunkPool, CubeBounds, Octree, UpdateConfig, UpdateState

    arena = Arena(arena_bytes)
    tree = Octree(CubeBounds((0.0, 0.0, 0.0), 1.0), arena, ChunkPool(arena, PARAMS["chunk_capacity"]),
                  grid_res=PARAMS["grid_res"], leaf_threshold=PARAMS["leaf_threshold"],
                  max_depth=PARAMS["max_depth"], device=device)
    state = UpdateState(UpdateConfig(backlog_capacity=64_000_000, spill_capacity=100_000_000))
    return tree, state


def run_multi(args, rank, world, local_rank):
    """N > 1: every step is a global batch of N x 1M points arriving striped
    (1M per rank); points are routed to the owners of their octant prefixes
    by the fused bucket scatter into the owners' peer-memory windows
    (multigpu.PeerRouter) and inserted into the owner's tree
    (paper_2310_03567_b200/multigpu.py).  Warm-up batches run the single-tree
    protocol on rank 0 until the top is inner, then rank 0's tree is
    broadcast.  Weak scaling: per-GPU input is fixed at 1M points per step."""
    import torch
    import torch.distributed as dist

    from paper_2310_03567_b200 import multigpu, partition

    # one process per GPU over NCCL; LOD_DIST_BACKEND=gloo (with ranks sharing
    # GPUs, local_rank modulo the visible devices) exercises this whole path on
    # a single-GPU box
    backend = os.environ.get("LOD_DIST_BACKEND", "nccl")
    local_rank = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local_rank)
    if backend == "nccl":
        os.environ.setdefault("NCCL_DEBUG", "WARN")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        dist.init_process_group(backend)
    # communicator check, logged per rank: every rank contributes its rank
    probe = torch.tensor([rank], dtype=torch.int64, device="cuda" if backend == "nccl" else "cpu")
    dist.all_reduce(probe)
    print(f"[bench] comm ready: backend={backend} rank={rank} nranks={dist.get_world_size()} "
          f"device=cuda:{local_rank} sum_of_ranks={int(probe.item())} (expected {world * (world - 1) // 2})",
          file=sys.stderr, flush=True)
    kind = CONFIGS[args.config][0]
    sample = [gen_stripe(kind, s, 0) for s in range(2)]
    plan = partition.plan_owners(sample, world)  # deterministic: same on every rank
    tree, state = new_tree(local_rank, int(args.arena_gib * (1 << 30)))
    ins = multigpu.PartitionedInserter(tree, state, plan, rank, world)
    step = 0
    while step < args.warmup or not ins.partitioned:
        x, c = gen_stripe(kind, step, rank)
        ins.insert(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda())
        step += 1
    stripes = [gen_stripe(kind, step + k, rank) for k in range(args.steps)]
    dev_b = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in stripes]
    pin_b = [(torch.from_numpy(x).pin_memory(), torch.from_numpy(c.view(np.int32)).pin_memory())
             for x, c in (gen_stripe(kind, step + args.steps + k, rank) for k in range(args.steps))]
    torch.cuda.synchronize()

    def timed(inputs, host):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        launches = h2d = 0
        d2h0 = state.stats.d2h_bytes
        e0.record()
        for x, c in inputs:
            if host:  # the stripe arrives in host memory: H2D inside the timed region
                x, c = x.cuda(non_blocking=True), c.cuda(non_blocking=True)
                h2d += 16 * c.numel()
            ins.insert(x, c)
            launches += int(state._bstats.launches)
        ins.flush()  # the last batch's replicated-top merge is inside the timed region
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        timed.d2h = state.stats.d2h_bytes - d2h0
        return e0.elapsed_time(e1), launches, h2d

    with ClockSampler(local_rank) as clocks:
        ms, launches, _ = timed(dev_b, False)
    # e2e: the next stripes of the stream from pinned host memory
    ms_e2e, _, h2d = timed(pin_b, True)
    v = torch.tensor([ms, float(sum(len(c) for _, c in stripes)), ms_e2e], device="cuda", dtype=torch.float64)
    allv = [torch.zeros_like(v) for _ in range(world)]
    dist.all_gather(allv, v)
    t_max = max(float(a[0]) for a in allv)
    t_e2e = max(float(a[2]) for a in allv)
    pts = sum(float(a[1]) for a in allv)
    line = None
    if rank == 0:
        value = pts / (t_max * 1e-3) / 1e6
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "Mpts/s", "n_gpus": world, "steps": args.steps,
            "warmup": step, "ms_per_step": round(t_max / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32", "data": "synthetic",
            "config": bench_config(args),
            "notes": {"global_batch": f"{world} x 1M points striped over ranks per step (weak scaling)",
                       "parallelism": f"octant-prefix partition depth {plan.depth} x{world}, "
                                      + (f"{backend.upper()} all-to-all routing (peer windows unavailable: "
                                         f"{ins.no_peers})" if ins.no_peers else
                                         f"peer-memory routing (bucket scatter into CUDA IPC windows, "
                                         f"sequence flags in the windows: no per-batch host barrier; "
                                         f"replicated-top voxels logged on the device, merged "
                                         f"{ins.flushes}x), {backend.upper()} for the warm-up, hand-off and "
                                         f"the top-node merges"),
                       "imbalance_max_over_mean": round(partition.imbalance(plan), 3)},
            "e2e": {"value": round(pts / (t_e2e * 1e-3) / 1e6, 2), "unit": "Mpts/s",
                    "h2d_bytes_per_step": h2d // max(args.steps, 1),
                    "d2h_bytes_per_step": timed.d2h // max(args.steps, 1),
                    "note": "the next K stripes of the stream, each H2D from pinned host memory + routing + "
                            "insert, max over ranks"},
            "gpu_launches": launches, "clocks": clocks.summary(),
        }
    ins.close()
    dist.destroy_process_group()
    return line


def gen_stripe(kind: str, step: int, rank: int):
    """Rank `rank`'s 1M-point stripe of global batch `step` (seeded per stripe)."""
    from paper_2310_03567_b200 import synth

    seed = 1000 + step * 64 + rank
    if kind == "mesh":
        return synth.gen_mesh(BATCH, seed, synth.mesh_scene())
    return synth.GENERATORS[kind](BATCH, seed)


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2310_03567_b200 import insert_batch, run_frame_updates, wait_settled

    if world > 1:
        return run_multi(args, rank, world, local_rank)
    torch.cuda.set_device(local_rank)
    dev = local_rank
    dist = None
    kind = CONFIGS[args.config][0]
    total = args.warmup + args.steps
    n_gen = max(total, FULL_STREAM) if not args.no_rows else total
    batches = gen_batches(kind, n_gen)
    full_stream = batches if len(batches) >= FULL_STREAM else None
    batches = batches[:total]
    if args.presort:  # experiment only: z-ordered input batches (changes the workload)
        batches = [morton_sorted(x, c) for x, c in batches]
    n_points = [len(c) for _, c in batches]
    arena_bytes = int(args.arena_gib * (1 << 30))
    # device-resident inputs (value) and pinned host inputs (e2e)
    dev_b = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in batches]
    pin_b = []
    for x, c in batches:
        px = torch.from_numpy(x).pin_memory()
        pc = torch.from_numpy(c.view(np.int32)).pin_memory()
        pin_b.append((px.numpy(), pc.numpy().view(np.uint32)))
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def timed_stream(inputs, profile=False, frames=False, keep=None):
        """Device-resident batches one insert_batch per step, or (frames=True)
        host batches through the frame loop a user runs (cli._build:
        run_frame_updates over a queue, 10 ms budget, ingest feed overlapped)."""
        tree, state = new_tree(dev, arena_bytes)
        per, launches, phases = [], 0, []
        h2d = d2h = 0
        if frames:  # the warm-up goes through the same frame loop (ingest feed, copy stream, staging slots)
            q = collections.deque(inputs[:args.warmup])
            while q:
                run_frame_updates(tree, q, state)
            wait_settled(tree, state)
        else:
            for i in range(args.warmup):
                insert_batch(tree, *inputs[i], state)
        barrier()
        s0 = dataclasses.replace(state.stats)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if frames:
            q = collections.deque(inputs[args.warmup:total])
            while q:
                run_frame_updates(tree, q, state)
        else:
            for i in range(args.warmup, total):
                insert_batch(tree, *inputs[i], state, profile=profile)
                b = state._bstats
                # a call that returned before its tail ran (-1) is timed by the next one
                if b.device_ms_prev >= 0 and per and per[-1] < 0:
                    per[-1] = float(b.device_ms_prev)
                per.append(float(b.device_ms))
                if profile:
                    ph = dict(state.last["phase_ms"])
                    ph["_counts"] = (int(b.n_batch), int(b.n_spill), int(b.n_voxels))
                    phases.append(ph)
        last = wait_settled(tree, state)  # the last update's tail is inside the timed region
        if per and per[-1] < 0:
            per[-1] = last
        e1.record()
        barrier()
        st = state.stats
        launches, h2d, d2h = st.launches - s0.launches, st.h2d_bytes - s0.h2d_bytes, st.d2h_bytes - s0.d2h_bytes
        ms = e0.elapsed_time(e1)
        info = dict(nodes=tree.num_nodes, points=tree.total_points() if args.steps <= 200 else None,
                    voxels_created=state.stats.voxels_created, arena=tree.arena.offset)
        if keep is not None:
            keep.extend([tree, state])
        else:
            tree.close()
        return ms, per, launches, phases, info, (h2d, d2h)

    with ClockSampler(dev) as clocks:
        ms, per, launches, _, info, _ = timed_stream(dev_b)
    ms_e2e, per_e2e, _, _, _, (h2d, d2h) = timed_stream(pin_b, frames=True)
    # profiled replay: per-phase CUDA events on the tree stream + per-batch B_alg inputs
    kept = []
    _, per_prof, _, phases, _, _ = timed_stream(dev_b, profile=True, keep=kept)
    rows = secondary_rows(args, kept[0], kept[1], dev_b, dev) if not args.no_rows else None
    kept[0].close()
    if rows is not None and full_stream is not None:
        rows["full_stream"] = full_stream_row(args, full_stream[:FULL_STREAM], dev, arena_bytes)
        rows["disk_ingest"] = disk_ingest_row(args, full_stream[:FULL_STREAM], dev, arena_bytes)

    timed_pts = sum(n_points[args.warmup:])
    t_max = ms
    t_e2e = ms_e2e
    if dist is not None:
        v = torch.tensor([ms, ms_e2e, float(timed_pts)], device="cuda", dtype=torch.float64)
        allv = [torch.zeros_like(v) for _ in range(world)]
        dist.all_gather(allv, v)
        t_max = max(float(a[0]) for a in allv)
        t_e2e = max(float(a[1]) for a in allv)
        timed_pts = sum(float(a[2]) for a in allv)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None

    value = timed_pts / (t_max * 1e-3) / 1e6
    e2e = timed_pts / (t_e2e * 1e-3) / 1e6
    # roofline of the dominant phase
    peak, peak_kind = measured_peak_hbm()
    roof, phase_summary = roofline_from_phases(phases, peak)
    roof["peak"] = peak
    roof["peak_source"] = peak_kind
    roof["frac"] = round(roof["achieved"] / peak, 4) if roof.get("achieved") else None
    roof["traffic"], roof["traffic_source"] = load_traffic(roof.get("kernel"), args)
    cpu = cpu_baseline(args, kind) if not args.no_cpu else None
    srt = sorted(per)
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "Mpts/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_max / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32", "data": "synthetic",
        "config": bench_config(args),
        "notes": {"parallelism": "single tree", "resident_batches_mb": total * 16, "final_nodes": info["nodes"],
                  "voxels_created": info["voxels_created"]},
        "batch_ms": {"avg": round(statistics.mean(per), 4), "p50": round(srt[len(srt) // 2], 4),
                     "p99": round(srt[min(len(srt) - 1, int(0.99 * len(srt)))], 4), "max": round(srt[-1], 4)},
        "e2e": {"value": round(e2e, 2), "unit": "Mpts/s", "h2d_bytes_per_step": h2d // max(args.steps, 1),
                "d2h_bytes_per_step": d2h // max(args.steps, 1)},
        "gpu_launches": launches,
        "roofline": roof,
        "phase_ms": phase_summary,
        "cpu_baseline": cpu,
        "clocks": clocks.summary(),
        "rows": rows,
    }
    if dist is not None:
        dist.destroy_process_group()
    return line


def full_stream_row(args, batches, dev, arena_bytes) -> dict:
    """The whole 100-batch config stream into a fresh tree (BASELINE config
    2's 100M points for the terrain config), device-resident, each batch's
    device time from its own CUDA events: avg / p50 / p99 / max ms per 1M
    batch and M points/s over the whole stream."""
    import torch

    from paper_2310_03567_b200 import insert_batch, wait_settled

    dev_b = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in batches]
    tree, state = new_tree(dev, arena_bytes)
    torch.cuda.synchronize()
    per = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for x, c in dev_b:
        insert_batch(tree, x, c, state)
        b = state._bstats
        if b.device_ms_prev >= 0 and per and per[-1] < 0:
            per[-1] = float(b.device_ms_prev)
        per.append(float(b.device_ms))
    last = wait_settled(tree)
    if per[-1] < 0:
        per[-1] = last
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    srt = sorted(per)
    pts = sum(int(c.numel()) for _, c in dev_b)
    out = {"batches": len(dev_b), "points": pts, "mpts_per_s": round(pts / (ms * 1e-3) / 1e6, 1),
           "stream_ms": round(ms, 3),
           "batch_ms": {"avg": round(statistics.mean(per), 4), "p50": round(srt[len(srt) // 2], 4),
                        "p99": round(srt[min(len(srt) - 1, int(0.99 * len(srt)))], 4), "max": round(srt[-1], 4)},
           "worst_batch": int(np.argmax(per)), "batches_over_1ms": int(sum(p > 1.0 for p in per)),
           "final_nodes": tree.num_nodes, "voxels_created": state.stats.voxels_created,
           "note": "per-batch device time from CUDA events on the tree stream (inputs resident in HBM); "
                   "stream_ms = events around the whole stream"}
    tree.close()
    return out


def disk_ingest_row(args, batches, dev, arena_bytes) -> dict:
    """The paper's system figure (disk -> insert -> render: 580
    M points/s, ~9.3 GB/s on an RTX 4090 + PCIe 5 SSD): the whole stream as a
    SIM file (1.6 GB), read by the native O_DIRECT reader thread into pinned
    slots, DMA'd and inserted, the bench camera rendered (device selection +
    splat, 1024 x 768) after every batch.  The file is written, fsync'd and
    evicted from the page cache (POSIX_FADV_DONTNEED) first; O_DIRECT reads
    bypass the cache anyway."""
    from paper_2310_03567_b200 import ingest
    from paper_2310_03567_b200.render import Camera

    path = os.path.join(args.sim_dir, f"lod_bench_{os.getpid()}.sim")
    try:
        with open(path, "wb") as f:
            for x, c in batches:
                rec = np.empty((len(c), 4), np.uint32)
                rec[:, :3] = x.view(np.uint32)
                rec[:, 3] = c
                rec.tofile(f)
            f.flush()
            os.fsync(f.fileno())
            os.posix_fadvise(f.fileno(), 0, 0, os.POSIX_FADV_DONTNEED)
        cam = Camera((0.5, 0.5, -1.5), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=100.0, width=1024, height=768)
        tree, state = new_tree(dev, arena_bytes)
        out = ingest.stream_sim(tree, path, state, batch_size=BATCH_SIM, camera=cam, render_every=1)
        tree.close()
        st = os.statvfs(args.sim_dir)
        out.update({"file": path, "page_cache": "evicted (POSIX_FADV_DONTNEED) before the run",
                    "fs_free_gb": round(st.f_bavail * st.f_frsize / 1e9, 1),
                    "note": "wall clock from opening the file to the settled tree; every batch rendered"})
        return {k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}
    except OSError as e:
        return {"unavailable": f"{type(e).__name__}: {e}"}
    finally:
        if os.path.exists(path):
            os.remove(path)


def secondary_rows(args, tree, state, dev_b, dev) -> dict:
    """The SURVEY 8(f) rows on the settled stream tree (device timings, wall
    clock around synchronous calls, best of a few):

    * render: ``rasterize`` = device selection + splat (lod_render, device
      framebuffer) at the bench camera of cli.py:325-328 (1024 x 768), and
      ``select_visible`` alone;
    * frame: config 3's loop, insert + render per frame (public API);
    * delta: insert_batch(collect_delta=True) vs plain on further batches;
    * morton: device Morton sort of 16M resident points (lod_morton_sort).
    """
    import ctypes

    import torch

    from paper_2310_03567_b200 import _lib, insert_batch, synth, wait_settled
    from paper_2310_03567_b200.render import Camera, frustum_planes, select_visible

    out = {}
    cam = Camera((0.5, 0.5, -1.5), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=100.0, width=1024, height=768)
    planes = np.ascontiguousarray(frustum_planes(cam), np.float64)
    cpk = np.ascontiguousarray(cam.packed(), np.float64)
    fb = torch.full((cam.width * cam.height,), -1, dtype=torch.int64, device=f"cuda:{dev}")
    sel = np.empty(tree.num_nodes, np.int32)
    n, drawn = ctypes.c_int64(0), ctypes.c_int64(0)

    def render_once():
        fb.fill_(-1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(tree._L.lod_render(tree.handle, _lib.ptr(planes), _lib.ptr(cpk), 128.0, _lib.ptr(fb), cam.width,
                                      cam.height, _lib.LOD_FLAG_DEVICE_FB, _lib.ptr(sel), len(sel), ctypes.byref(n),
                                      ctypes.byref(drawn)), "render")
        return time.perf_counter() - t0

    render_once()
    t_r = min(render_once() for _ in range(10))
    t0 = time.perf_counter()
    for _ in range(10):
        select_visible(tree, cam, 128.0)
    t_s = (time.perf_counter() - t0) / 10
    out["render"] = {"camera": "cli.py:325-328 bench camera, 1024x768, threshold 128", "ms": round(t_r * 1e3, 3),
                     "select_ms": round(t_s * 1e3, 3), "nodes_selected": int(n.value),
                     "samples_drawn": int(drawn.value),
                     "msamples_per_s": round(drawn.value / t_r / 1e6, 1)}
    # config 3's frame loop: insert one 1M batch + render the bench camera per
    # frame through the public API (render.rasterize: device selection +
    # splat, host framebuffer), on a fresh tree over the same stream
    from paper_2310_03567_b200.render import rasterize

    ftree, fstate = new_tree(dev, int(args.arena_gib * (1 << 30)))
    for i in range(args.warmup):
        insert_batch(ftree, *dev_b[i], fstate)
    # two live targets, as in the loop (a frame's framebuffer is still held
    # when the next one renders): the pinned-buffer pool holds both afterwards
    w1, w2 = rasterize(ftree, cam), rasterize(ftree, cam)
    del w1, w2
    torch.cuda.synchronize()
    fr, rr, pts = [], [], 0
    for i in range(args.warmup, len(dev_b)):
        t0 = time.perf_counter()
        insert_batch(ftree, *dev_b[i], fstate)
        t1 = time.perf_counter()
        _, rep = rasterize(ftree, cam)
        t2 = time.perf_counter()
        fr.append(t2 - t0)
        rr.append(t2 - t1)
        pts += int(dev_b[i][1].numel())
    ftree.close()
    fr_s = sorted(fr)
    out["frame"] = {"note": "per frame: insert_batch (device-resident 1M batch) + rasterize (bench camera, "
                            "1024x768, threshold 128, host framebuffer); wall clock, the render's sync "
                            "settles the insert",
                    "frames": len(fr), "mpts_per_s": round(pts / sum(fr) / 1e6, 1),
                    "ms_per_frame": {"avg": round(statistics.mean(fr) * 1e3, 3),
                                     "p50": round(fr_s[len(fr_s) // 2] * 1e3, 3),
                                     "p99": round(fr_s[min(len(fr_s) - 1, int(0.99 * len(fr_s)))] * 1e3, 3)},
                    "render_ms_avg": round(statistics.mean(rr) * 1e3, 3),
                    "samples_drawn_last": int(rep.samples_drawn)}
    # delta capture overhead on further batches
    extra = [synth.gen_surface(BATCH, 9000 + i) for i in range(6)]
    ex = [(torch.from_numpy(x).cuda(), torch.from_numpy(c.view(np.int32)).cuda()) for x, c in extra]
    tp, td = [], []
    for i, (x, c) in enumerate(ex):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        insert_batch(tree, x, c, state, collect_delta=bool(i % 2))
        wait_settled(tree, state)  # both arms to the settled tree
        (td if i % 2 else tp).append(time.perf_counter() - t0)
    out["delta"] = {"plain_ms": round(min(tp) * 1e3, 3), "collect_delta_ms": round(min(td) * 1e3, 3),
                    "note": "wall ms per 1M-point insert incl. delta assembly + D2H, same tree, alternating"}
    # tiny host batches (acceptance C1's regime, test_acceptance.py:81-101:
    # G=16, T=100, C=1000, depth 12): wall us per insert_batch call through
    # the facade, the one-kernel small path for n <= 256
    out["small_batches"] = small_batch_row()
    # Morton sort of 16M device-resident points
    mx = torch.cat([b[0] for b in dev_b[:16]])
    mc = torch.cat([b[1] for b in dev_b[:16]])
    mo_x, mo_c = torch.empty_like(mx), torch.empty_like(mc)
    bmin = np.zeros(3, np.float64)
    L = _lib.load()

    def morton_once():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        _lib.check(L.lod_morton_sort(dev, _lib.ptr(bmin), float(1 << 21), 21, _lib.ptr(mx), _lib.ptr(mc),
                                     mc.numel(), _lib.ptr(mo_x), _lib.ptr(mo_c), None, _lib.LOD_FLAG_DEVICE_INPUT),
                   "morton")
        return time.perf_counter() - t0

    morton_once()
    t_m = min(morton_once() for _ in range(5))
    out["morton_sort"] = {"points": int(mc.numel()), "ms": round(t_m * 1e3, 3),
                          "mpts_per_s": round(mc.numel() / t_m / 1e6, 1)}
    return out


def small_batch_row() -> dict:
    from paper_2310_03567_b200 import Arena, ChunkPool, CubeBounds, Octree, UpdateConfig, UpdateState, insert_batch

    rows = {}
    for bs, total in ((1, 20_000), (7, 70_000), (100, 200_000), (1000, 200_000)):
        rng = np.random.default_rng(bs)
        xyz = rng.random((total, 3)).astype(np.float32)
        rgba = rng.integers(0, 1 << 32, total, dtype=np.uint64).astype(np.uint32)
        arena = Arena(1 << 30)
        tree = Octree(CubeBounds((0.0, 0.0, 0.0), 1.0), arena, ChunkPool(arena, 1000), grid_res=16,
                      leaf_threshold=100, max_depth=12)
        state = UpdateState(UpdateConfig())
        parts = [(xyz[i:i + bs], rgba[i:i + bs]) for i in range(0, total, bs)]
        for x, c in parts[:20]:
            insert_batch(tree, x, c, state)
        _ = state.stats
        t0 = time.perf_counter()
        for x, c in parts[20:]:
            insert_batch(tree, x, c, state)
        _ = state.stats  # settled: the queued cycles' device work is inside the time
        dt = time.perf_counter() - t0
        calls = len(parts) - 20
        rows[f"n={bs}"] = {"us_per_call": round(dt / calls * 1e6, 2), "calls": calls,
                           "path": "one-kernel cycle" if bs <= 256 else "pipeline"}
        tree.close()
    rows["note"] = ("wall time per insert_batch of a host batch through the facade, settled at the end; "
                    "acceptance C1 makes 1.52M such calls of 1 or 7 points within 60 s")
    return rows


def phase_bytes(phase: str, n_b: int, n_s: int, n_v: int) -> int | None:
    """Algorithmic HBM bytes of one batch's phase.

    count:   every point's 16-byte record read once + its 4-byte leaf id written
    resolve: per new voxel: claim slot read+clear (32), grid word RMW (8), win (8), mask RMW (16)
    sort:    radix pass 1 (key read, key + item write: 12 per item), pass 2 (key + item read: 8)
             + the store its last pass performs (source records read 16 n_all, written 16 per item)
    total:   B_alg = 32 n_b + 32 n_s + 16 n_v
    """
    n_all = n_b + n_s
    n_items = n_all + n_v
    return {
        "count": 20 * n_all,
        "resolve": 64 * n_v,
        "sort": 20 * n_items + 16 * n_all + 16 * n_items,
        "total": 32 * n_b + 32 * n_s + 16 * n_v,
    }.get(phase)


def roofline_from_phases(phases: list[dict], peak: float) -> tuple[dict, dict]:
    """Dominant kernel phase: algorithmic bytes / its CUDA-event time (profiled replay)."""
    if not phases:
        return {"bound": "hbm", "achieved": None, "unit": "GB/s", "traffic": None}, {}
    names = [k for k in phases[0] if not k.startswith("_") and k not in ("h2d", "total")]
    tot = {k: sum(p[k] for p in phases) for k in names + ["total"]}
    med = {k: round(statistics.median(p[k] for p in phases), 4) for k in names + ["total"]}
    byts = {k: sum(phase_bytes(k, *p["_counts"]) or 0 for p in phases) for k in names + ["total"]}
    dom = max((k for k in names if phase_bytes(k, 1, 1, 1) is not None), key=lambda k: tot[k])
    gbs = {k: round(byts[k] / (tot[k] * 1e-3) / 1e9, 1) for k in byts if byts[k] and tot[k] > 0}
    roof = {
        "bound": "hbm", "kernel": {"count": "k_count", "sort": "k_onesweep", "resolve": "k_resolve"}[dom],
        "achieved": gbs.get(dom), "unit": "GB/s", "traffic": None,
        "kernel_share_of_step": round(tot[dom] / tot["total"], 3) if tot["total"] else None,
        "whole_update": {"achieved": gbs.get("total"), "frac": round(gbs.get("total", 0) / peak, 4)},
        "phase_gbs": gbs,
    }
    # the count phase is bound by L2 atomics, not bytes: one 128-bit CAS install
    # per new voxel (claims are ~1.04x the new voxels), against the measured
    # random-install rate of tools/cas_bench.cu (profiles/r01_cas_roofline.txt)
    cas = cas_peak()
    if cas and tot.get("count"):
        n_v = sum(p["_counts"][2] for p in phases)
        rate = n_v / (tot["count"] * 1e-3) / 1e9
        roof["atomics"] = {"bound": "l2_atomics", "kernel": "k_count", "achieved": round(rate, 2),
                           "unit": "G installs/s", "peak": round(cas[0], 2), "frac": round(rate / cas[0], 3),
                           "peak_source": cas[1]}
    return roof, {"median_ms": med, "mean_ms": {k: round(tot[k] / len(phases), 4) for k in tot}}


def cas_peak():
    """Best measured 128-bit CAS install rate (G/s) from the committed
    microbenchmark output, or None."""
    import re

    path = os.path.join(ROOT, "profiles", "r01_cas_roofline.txt")
    try:
        best = 0.0
        for line in open(path):
            m = re.search(r"([0-9.]+)M installs\s+cas128\s+([0-9.]+) us", line)
            if m:
                best = max(best, float(m.group(1)) * 1e6 / (float(m.group(2)) * 1e-6) / 1e9)
        return (best, "tools/cas_bench.cu, profiles/r01_cas_roofline.txt") if best else None
    except OSError:
        return None


def load_traffic(kernel: str | None, args):
    """DRAM bytes per launch of the dominant kernel over THIS run's timed
    batch range, from the committed ncu capture of the same batches
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.sh); null when no
    capture covers this config and range."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            caps = json.load(f)["captures"]
    except Exception:
        return None, "no committed ncu capture"
    want = [args.warmup, args.warmup + args.steps]
    for c in caps:
        if c.get("config") == args.config and c.get("batches") == want and kernel in c.get("per_launch_bytes", {}):
            return c["per_launch_bytes"][kernel], f"ncu over the same batches: {c['command']} ({c['when']})"
    return None, f"no committed ncu capture of {args.config} batches {want[0]}..{want[1] - 1}"


REF_STAGED = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tests", "ref_suite", "_ref")


def cpu_tree(args):
    """(insert(x, c), kind) for the CPU legs: the reference package itself
    (unmodified lodstream, numba) when staged, else the C oracle port."""
    if os.path.isdir(os.path.join(REF_STAGED, "lodstream")) and not os.environ.get("LOD_BENCH_PORT"):
        try:
            if REF_STAGED not in sys.path:
                sys.path.insert(0, REF_STAGED)
            from lodstream.octree import CubeBounds as RCube, Octree as ROctree
            from lodstream.store import Arena as RArena, ChunkPool as RPool
            from lodstream.update import UpdateConfig as RConfig, UpdateState as RState
            from lodstream.update import insert_batch as r_insert

            arena = RArena(int(args.arena_gib * (1 << 30)))
            tree = ROctree(RCube((0.0, 0.0, 0.0), 1.0), arena, RPool(arena, PARAMS["chunk_capacity"]),
                           grid_res=PARAMS["grid_res"], leaf_threshold=PARAMS["leaf_threshold"],
                           max_depth=PARAMS["max_depth"])
            state = RState(RConfig(backlog_capacity=64_000_000))
            return (lambda x, c: r_insert(tree, x, c, state)), "reference"
        except ImportError:  # numba missing on this host: the port
            pass
    import oracle

    t = oracle.OracleTree(grid_res=PARAMS["grid_res"], leaf_threshold=PARAMS["leaf_threshold"],
                          max_depth=PARAMS["max_depth"], chunk_capacity=PARAMS["chunk_capacity"],
                          arena_bytes=int(args.arena_gib * (1 << 30)), backlog_capacity=64_000_000)
    return t.insert_batch, "port"


def cpu_baseline(args, kind) -> dict:
    """The reference implementation (or its port) on a bounded prefix; the
    first two batches are untimed (numba compiles its kernels on first use)."""
    n_b = args.cpu_batches
    batches = gen_batches(kind, n_b)
    insert, how = cpu_tree(args)
    for x, c in batches[:2]:
        insert(x, c)
    t0 = time.perf_counter()
    for x, c in batches[2:]:
        insert(x, c)
    dt = time.perf_counter() - t0
    return {"value": round((n_b - 2) * BATCH / dt / 1e6, 3), "unit": "Mpts/s", "cores": 1, "kind": how,
            "sample": f"batches 2..{n_b - 1} of the same stream ({n_b - 2}M points, {dt:.1f} s) after 2 untimed",
            "host_nproc": os.cpu_count()}


def run_reference(args, rank, world):
    """--impl reference: the reference implementation (lodstream itself when
    staged, else the C port; 1 thread by design) on the same steps."""
    if rank != 0:
        return None
    kind = CONFIGS[args.config][0]
    total = args.warmup + args.steps
    batches = gen_batches(kind, total)
    insert, how = cpu_tree(args)
    for i in range(args.warmup):
        insert(*batches[i])
    per = []
    for i in range(args.warmup, total):
        t0 = time.perf_counter()
        insert(*batches[i])
        per.append(time.perf_counter() - t0)
    secs = sum(per)
    value = args.steps * BATCH / secs / 1e6
    return {
        "metric": METRIC, "value": round(value, 3), "unit": "Mpts/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(secs / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32", "data": "synthetic", "impl": "reference",
        "config": bench_config(args),
        "cpu_baseline": {"value": round(value, 3), "unit": "Mpts/s", "cores": 1, "kind": how,
                         "sample": f"{args.steps} timed 1M-point batches after {args.warmup} warm-up batches",
                         "host_nproc": os.cpu_count()},
        "e2e": {"value": round(value, 3), "unit": "Mpts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=95)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="terrain", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--arena-gib", type=float, default=8.0)
    ap.add_argument("--cpu-batches", type=int, default=12)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-rows", action="store_true", help="skip the render / delta / Morton rows")
    ap.add_argument("--presort", action="store_true", help="experiment: z-order each batch on the host")
    ap.add_argument("--sim-dir", default="/tmp", help="where the disk-ingest row writes its SIM file")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank, world, local_rank = rank_env()
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_ours(args, rank, world, local_rank)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
