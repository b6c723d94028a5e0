"""The reference itself (lodstream, numba) vs its 1-thread C restatement (the
oracle the bench's --impl reference arm times) on the same host and batches:
the terrain stream's batches 5..K after 5 untimed warm-up batches (numba's
JIT compiles during the warm-up).  Uses the staged copy of the reference
(tests/ref_suite/_ref, built by __graft_entry__.build() where /root/reference
exists; git-ignored, it travels to the GPU box with the working tree).

    python tools/ref_vs_port.py [--batches 12]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=12)
    ap.add_argument("--warmup", type=int, default=5)
    a = ap.parse_args()
    from bench import PARAMS, gen_batches

    batches = gen_batches("surface", a.batches)
    out = {"batches_timed": [a.warmup, a.batches], "host_nproc": os.cpu_count()}

    # the port (bench.py's reference arm)
    import oracle

    t = oracle.OracleTree(grid_res=PARAMS["grid_res"], leaf_threshold=PARAMS["leaf_threshold"],
                          max_depth=PARAMS["max_depth"], chunk_capacity=PARAMS["chunk_capacity"],
                          arena_bytes=8 << 30, backlog_capacity=64_000_000)
    for x, c in batches[:a.warmup]:
        t.insert_batch(x, c)
    t0 = time.perf_counter()
    for x, c in batches[a.warmup:]:
        t.insert_batch(x, c)
    dt = time.perf_counter() - t0
    out["port_mpts_s"] = round((a.batches - a.warmup) * 1e6 / dt / 1e6, 3)
    port_state = t.state()
    del t

    # the reference package, unmodified
    ref = os.path.join(ROOT, "tests", "ref_suite", "_ref")
    if not os.path.isdir(os.path.join(ref, "lodstream")):
        out["reference"] = "not staged (needs /root/reference at build time)"
        print(json.dumps(out))
        return
    sys.path.insert(0, ref)
    from lodstream.octree import CubeBounds, Octree
    from lodstream.store import Arena, ChunkPool
    from lodstream.update import UpdateConfig, UpdateState, insert_batch

    arena = Arena(8 << 30)
    tree = Octree(CubeBounds((0.0, 0.0, 0.0), 1.0), arena, ChunkPool(arena, PARAMS["chunk_capacity"]),
                  grid_res=PARAMS["grid_res"], leaf_threshold=PARAMS["leaf_threshold"], max_depth=PARAMS["max_depth"])
    state = UpdateState(UpdateConfig(backlog_capacity=64_000_000))
    for x, c in batches[:a.warmup]:
        insert_batch(tree, x, c, state)
    t0 = time.perf_counter()
    for x, c in batches[a.warmup:]:
        insert_batch(tree, x, c, state)
    dt = time.perf_counter() - t0
    out["reference_mpts_s"] = round((a.batches - a.warmup) * 1e6 / dt / 1e6, 3)
    out["same_tree"] = {"num_nodes": [int(tree.num_nodes), int(port_state["num_nodes"])]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
