"""One rank of the peer-memory multi-GPU path (launched by
tests/test_gpu_peer.py under torchrun; ranks may share one GPU, exchanging
over gloo).  Every global batch arrives striped (rank r holds points
[r*S, (r+1)*S)); PartitionedInserter warms up on rank 0, hands the packed tree
off and then routes the stripes through PeerRouter (bucket scatter straight
into the owners' IPC windows).  The rank then renders its tree into its
PeerFramebuffers window, composites over peer memory, and writes its owned
prefix subtrees (path -> samples), its copies of the replicated top nodes
(merged by global index after every batch) and the composite to
OUT/rank<r>.npz.

A second, standalone PeerRouter with a deliberately small window checks the
collective window growth and the routed records against the bucketing rule
applied to every rank's stripe (partition.take)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main() -> None:
    import torch
    import torch.distributed as dist

    from common import make_product
    from oracle.rebuild import tree_paths
    from paper_2310_03567_b200 import multigpu, partition, synth
    from paper_2310_03567_b200.render import Camera

    out = sys.argv[1]
    n_batches, stripe, depth = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = int(os.environ.get("LOCAL_RANK", 0)) % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    P = dict(bmin=(0.0, 0.0, 0.0), size=1.0, arena_bytes=512 << 20, chunk_capacity=256, grid_res=32,
             leaf_threshold=400, max_depth=14, backlog_capacity=10_000_000, spill_capacity=100_000_000)
    batches = [synth.gen_surface(world * stripe, 300 + i) for i in range(n_batches)]
    plan = partition.plan_owners(batches[:2], world, depth=depth)

    # standalone router: growth from a tiny window + record-exact routing
    router = multigpu.PeerRouter(dev, rank, world, plan, half_records=100)
    for i in range(3):
        x, c = batches[i]
        sl = slice(rank * stripe, (rank + 1) * stripe)
        rec = router.route(torch.from_numpy(x[sl]).cuda(), torch.from_numpy(c[sl].view(np.int32)).cuda())
        got = rec.cpu().numpy()
        want = []
        for s in range(world):
            ss = slice(s * stripe, (s + 1) * stripe)
            xr, cr = partition.take(plan, x[ss], c[ss], rank)
            want.append(np.concatenate([xr.view(np.int32), cr.view(np.int32).reshape(-1, 1)], axis=1))
        want = np.concatenate(want)
        assert got.shape == want.shape and np.array_equal(got, want), (rank, i, got.shape, want.shape)
    assert router.half_records > 100
    router.close()

    tree, state = make_product(P, device=dev)
    ins = multigpu.PartitionedInserter(tree, state, plan, rank, world)
    for x, c in batches:
        sl = slice(rank * stripe, (rank + 1) * stripe)
        ins.insert(torch.from_numpy(x[sl]).cuda(), torch.from_numpy(c[sl].view(np.int32)).cuda())
    ins.flush()  # the last batch's replicated-top merge
    assert ins.partitioned
    res = {}
    for path, nid in tree_paths(tree.inner, tree.children).items():
        if len(path) < plan.depth:  # a replicated top node: merged, every rank holds the single-tree sequence
            xs, cs = tree.gather_samples(nid)
            key = "t_" + "".join(map(str, path))
            res[key] = np.concatenate([xs.view(np.uint32), cs.reshape(-1, 1)], axis=1)
            res["tg_" + key[2:]] = tree.occupied_cells(nid)
            continue
        prefix = 0
        for o in path[: plan.depth]:
            prefix = prefix * 8 + o
        if int(plan.owner[prefix]) != rank:
            continue
        xs, cs = tree.gather_samples(nid)
        key = "p_" + "".join(map(str, path))
        res[key] = np.concatenate([xs.view(np.uint32), cs.reshape(-1, 1)], axis=1)
        if tree.inner[nid]:
            res["g_" + key[2:]] = tree.occupied_cells(nid)
    # render: this rank's tree into its window, depth-min composite over peer memory
    cam = Camera((0.5, 0.45, -1.3), (0.5, 0.5, 0.5), fov_deg=60.0, near=0.05, far=50.0, width=320, height=240)
    fbs = multigpu.PeerFramebuffers(dev, rank, world, cam.width, cam.height)
    comps = []
    for thr in (-1.0, 64.0):
        fbs.render(tree, cam, plan, thr)
        comps.append(fbs.composite().cells.copy())
    fbs.close()
    ins.close()
    np.savez(os.path.join(out, f"rank{rank}.npz"), comp_all=comps[0], comp_64=comps[1], **res)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
