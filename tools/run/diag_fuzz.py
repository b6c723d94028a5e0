import os, sys
import numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from test_gpu_fuzz import _case
from common import run_oracle, run_product, product_state, oracle_state

seed = int(sys.argv[1])
params, batches = _case(1000 + seed)
print("params", params, "batches", len(batches), "sizes", sorted(set(len(c) for _, c in batches)))
ot, oerr, oper = run_oracle(params, batches)
tree, state, err, per = run_product(params, batches)
print("err", err, oerr)
bad = next((i for i, (a, b) in enumerate(zip(per, oper)) if a != b), None)
print("first differing batch", bad, per[bad] if bad is not None else None, oper[bad] if bad is not None else None)
if bad is not None:
    ot2, _, _ = run_oracle(params, batches[:bad + 1])
    t2, s2, _, _ = run_product(params, batches[:bad + 1])
    a, b = product_state(t2), oracle_state(ot2)
    print("nodes", a["num_nodes"], b["num_nodes"])
    n = min(a["num_nodes"], b["num_nodes"])
    for k in ("parent", "level", "inner", "count"):
        d = np.flatnonzero(np.asarray(a[k][:n]) != np.asarray(b[k][:n]))
        print(k, "differs at", d[:10])
    ao, bo = a["rec_offsets"], b["rec_offsets"]
    for nid in range(n):
        ra = a["records"][ao[nid]:ao[nid + 1]].view(np.uint32)
        rb = b["records"][bo[nid]:bo[nid + 1]].view(np.uint32)
        if ra.shape != rb.shape or not np.array_equal(ra, rb):
            print("node", nid, "level", b["level"][nid], "inner", b["inner"][nid], "counts", len(ra), len(rb))
            print(" prod", ra[:6].tolist())
            print(" orac", rb[:6].tolist())
            break
    ca, cb = a["cell_offsets"], b["cell_offsets"]
    for nid in range(n):
        x, y = a["cells"][ca[nid]:ca[nid + 1]], b["cells"][cb[nid]:cb[nid + 1]]
        if not np.array_equal(x, y):
            print("cells differ node", nid, "prod-only", sorted(set(x) - set(y))[:10], "orac-only", sorted(set(y) - set(x))[:10])
            break
