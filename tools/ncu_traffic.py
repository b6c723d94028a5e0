"""Merge ncu metric captures (tools/ncu_traffic.sh) into profiles/ncu_traffic.json:
per kernel, mean DRAM bytes (read + write) per launch over the captured
batch range, keyed by (config, [W, W+K]) so bench.py uses a capture only for
the batches it timed."""
import collections
import csv
import datetime
import json
import os
import re
import sys

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def parse(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, mi, ui, vi = (hdr.index(c) for c in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    idi = hdr.index("ID")
    per = collections.defaultdict(lambda: collections.defaultdict(float))
    names = {}
    for r in rows[1:]:
        lid = r[idi]
        names[lid] = r[ki].split("(")[0].replace("void ", "").split("<")[0].strip()
        v = float(r[vi].replace(",", ""))
        if r[mi].startswith("dram__bytes"):
            per[lid]["bytes"] += v * SCALE.get(r[ui], 1)
        elif r[mi] == "gpu__time_duration.sum":
            per[lid]["ns"] += v * (1e3 if r[ui] == "usecond" else 1e6 if r[ui] == "msecond" else 1)
    agg = collections.defaultdict(list)
    for lid, d in per.items():
        agg[names[lid]].append(d["bytes"])
    return {k: int(sum(v) / len(v)) for k, v in agg.items()}, {k: len(v) for k, v in agg.items()}


def main():
    try:
        doc = json.load(open(OUT))
        caps = doc.get("captures", [])
    except Exception:
        caps = []
    for path in sys.argv[1:]:
        m = re.search(r"traffic_(\w+?)_(\d+)_(\d+)\.csv$", path)
        cfg, w, k = m.group(1), int(m.group(2)), int(m.group(3))
        byts, launches = parse(path)
        caps = [c for c in caps if not (c["config"] == cfg and c["batches"] == [w, w + k])]
        caps.append({"config": cfg, "batches": [w, w + k], "per_launch_bytes": byts, "launches": launches,
                     "command": f"bash tools/ncu_traffic.sh {cfg} {w} {k}",
                     "when": datetime.date.today().isoformat()})
    json.dump({"captures": caps}, open(OUT, "w"), indent=1, sort_keys=True)
    print(json.dumps(caps[-1], indent=1)[:2000])


if __name__ == "__main__":
    main()
