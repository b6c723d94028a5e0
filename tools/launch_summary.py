"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv [--skip-first N]
"""
import collections
import csv
import sys

UNITS = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "").split("<")[0].strip()
        us = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1.0)
        tot[name] += us
        cnt[name] += 1
    return tot, cnt


if __name__ == "__main__":
    tot, cnt = summarize(sys.argv[1])
    T = sum(tot.values())
    print(f"{'kernel':28s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:28s} {cnt[k]:8d} {v:12.1f} {v / cnt[k]:10.2f} {v / T * 100:6.1f}%")
    print(f"{'TOTAL':28s} {sum(cnt.values()):8d} {T:12.1f}")
