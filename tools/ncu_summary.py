"""Summarise an ``ncu --set full`` capture per kernel launch and record the
DRAM traffic of each kernel for bench.py's ``roofline.traffic``.

    ncu -i gpurun_out/X.ncu-rep --page raw --csv > /tmp/raw.csv
    python tools/ncu_summary.py /tmp/raw.csv [--json profiles/ncu_traffic.json] > profiles/rNN_ncu_full_summary.txt
"""
import argparse
import collections
import csv
import json

COLS = {
    "time_us": "gpu__time_duration.sum",
    "dram_rd_MB": "dram__bytes_read.sum",
    "dram_wr_MB": "dram__bytes_write.sum",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "mem_tput_pct": "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_tput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
}
SCALE = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}


def load(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").split("<")[0].strip()}
        for k, c in COLS.items():
            if c not in hdr:
                continue
            i = hdr.index(c)
            v = float(r[i].replace(",", "")) if r[i] else 0.0
            d[k] = v * SCALE.get(units[i], 1.0)
        out.append(d)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--json")
    a = ap.parse_args()
    launches = load(a.raw)
    tot_t = sum(d["time_us"] for d in launches)
    print(f"{'kernel':16s} {'us':>8s} {'share':>6s} {'dramRd':>8s} {'dramWr':>8s} {'GB/s':>7s} {'L2hit':>6s} "
          f"{'warps%':>6s} {'mem%':>6s} {'sm%':>6s} {'regs':>4s} {'grid':>6s}")
    for d in launches:
        gbs = (d["dram_rd_MB"] + d["dram_wr_MB"]) * 1e6 / (d["time_us"] * 1e-6) / 1e9
        print(f"{d['kernel'][:16]:16s} {d['time_us']:8.1f} {100 * d['time_us'] / tot_t:5.1f}% {d['dram_rd_MB']:7.2f}M "
              f"{d['dram_wr_MB']:7.2f}M {gbs:7.0f} {d.get('l2_hit_pct', 0):6.1f} {d.get('warps_active_pct', 0):6.1f} "
              f"{d.get('mem_tput_pct', 0):6.1f} {d.get('sm_tput_pct', 0):6.1f} {int(d.get('regs', 0)):4d} "
              f"{int(d.get('grid', 0)):6d}")
    print(f"TOTAL {tot_t:.1f} us over {len(launches)} launches (serialised, replayed: shares, not absolutes)")
    if a.json:
        per = collections.defaultdict(list)
        for d in launches:
            per[d["kernel"]].append((d["dram_rd_MB"] + d["dram_wr_MB"]) * 1e6)
        traffic = {k: int(sum(v) / len(v)) for k, v in per.items()}
        json.dump(traffic, open(a.json, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
