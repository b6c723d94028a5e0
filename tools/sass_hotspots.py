"""Top stall-sampled SASS instructions of one kernel from an ncu report.

    python tools/sass_hotspots.py report.ncu-rep KERNEL [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "-k", kern, "-c", "1", "--page", "source", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
    si, src, ex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Source"), hdr.index("Instructions Executed")
    tot = sum(int(r[si] or 0) for r in data) or 1
    print(f"{kern}: {tot} stall samples over {len(data)} SASS instructions")
    for r in sorted(data, key=lambda r: -int(r[si] or 0))[:n]:
        print(f"{int(r[si]) / tot * 100:5.1f}%  {r[0][-5:]}  {r[src].strip()[:64]:64s} exec={r[ex]}")


if __name__ == "__main__":
    main()
