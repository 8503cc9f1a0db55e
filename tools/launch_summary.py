"""Summarise an ncu launch list (--metrics gpu__time_duration.sum [, dram bytes] --csv)
into per-kernel shares:  python tools/launch_summary.py launches.csv "title" > summary.csv"""

import collections
import csv
import sys


UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, title):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    iK, iM, iV, iID = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    iG = hdr.index("Grid Size") if "Grid Size" in hdr else None
    iU = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    per = collections.defaultdict(dict)
    for r in data:
        d = per[r[iID]]
        scale = UNITS.get(r[iU], 1.0) if iU is not None and r[iM].startswith("dram__bytes") else 1.0
        d[r[iM]] = float(r[iV].replace(",", "")) * scale
        d["k"] = r[iK].split("(")[0] + (f" grid{r[iG]}" if iG is not None else "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        a = agg[d["k"]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"# {title}")
    print("# ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none")
    print("# (cold cache, serialised launches: compare shares; dram_GBs = DRAM bytes / duration per kernel)")
    print(f"# kernels: {len(per)}, sum of durations: {tot / 1e3:.1f} us")
    print("share_pct,total_us,launches,us_per_launch,dram_GBs,kernel")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = a[2] / a[1] if a[1] > 0 else 0.0  # bytes / ns = GB/s
        print(f"{100 * a[1] / tot:.2f},{a[1] / 1e3:.1f},{a[0]},{a[1] / a[0] / 1e3:.2f},{gbs:.0f},{k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
