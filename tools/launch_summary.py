"""Summarise an ncu launch list (--metrics gpu__time_duration.sum [, dram bytes] --csv)
into per-kernel shares:  python tools/launch_summary.py launches.csv "title" > summary.csv"""

import collections
import csv
import sys


def main(path, title):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr, data = rows[h], rows[h + 1:]
    iK, iM, iV, iID = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    iG = hdr.index("Grid Size") if "Grid Size" in hdr else None
    per = collections.defaultdict(dict)
    for r in data:
        d = per[r[iID]]
        d[r[iM]] = float(r[iV].replace(",", ""))
        d["k"] = r[iK].split("(")[0] + (f" grid{r[iG]}" if iG is not None else "")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in per.values():
        a = agg[d["k"]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"# {title}")
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: compare shares)")
    print(f"# kernels: {len(per)}, sum of durations: {tot / 1e3:.1f} us")
    print("share_pct,total_us,launches,us_per_launch,kernel")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{100 * a[1] / tot:.2f},{a[1] / 1e3:.1f},{a[0]},{a[1] / a[0] / 1e3:.2f},{k}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
