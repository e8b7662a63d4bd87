"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv)
into a markdown table of per-kernel totals and shares.

    python tools/launches_summary.py launches.csv "title" > profiles/launches_X.md
"""
import csv
import sys
from collections import defaultdict


def main():
    path, title = sys.argv[1], sys.argv[2]
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if "Kernel Name" in r and "Metric Name" in r:
            hdr = {h: i for i, h in enumerate(r)}
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        if r[hdr["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = r[hdr["Metric Unit"]]
        v = float(r[hdr["Metric Value"]].replace(",", ""))
        scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3,
                 "msecond": 1.0, "ms": 1.0, "second": 1e3,
                 "s": 1e3}.get(unit, 1.0)
        name = r[hdr["Kernel Name"]][:60]
        tot[name] += v * scale
        cnt[name] += 1
    allms = sum(tot.values()) or 1.0
    print(f"# {title}\n")
    print("ncu --metrics gpu__time_duration.sum --clock-control none "
          "(cold-cache, serialised: compare shares, not absolutes).\n")
    print("| kernel | launches | total ms | share |")
    print("|---|---|---|---|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {cnt[k]} | {v:.2f} | {100 * v / allms:.1f}% |")


if __name__ == "__main__":
    main()
