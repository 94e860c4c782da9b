"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) as the
markdown table used in profiles/*.md:  python tools/launch_table.py <csv>"""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = {k: j for j, k in enumerate(rows[start])}
    agg = collections.defaultdict(lambda: [0.0, 0])
    tot, n = 0.0, 0
    for r in rows[start + 1:]:
        if len(r) < len(h) or r[h["Metric Name"]] != "gpu__time_duration.sum":
            continue
        v = float(r[h["Metric Value"]].replace(",", ""))
        unit = r[h["Metric Unit"]]
        v = v / 1000 if unit in ("nsecond", "ns") else v * 1000 if unit == "msecond" else v
        key = re.sub(r"\(.*", "", r[h["Kernel Name"]])[:60]
        agg[key][0] += v
        agg[key][1] += 1
        tot += v
        n += 1
    print("| kernel | us | launches | share |\n|---|---:|---:|---:|")
    for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"| {k} | {v:.1f} | {c} | {100 * v / tot:.1f} % |")
    print(f"| **total** | **{tot:.1f}** | {n} | |")


if __name__ == "__main__":
    main(sys.argv[1])
