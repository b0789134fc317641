"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hdr_i]
    kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows[hdr_i + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        name = r[kn].split("(")[0].split("<")[0].replace("void ", "").strip()
        v = float(r[mv].replace(",", ""))
        tot[name] += v
        cnt[name] += 1
    total = sum(tot.values())
    unit = hdr[hdr.index("Metric Unit")] if "Metric Unit" in hdr else ""
    print(f"{'kernel':40s} {'launches':>8s} {'total':>14s} {'share':>7s}")
    for name, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{name:40s} {cnt[name]:8d} {v:14.0f} {100*v/total:6.1f}%")
    print(f"{'TOTAL':40s} {sum(cnt.values()):8d} {total:14.0f}")


if __name__ == "__main__":
    main(sys.argv[1])
