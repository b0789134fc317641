"""Stall summary of one kernel's SASS from
`ncu -i rep --page source --csv --print-source=sass [-k regex:name]`.
Usage: python tools/ncu_sass_stalls.py file.csv [top] [block_index]"""
import collections
import csv
import sys


def main(path, top=20, which=0):
    rows = list(csv.reader(open(path)))
    starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
    a = starts[which]
    b = starts[which + 1] if which + 1 < len(starts) else len(rows)
    blk = rows[a:b]
    hdr, data = blk[1], blk[2:]
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ti = hdr.index("Avg. Threads Executed")
    sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    num = lambda v: int(v) if v.isdigit() else 0
    tot = sum(num(r[si]) for r in data) or 1
    agg = collections.Counter()
    for r in data:
        for i in sc:
            agg[hdr[i]] += num(r[i])
    print(blk[0][1][:80], "samples", tot)
    print(" ", [(k, round(100 * v / tot, 1)) for k, v in agg.most_common(8)])
    order = sorted(range(len(data)), key=lambda i: -num(data[i][si]))[:top]
    for i in order:
        r = data[i]
        why = sorted(((num(r[j]), hdr[j][6:]) for j in sc if num(r[j])), reverse=True)[:2]
        print(f"{100 * num(r[si]) / tot:5.1f}% #{i:5d} th={r[ti]:>5} {r[1].strip()[:52]:52s} {why}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20,
         int(sys.argv[3]) if len(sys.argv) > 3 else 0)
