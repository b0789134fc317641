"""Per-CUDA-source-line stall samples split by reason, from
`ncu -i rep --page source --csv --print-source=cuda,sass`.
Usage: python tools/ncu_line_stalls.py file.csv [reason] [top]"""
import collections
import csv
import sys


def main(path, reason="stall_long_sb", top=15):
    fname, hdr = None, None
    samp, src = collections.Counter(), {}
    total = 0
    for r in csv.reader(open(path)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r[0].isdigit() or r[2] != "-":
            continue
        key = (fname, int(r[0]))
        src[key] = r[1].strip()[:80]
        v = int(r[hdr.index(reason)] or 0)
        samp[key] += v
        total += v
    print(reason, "samples", total)
    for key, v in samp.most_common(top):
        print(f"{100 * v / max(total, 1):5.1f}% {key[0]}:{key[1]} {src[key]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb",
         int(sys.argv[3]) if len(sys.argv) > 3 else 15)
