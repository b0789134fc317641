"""Per-CUDA-source-line instruction and stall-sample shares of one kernel from
`ncu -i rep --page source --csv --print-source=cuda,sass -k regex:NAME`.
Usage: python tools/ncu_lines.py file.csv [top]"""
import collections
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    fname, hdr = None, None
    inst, samp, src = collections.Counter(), collections.Counter(), {}
    for r in rows:
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
        src[key] = r[1].strip()[:72]
        inst[key] += int(r[hdr.index("Instructions Executed")] or 0)
        samp[key] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    ti, ts = sum(inst.values()) or 1, sum(samp.values()) or 1
    print("instructions", ti, "samples", ts)
    for key, v in inst.most_common(top):
        print(f"{100 * v / ti:5.1f}% inst {100 * samp[key] / ts:5.1f}% smp {key[0]}:{key[1]} {src[key]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
