"""Per-source-line stall summary from `ncu --page source --csv --print-source=cuda,sass`."""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    out = []
    hdr = None
    fname = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or not r[0].isdigit():
            continue
        d = dict(zip(hdr, r))
        try:
            samp = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        stalls = {k[6:]: int(v) for k, v in d.items() if k.startswith("stall_") and v.isdigit() and int(v) > 0}
        out.append((samp, fname, r[0], r[1].strip()[:90], stalls,
                    d.get("L1 Wavefronts Shared Excessive", ""), d.get("Instructions Executed", "")))
    tot = sum(o[0] for o in out) or 1
    out.sort(key=lambda x: -x[0])
    for samp, f, ln, src, st, exc, ins in out[:top]:
        top3 = sorted(st.items(), key=lambda x: -x[1])[:3]
        print(f"{100*samp/tot:5.1f}% {f}:{ln:5s} inst={ins:>9s} shExc={exc:>6s} {top3} | {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
