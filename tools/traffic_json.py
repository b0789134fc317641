"""Per-launch DRAM traffic of one kernel from an ncu --csv launch list with
gpu__time_duration.sum, dram__bytes_read.sum and dram__bytes_write.sum, as
the JSON bench.py attaches to its roofline (profiles/r2_<kernel>_traffic.json).
Usage: python tools/traffic_json.py list.csv <regex> <label> <source> > out.json"""
import csv
import json
import re
import sys
from collections import defaultdict


def main(path, pattern, label, source):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, ni, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    per = defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi or not re.search(pattern, r[ki]):
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        if r[ni].startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif r[ni] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
        per[int(r[idi])][r[ni]] = v
        names[int(r[idi])] = r[ki].split("(")[0]
    ids = sorted(per)
    rd = [per[i].get("dram__bytes_read.sum", 0.0) for i in ids]
    wr = [per[i].get("dram__bytes_write.sum", 0.0) for i in ids]
    ms = [per[i].get("gpu__time_duration.sum", 0.0) for i in ids]
    tot = [a + b for a, b in zip(rd, wr)]
    out = {"kernel": label, "source": source, "launches": len(ids),
           "dram_bytes_per_launch_avg": sum(tot) / max(1, len(ids)), "dram_bytes_per_step": sum(tot),
           "dram_bytes_per_launch": tot, "dram_read_bytes_per_launch": rd,
           "dram_write_bytes_per_launch": wr, "ncu_ms_per_launch": ms,
           "note": "cold-cache, serialised ncu replay; per-launch DRAM read+write bytes"}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:5])
