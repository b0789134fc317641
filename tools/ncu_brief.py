"""Print the headline metrics of each kernel in an .ncu-rep (details page)."""
import csv
import subprocess
import sys

WANT = ['Duration', 'DRAM Throughput', 'L2 Cache Throughput', 'L1/TEX Cache Throughput',
        'Compute (SM) Throughput', 'Achieved Occupancy', 'Theoretical Occupancy',
        'Registers Per Thread', 'Executed Ipc Active', 'No Eligible',
        'Dynamic Shared Memory Per Block', 'L2 Hit Rate', 'Warp Cycles Per Issued Instruction',
        'Avg. Active Threads Per Warp', 'Block Limit Shared Mem', 'Block Limit Registers',
        'Memory Throughput']


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    idi = hdr.index("ID")
    seen = set()
    for r in rows[1:]:
        key = (r[idi], r[mi], r[ui])
        if r[mi] in WANT and key not in seen:
            seen.add(key)
            print(f"[{r[idi]}] {r[ki][:24]:24s} | {r[mi]} = {r[vi]} {r[ui]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
