"""Run one config-2-shaped S-Merge with the CUDA profiler range around the
merge only (for `ncu --profile-from-start off`), plus host-side phase wall
times.  Usage: python tools/profile_merge.py [scale] [--merges N]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import torch
    import paper_1908_00814_b200 as km

    scale = float(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 0.1
    merges = int(sys.argv[sys.argv.index("--merges") + 1]) if "--merges" in sys.argv else 1
    n = int(bench.CFG["n"] * scale)
    ds, s1, s2 = bench.make_inputs(km, n)
    g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 1, member_ids=s1)
    h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 2, member_ids=s2)
    params = km.MergeParams(k=20, seed=3)
    km.s_merge(ds, g, h, params)  # warm
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for _ in range(merges):
        t0 = time.perf_counter()
        u, rep = km.s_merge(ds, g, h, params, return_report=True)
        dt = time.perf_counter() - t0
    torch.cuda.profiler.stop()
    print(f"n={n} merge wall {dt*1e3:.1f} ms rounds={len(rep.rounds)} "
          f"pairs={[r.pairs for r in rep.rounds]}", flush=True)


if __name__ == "__main__":
    main()
