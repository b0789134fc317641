"""cProfile of one full-size config-2 s_merge (host-side time breakdown)."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1908_00814_b200 as km  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
n = int(bench.CFG["n"] * scale)
ds, s1, s2 = bench.make_inputs(km, n)
g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 1, member_ids=s1, out_device=True)
h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 2, member_ids=s2, out_device=True)
p = km.MergeParams(k=20, seed=3)
km.s_merge(ds, g, h, p, out_device=True)
t = time.perf_counter()
km.s_merge(ds, g, h, p, out_device=True)
print("merge wall", time.perf_counter() - t)
pr = cProfile.Profile()
pr.enable()
km.s_merge(ds, g, h, p, out_device=True)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
