"""cProfile of one device-resident merge of a BASELINE config (host-side time
breakdown): python tools/host_profile_cfg.py c3 [scale]"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1908_00814_b200 as km  # noqa: E402

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
ds, metric, k, op, s1, s2, mpk = bench.config_inputs(km, name, scale)
g = km.nn_descent(ds, metric, km.DescentParams(k=k), 1, member_ids=s1, out_device=True)
h = km.nn_descent(ds, metric, km.DescentParams(k=k), 2, member_ids=s2, out_device=True) if op == "s" else None
p = km.MergeParams(k=k, seed=3, **mpk)


def run():
    if op == "s":
        return km.s_merge(ds, g, h, p, out_device=True)
    return km.j_merge(ds, g, s2, p, out_device=True)


run()
t = time.perf_counter()
run()
print("merge wall", time.perf_counter() - t)
pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(16)
