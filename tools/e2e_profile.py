"""Where does the e2e (host-buffer) s_merge time go?  cProfile of one call."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1908_00814_b200 as km  # noqa: E402
from paper_1908_00814_b200.engine import get_engine, pinned_copy  # noqa: E402

ds, s1, s2 = bench.make_inputs(km, 1_000_000)
g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 1, member_ids=s1)
h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 2, member_ids=s2)
dsp = km.Dataset.from_dense(pinned_copy(ds.vectors), validate=False)
for gr in (g, h):
    gr.ids, gr.dists, gr.sizes = pinned_copy(gr.ids), pinned_copy(gr.dists), pinned_copy(gr.sizes)
eng = get_engine()
p = km.MergeParams(k=20, seed=3)
for _ in range(2):
    eng.invalidate()
    eng.pinned_outputs = True
    t = time.perf_counter()
    km.s_merge(dsp, g, h, p)
    print("e2e wall", time.perf_counter() - t, flush=True)
t = time.perf_counter(); eng.set_dataset(dsp.vectors, 1); print("set_dataset", time.perf_counter() - t)
eng.invalidate()
pr = cProfile.Profile()
pr.enable()
km.s_merge(dsp, g, h, p)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
