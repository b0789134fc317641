import sys, time; sys.path.insert(0,'/root/repo')
import bench, paper_1908_00814_b200 as km
from paper_1908_00814_b200.engine import get_engine
n=1000000
ds, s1, s2 = bench.make_inputs(km, n)
g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 1, member_ids=s1, out_device=True)
h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 2, member_ids=s2, out_device=True)
eng = get_engine()
p = km.MergeParams(k=20, seed=3)
for it in (0, 2, 4, 8, 16, 32):
    eng.set_locality(it)
    km.s_merge(ds, g, h, p, out_device=True)
    eng.reset_stats(); eng.set_profiling(True)
    t=time.perf_counter(); km.s_merge(ds, g, h, p, out_device=True); dt=time.perf_counter()-t
    st=eng.stats(); eng.set_profiling(False)
    print(it, "wall %.1f ms" % (dt*1e3), {k: round(st[k],1) for k in ("join_ms","assemble_ms","update_ms","reverse_ms","other_ms")}, flush=True)
