"""Join / apply kernel time of the first N rounds of a BASELINE config (device-resident inputs):
    python tools/join_round_time.py c3 0.3 1   # config, scale, rounds
KNNM_LIB selects another build of libknnm.so (ablation variants)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
import paper_1908_00814_b200 as km
from paper_1908_00814_b200.engine import get_engine

name = sys.argv[1]; scale = float(sys.argv[2]); iters = int(sys.argv[3]) if len(sys.argv) > 3 else 1
ds, metric, k, op, s1, s2, mpk = bench.config_inputs(km, name, scale)
g = km.nn_descent(ds, metric, km.DescentParams(k=k), 1, member_ids=s1, device=0, out_device=True)
h = km.nn_descent(ds, metric, km.DescentParams(k=k), 2, member_ids=s2, device=0, out_device=True) if op == "s" else None
mpk = dict(mpk); mpk["max_iters"] = iters
params = km.MergeParams(k=k, seed=3, **mpk)
eng = get_engine(0)
def run():
    c = km.DistanceCounter()
    if op == "s":
        return km.s_merge(ds, g, h, params, counter=c, device=0, out_device=True)
    return km.j_merge(ds, g, s2, params, counter=c, device=0, out_device=True)
run()
eng.reset_stats(); eng.set_profiling(True)
for _ in range(3): run()
st = eng.stats()
print(os.environ.get("KNNM_LIB", "default").split("/")[-1], name, scale, "join_kernel_ms", round(st["join_kernel_ms"] / 3, 2),
      "apply_kernel_ms", round(st["apply_kernel_ms"] / 3, 2), "rounds", st["rounds"] / 3)
