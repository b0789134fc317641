"""Per-step times of the bench's device-resident config-2 merge (jitter
check): wall clock and engine-stream events around every step.
Usage: python tools/step_jitter.py [steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import torch
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200.engine import get_engine

    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    n = bench.CFG["n"]
    ds, s1, s2 = bench.make_inputs(km, n)
    eng = get_engine(0)
    g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), bench.CFG["g_seed"], member_ids=s1, out_device=True)
    h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), bench.CFG["h_seed"], member_ids=s2, out_device=True)
    p = km.MergeParams(k=20, r=bench.CFG["r"], seed=bench.CFG["merge_seed"])
    for _ in range(3):
        km.s_merge(ds, g, h, p, out_device=True)
    torch.cuda.synchronize()
    eng.set_profiling(True)
    for i in range(steps):
        eng.reset_stats()
        eng.mark(0)
        t = time.perf_counter()
        u = km.s_merge(ds, g, h, p, out_device=True)
        eng.mark(1)
        ms = eng.elapsed_ms(0, 1)
        wall = (time.perf_counter() - t) * 1e3
        st = eng.stats()
        print(f"step {i}: dev {ms:.1f} ms wall {wall:.1f} ms  " +
              " ".join(f"{k[:-3]}={st[k]:.1f}" for k in ("join_ms", "assemble_ms", "update_ms", "reverse_ms", "other_ms")),
              flush=True)
        del u


if __name__ == "__main__":
    main()
