"""One warm merge of a BASELINE config (c2 / c3 / c4 stand-in) at a given
scale, with the CUDA profiler range around a second merge only (for
`ncu --profile-from-start off`).  Usage:
    python tools/profile_config.py c3 [--scale 0.1]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def main():
    import torch
    import paper_1908_00814_b200 as km
    from configs_bench import split

    name = sys.argv[1]
    scale = float(sys.argv[sys.argv.index("--scale") + 1]) if "--scale" in sys.argv else 0.1
    if name == "c2":
        n = int(1_000_000 * scale)
        ds, metric, k, op = km.generate_int_gmm(n, 128, 1000, 20.0, seed=7), km.Metric.L2, 20, "s"
    elif name == "c3":
        n = int(1_000_000 * scale)
        ds, metric, k, op = km.generate_unit_gmm(n, 960, 500, 0.05, seed=7), km.Metric.L2, 20, "j"
    else:
        n = int(1_200_000 * scale)
        ds, metric, k, op = km.generate_sphere_gmm(n, 100, 2000, 0.3, seed=7), km.Metric.COSINE, 40, "s"
    s1, s2 = split(n)
    g = km.nn_descent(ds, metric, km.DescentParams(k=k), 1, member_ids=s1)
    h = km.nn_descent(ds, metric, km.DescentParams(k=k), 2, member_ids=s2) if op == "s" else None
    params = km.MergeParams(k=k, seed=3)

    def once():
        c = km.DistanceCounter()
        t = time.perf_counter()
        u = km.s_merge(ds, g, h, params, counter=c) if op == "s" else km.j_merge(ds, g, s2, params, counter=c)
        return time.perf_counter() - t, c.count, u

    once()
    torch.cuda.synchronize()
    if "--timeline" in sys.argv:
        # CUPTI kernel/memcpy activity: busy vs idle and the largest gaps
        from torch.profiler import ProfilerActivity, profile

        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
            dt, cnt, _ = once()
            torch.cuda.synchronize()
        ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
        iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
        busy, gaps, cur, prev = 0.0, [], iv[0][0], None
        for s0, e0, nm in iv:
            if s0 > cur:
                gaps.append((s0 - cur, prev, nm))
            if e0 > cur:
                busy += e0 - max(s0, cur)
                cur = e0
            prev = nm
        print(f"{name}: wall {dt * 1e3:.1f} ms, gpu span {(cur - iv[0][0]) / 1e3:.1f} ms, "
              f"busy {busy / 1e3:.1f} ms, gaps {len(gaps)}")
        cat = {}
        for s0, e0, nm in iv:
            key = nm.split("(")[0] if nm.startswith(("Memcpy", "Memset")) else "kernels"
            cat[key] = cat.get(key, 0.0) + (e0 - s0)
        print("  by activity:", {k: round(v / 1e3, 1) for k, v in sorted(cat.items(), key=lambda x: -x[1])})
        for d0, a, b in sorted(gaps, reverse=True)[:12]:
            print(f"  gap {d0 / 1e3:8.3f} ms after {str(a)[:38]:38s} before {str(b)[:38]}")
        return
    from paper_1908_00814_b200.engine import get_engine

    get_engine().reset_stats()
    get_engine().set_profiling(True)
    torch.cuda.profiler.start()
    dt, cnt, _ = once()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    st = get_engine().stats()
    print(f"{name} scale {scale}: merge {dt:.3f} s evals {cnt}; join kernel {st['join_kernel_ms']:.1f} ms "
          f"apply kernel {st['apply_kernel_ms']:.1f} ms, tc joins {st['tc_join_launches']}, join launches {st['join_launches']}")


if __name__ == "__main__":
    main()
