"""GPU timeline of one config-2 S-Merge via torch.profiler (CUPTI kernel
activity): busy vs idle time, the largest idle gaps and the kernels around
them.  Usage: python tools/timeline.py [scale]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import torch
    from torch.profiler import ProfilerActivity, profile

    import paper_1908_00814_b200 as km

    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    n = int(bench.CFG["n"] * scale)
    ds, s1, s2 = bench.make_inputs(km, n)
    g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 1, member_ids=s1, out_device=True)
    h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 2, member_ids=s2, out_device=True)
    p = km.MergeParams(k=20, seed=3)
    km.s_merge(ds, g, h, p, out_device=True)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        km.s_merge(ds, g, h, p, out_device=True)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
    iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
    if not iv:
        print("no CUDA activity recorded")
        return
    busy, gaps, cur_end, prev = 0.0, [], iv[0][0], None
    for s, e, name in iv:
        if s > cur_end:
            gaps.append((s - cur_end, prev, name))
        if e > cur_end:
            busy += e - max(s, cur_end)
            cur_end = e
        prev = name
    span = cur_end - iv[0][0]
    print(f"wall {wall * 1e3:.1f} ms, gpu span {span / 1e3:.1f} ms, busy {busy / 1e3:.1f} ms, "
          f"idle {(span - busy) / 1e3:.1f} ms in {len(gaps)} gaps, activities {len(iv)}")
    by = {}
    for s_, e_, name in iv:
        key = "memset" if name.startswith("Memset") else "memcpy " + name.split("(")[1].split(")")[0] \
            if name.startswith("Memcpy") else name.split("(")[0].split("<")[0].replace("void ", "")
        by[key] = by.get(key, 0.0) + (e_ - s_)
    for key, v in sorted(by.items(), key=lambda kv: -kv[1])[:14]:
        print(f"  {key[:48]:48s} {v / 1e3:8.3f} ms")
    for d, a, b in sorted(gaps, reverse=True)[:15]:
        print(f"  gap {d / 1e3:7.3f} ms  after {str(a)[:40]:40s} before {str(b)[:40]}")


if __name__ == "__main__":
    main()
