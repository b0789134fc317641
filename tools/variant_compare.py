"""Time one BASELINE config under several local-join routes and check that
they agree bit for bit (ids, dists, counts, per-round updates).

    python tools/variant_compare.py c4 [--scale 1.0] [--variants 1,-1] [--reps 3]

Prints one JSON line per variant (merge seconds, join-kernel and apply
milliseconds from the engine's CUDA-event phase timers, exact evaluations).
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))


def arg(name, default):
    return sys.argv[sys.argv.index(name) + 1] if name in sys.argv else default


def main():
    import torch
    import paper_1908_00814_b200 as km
    from configs_bench import split
    from paper_1908_00814_b200.engine import get_engine

    name = sys.argv[1]
    scale = float(arg("--scale", "1.0"))
    variants = [int(v) for v in arg("--variants", "1,-1").split(",")]
    reps = int(arg("--reps", "3"))
    if name == "c1":
        n = int(10_000 * scale)
        ds, metric, k, op = km.generate_uniform(n, 32, seed=7), km.Metric.L2, 20, "s"
    elif name == "c2":
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
    eng = get_engine()
    ref = None
    for v in variants:
        eng.set_join_variant(v)
        times, st = [], None
        for r in range(reps + 2):
            eng.set_profiling(r == reps + 1)  # last merge: phase timers on (not in merge_s)
            c = km.DistanceCounter()
            eng.reset_stats()
            torch.cuda.synchronize()
            t = time.perf_counter()
            if op == "s":
                u, rep = km.s_merge(ds, g, h, params, counter=c, return_report=True)
            else:
                u, rep = km.j_merge(ds, g, s2, params, counter=c, return_report=True)
            torch.cuda.synchronize()
            if 0 < r <= reps:
                times.append(time.perf_counter() - t)
            st = eng.stats()
        out = (u.ids.copy(), u.dists.copy(), c.count, [x.updates for x in rep.rounds])
        same = None
        if ref is None:
            ref = out
        else:
            same = (np.array_equal(ref[0], out[0]) and np.array_equal(ref[1], out[1])
                    and ref[2] == out[2] and ref[3] == out[3])
        print(json.dumps({"config": name, "scale": scale, "variant": v, "merge_s": min(times),
                          "join_kernel_ms": st["join_kernel_ms"], "apply_kernel_ms": st["apply_kernel_ms"],
                          "update_ms": st["update_ms"], "exact_evals": st["exact_evals"],
                          "written_slots": st["written_slots"], "dense_launches": st.get("dense_join_launches"),
                          "rounds": len(rep.rounds), "evals": c.count, "same_as_first": same}), flush=True)
    eng.set_join_variant(-1)
    eng.set_profiling(False)


if __name__ == "__main__":
    main()
