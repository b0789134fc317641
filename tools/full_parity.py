"""Full-size parity: BASELINE config 2 (S-Merge of 2 x 500,000, d=128, k=20)
and a config-3-shaped J-Merge on the GPU against the CPU oracle on the same
inputs (subgraphs from the GPU NN-Descent, which the test suite pins to the
oracle), comparing ids, fp64 dists, sizes, distance counts and every round
of the report.  The oracle is the checker here.
Usage: python tools/full_parity.py [scale] -> JSON on stdout"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import paper_1908_00814_b200 as km
    from oracle import oracle as O

    O.build()
    scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    n = int(bench.CFG["n"] * scale)
    ds, s1, s2 = bench.make_inputs(km, n)
    k = bench.CFG["k"]
    g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=k), bench.CFG["g_seed"], member_ids=s1)
    h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=k), bench.CFG["h_seed"], member_ids=s2)

    def og(gr):
        o = O.OGraph(gr.member_ids, gr.k, int(gr.metric))
        o.ids, o.dists, o.sizes = gr.ids.copy(), gr.dists.copy(), gr.sizes.copy()
        return o

    out = {"n": n, "cases": {}}
    mp = km.MergeParams(k=k, r=bench.CFG["r"], seed=bench.CFG["merge_seed"])
    for op in ("s_merge", "j_merge"):
        c = km.DistanceCounter()
        t = time.perf_counter()
        if op == "s_merge":
            u, rep = km.s_merge(ds, g, h, mp, counter=c, return_report=True)
        else:
            u, rep = km.j_merge(ds, g, s2, mp, counter=c, return_report=True)
        t_gpu = time.perf_counter() - t
        t = time.perf_counter()
        if op == "s_merge":
            ou, orep, ocount = O.s_merge(ds.vectors, og(g), og(h), k, r=bench.CFG["r"],
                                         seed=bench.CFG["merge_seed"])
        else:
            ou, orep, ocount = O.j_merge(ds.vectors, og(g), s2, k, r=bench.CFG["r"],
                                         seed=bench.CFG["merge_seed"])
        t_cpu = time.perf_counter() - t
        got = [(x.iteration, x.pairs, x.updates, x.phi, x.distance_count) for x in rep.rounds]
        want = [(x.iteration, x.pairs, x.updates, x.phi, x.distance_count) for x in orep.rounds]
        out["cases"][op] = {
            "ids_equal": bool(np.array_equal(u.ids, ou.ids)),
            "dists_equal": bool(np.array_equal(u.dists, ou.dists)),
            "sizes_equal": bool(np.array_equal(u.sizes, ou.sizes)),
            "count_equal": c.count == ocount, "count": int(c.count),
            "report_equal": got == want, "rounds": len(got),
            "gpu_seconds_incl_host_copies": round(t_gpu, 3), "oracle_seconds": round(t_cpu, 2),
            "oracle_threads": os.cpu_count(),
        }
        print(op, out["cases"][op], file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
