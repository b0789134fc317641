"""Full-size parity: BASELINE configs on the GPU against the CPU oracle on
identical inputs (subgraphs from the GPU NN-Descent, which the test suite
pins to the oracle).  Compares ids, fp64 dists, sizes, distance counts and
every round of the report, and computes recall@10 of BOTH outputs on the
same 1,000-node sample against exact brute force (GPU, fp64, (dist, id)
order).  The oracle is the checker here.

Usage: python tools/full_parity.py c3 c4 c5l1 [--scale s] -> JSON on stdout
(c2 and c2j -- a J-Merge of config-2 data -- are also accepted)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def recall(km, ds, metric, graph, q, truth):
    rows = np.searchsorted(np.asarray(graph.member_ids), q)
    got = np.asarray(graph.ids)[rows, :10]
    return sum(len(set(t) & set(g.tolist())) for t, g in zip(truth, got)) / (len(q) * 10)


def main():
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200.engine import get_engine
    from oracle import oracle as O

    O.build()
    args = sys.argv[1:]
    scale = float(args[args.index("--scale") + 1]) if "--scale" in args else 1.0
    names = [a for a in args if a.startswith("c") and not a.startswith("--")]
    out = {"scale": scale, "oracle_threads": os.cpu_count(), "cases": {}}
    for name in names:
        base = "c2" if name == "c2j" else name
        ds, metric, k, op, s1, s2, mpk = bench.config_inputs(km, base, scale)
        if name == "c2j":
            op = "j"
        t = time.perf_counter()
        g = km.nn_descent(ds, metric, km.DescentParams(k=k), 1, member_ids=s1)
        h = km.nn_descent(ds, metric, km.DescentParams(k=k), 2, member_ids=s2) if op == "s" else None
        t_build = time.perf_counter() - t

        def og(gr):
            o = O.OGraph(gr.member_ids, gr.k, int(gr.metric))
            o.ids, o.dists, o.sizes = gr.ids.copy(), gr.dists.copy(), gr.sizes.copy()
            return o

        mp = km.MergeParams(k=k, seed=3, **mpk)
        c = km.DistanceCounter()
        t = time.perf_counter()
        if op == "s":
            u, rep = km.s_merge(ds, g, h, mp, counter=c, return_report=True)
        else:
            u, rep = km.j_merge(ds, g, s2, mp, counter=c, return_report=True)
        t_gpu = time.perf_counter() - t
        okw = dict(max_iters=mp.max_iters, min_update_fraction=mp.min_update_fraction)
        t = time.perf_counter()
        if op == "s":
            ou, orep, ocount = O.s_merge(ds.vectors, og(g), og(h), k, seed=3, **okw)
        else:
            ou, orep, ocount = O.j_merge(ds.vectors, og(g), s2, k, seed=3, **okw)
        t_cpu = time.perf_counter() - t
        got = [(x.iteration, x.pairs, x.updates, x.phi, x.distance_count) for x in rep.rounds]
        want = [(x.iteration, x.pairs, x.updates, x.phi, x.distance_count) for x in orep.rounds]
        # recall@10 of both outputs on one 1,000-node sample (self excluded)
        eng = get_engine()
        q = np.sort(np.random.default_rng(0).choice(ds.n, size=min(1000, ds.n), replace=False))
        eng.set_dataset(ds.vectors, int(metric))
        tid, _ = eng.bf_topk(11, queries=ds.vectors[q])
        truth = [[int(v) for v in row if v != qq][:10] for row, qq in zip(tid, q)]
        r_gpu = recall(km, ds, metric, u, q, truth)
        r_orc = recall(km, ds, metric, ou, q, truth)
        case = {
            "op": {"s": "s_merge", "j": "j_merge"}[op], "n": int(ds.n), "d": int(ds.d), "k": k,
            "metric": metric.name.lower(),
            "ids_equal": bool(np.array_equal(u.ids, ou.ids)),
            "dists_equal": bool(np.array_equal(u.dists, ou.dists)),
            "sizes_equal": bool(np.array_equal(u.sizes, ou.sizes)),
            "members_equal": bool(np.array_equal(np.asarray(u.member_ids), np.asarray(ou.member_ids))),
            "count_equal": c.count == ocount, "count": int(c.count),
            "report_equal": got == want, "phi_initial_equal": rep.phi_initial == orep.phi_initial,
            "rounds": len(got), "report": got,
            "recall_at_10_gpu": r_gpu, "recall_at_10_oracle": r_orc, "recall_delta": r_gpu - r_orc,
            "recall_sample": "1,000 nodes, numpy default_rng(0).choice; GPU exact brute force",
            "gpu_seconds_incl_host_copies": round(t_gpu, 3), "oracle_seconds": round(t_cpu, 2),
            "subgraph_build_seconds_gpu": round(t_build, 2),
        }
        out["cases"][name] = case
        print(name, {k2: v for k2, v in case.items() if k2 != "report"}, file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
