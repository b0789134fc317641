"""Host/GPU time of each phase of one device-resident config-2 s_merge
(the bench's `value` step), synchronising after every phase.
Usage: python tools/prologue_time.py"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    import torch
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import merge as M
    from paper_1908_00814_b200.construct import MODE_CROSS, BuildReport, _descent_rounds
    from paper_1908_00814_b200.engine import get_engine

    n = bench.CFG["n"]
    ds, s1, s2 = bench.make_inputs(km, n)
    g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 1, member_ids=s1, out_device=True)
    h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), 2, member_ids=s2, out_device=True)
    p = km.MergeParams(k=20, seed=3)
    for _ in range(3):
        km.s_merge(ds, g, h, p, out_device=True)
    eng = get_engine(0)
    for rep in range(3):
        T = {}
        torch.cuda.synchronize()

        def tick(name, t0):
            eng.sync()
            t1 = time.perf_counter()
            T[name] = (t1 - t0) * 1e3
            return t1

        t = time.perf_counter()
        t0 = t
        u, rg, rh, ov = M._merge_members(np.asarray(g.member_ids), np.asarray(h.member_ids), with_overlap=True)
        t = tick("merge_members", t)
        M._check_merge_inputs(ds, g, h.member_ids, p, h, overlap=ov)
        lab = np.zeros(u.shape[0], dtype=np.int8)
        lab[rh] = 1
        rng = np.random.default_rng(p.seed)
        t = tick("check+labels", t)
        eng.set_dataset(ds.vectors, 1)
        t = tick("set_dataset", t)
        eng.begin(u, lab, 20)
        t = tick("begin", t)
        eng.load_graph(rg, g, p.k1)
        eng.load_graph(rh, h, p.k1)
        t = tick("load_graph x2", t)
        c = km.DistanceCounter()
        M._append_random(eng, rg, rh, 10, rng, c, None, u)
        M._append_random(eng, rh, rg, 10, rng, c, None, u)
        t = tick("append_random x2", t)
        rep_ = BuildReport(phi_initial=eng.phi())
        t = tick("phi0", t)
        _descent_rounds(eng, u.shape[0], MODE_CROSS, 20, p.descent_params(), rng, c, None, u, rep_)
        t = tick("rounds", t)
        out = eng.export(merge_rear=True, on_device=True)
        t = tick("export", t)
        T["total"] = (t - t0) * 1e3
        print(" ".join(f"{k}={v:.2f}" for k, v in T.items()), flush=True)


if __name__ == "__main__":
    main()
