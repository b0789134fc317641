"""BASELINE config 5 on ONE GPU: 8 k=20 subgraphs of 1,000,000 points each
(config-2 distribution, d=128, 8M points), merged pairwise by S-Merge in a
3-level tree (4 merges of 2M, 2 of 4M, 1 of 8M).  The reference runs the
tree serially on CPU (1,460 s); the 8-GPU placement of the
config is not available here, so the levels run one after another on one
device.  Subgraphs are built untimed by this package's NN-Descent.
Usage: python tools/c5_tree.py [--scale s] [--no-recall]"""
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
    from configs_bench import recall

    scale = float(sys.argv[sys.argv.index("--scale") + 1]) if "--scale" in sys.argv else 1.0
    per = int(1_000_000 * scale)
    n = 8 * per
    t = time.perf_counter()
    ds = km.generate_int_gmm(n, 128, 1000, 20.0, seed=7)
    parts = [np.arange(i * per, (i + 1) * per, dtype=np.int64) for i in range(8)]
    graphs = [km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=20), i + 1, member_ids=p, out_device=True)
              for i, p in enumerate(parts)]
    torch.cuda.synchronize()
    print(f"setup: data + 8 subgraphs of {per} points in {time.perf_counter() - t:.1f} s", flush=True)
    params = km.MergeParams(k=20, seed=3)
    total_evals, level_times = 0, []
    t_all = time.perf_counter()
    level = graphs
    while len(level) > 1:
        t_l = time.perf_counter()
        nxt = []
        for a, b in zip(level[0::2], level[1::2]):
            c = km.DistanceCounter()
            nxt.append(km.s_merge(ds, a, b, params, counter=c, out_device=True))
            total_evals += c.count
        torch.cuda.synchronize()
        level_times.append(time.perf_counter() - t_l)
        level = nxt
    wall = time.perf_counter() - t_all
    out = level[0]
    rec = None
    if "--no-recall" not in sys.argv:
        host = km.KnnGraph(out.member_ids, out.k, out.metric)
        host.ids, host.dists, host.sizes = (out.ids.cpu().numpy(), out.dists.cpu().numpy(),
                                            out.sizes.cpu().numpy())
        rec = recall(ds, km.Metric.L2, host)
    print(f"c5 tree on 1 GPU: n={n} levels {[round(x, 3) for x in level_times]} s, total {wall:.3f} s, "
          f"evals {total_evals}, {total_evals / wall:.3e} evals/s, recall@10 {rec}", flush=True)


if __name__ == "__main__":
    main()
