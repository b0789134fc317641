"""Time the BASELINE.json configs 1-4 on one GPU (merge seconds, distance
evals/s, recall@10 on a 1,000-node sample), inputs built by the GPU
NN-Descent.  Usage: python tools/configs_bench.py [c1 c2 c3 c4] [--scale s]"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1908_00814_b200 as km  # noqa: E402
from paper_1908_00814_b200.engine import get_engine  # noqa: E402


def split(n, seed=1):
    perm = np.random.default_rng(seed).permutation(n)
    return np.sort(perm[: n // 2]), np.sort(perm[n // 2:])


def recall(ds, metric, g, nq=1000):
    eng = get_engine()
    q = np.sort(np.random.default_rng(0).choice(ds.n, size=min(nq, ds.n), replace=False))
    eng.set_dataset(ds.vectors, int(metric))
    ids, _ = eng.bf_topk(11, queries=ds.vectors[q])
    truth = [[int(v) for v in row if v != qq][:10] for row, qq in zip(ids, q)]
    got = np.asarray(g.ids)[np.searchsorted(g.member_ids, q), :10]
    return sum(len(set(t) & set(x.tolist())) for t, x in zip(truth, got)) / (len(q) * 10)


def run(name, scale):
    if name == "c1":
        ds = km.generate_uniform(10000, 32, seed=1)
        s1, s2 = np.arange(5000), np.arange(5000, 10000)
        metric, k, op, mp = km.Metric.L2, 20, "s", dict(max_iters=10, min_update_fraction=0.0)
    elif name == "c2":
        n = int(1_000_000 * scale)
        ds = km.generate_int_gmm(n, 128, 1000, 20.0, seed=7)
        s1, s2 = split(n)
        metric, k, op, mp = km.Metric.L2, 20, "s", {}
    elif name == "c3":
        n = int(1_000_000 * scale)
        ds = km.generate_unit_gmm(n, 960, 500, 0.05, seed=7)
        s1, s2 = split(n)
        metric, k, op, mp = km.Metric.L2, 20, "j", {}
    else:
        n = int(1_200_000 * scale)
        ds = km.generate_sphere_gmm(n, 100, 2000, 0.3, seed=7)
        s1, s2 = split(n)
        metric, k, op, mp = km.Metric.COSINE, 40, "s", {}
    t = time.perf_counter()
    g = km.nn_descent(ds, metric, km.DescentParams(k=k), 1, member_ids=s1)
    h = km.nn_descent(ds, metric, km.DescentParams(k=k), 2, member_ids=s2) if op == "s" else None
    setup = time.perf_counter() - t
    params = km.MergeParams(k=k, seed=3, **mp)
    eng = get_engine()
    for it in range(2):
        c = km.DistanceCounter()
        eng.reset_stats()
        eng.set_profiling(it == 1)
        if it == 1:
            torch.cuda.profiler.start()  # ncu --profile-from-start off: the timed merge only
        t = time.perf_counter()
        u = km.s_merge(ds, g, h, params, counter=c) if op == "s" else km.j_merge(ds, g, s2, params, counter=c)
        dt = time.perf_counter() - t
        if it == 1:
            torch.cuda.profiler.stop()
    st = eng.stats()
    eng.set_profiling(False)
    print(f"{name}: n={ds.n} d={ds.d} merge {dt:.3f} s, {c.count/dt:.3e} evals/s, evals {c.count}, "
          f"recall@10 {recall(ds, metric, u):.4f}, setup {setup:.1f} s, exact_evals {st["exact_evals"]}, accepted {st["accepted"]}, "
          f"phases ms " + " ".join(f"{k}={st[k]:.1f}" for k in ("join_ms", "join_kernel_ms", "assemble_ms",
                                                                "update_ms", "reverse_ms", "other_ms")),
          flush=True)


if __name__ == "__main__":
    scale = float(sys.argv[sys.argv.index("--scale") + 1]) if "--scale" in sys.argv else 1.0
    names = [a for a in sys.argv[1:] if a.startswith("c") and len(a) == 2] or ["c1", "c2", "c3", "c4"]
    for nm in names:
        run(nm, scale)
