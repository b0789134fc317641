"""Exact k-NN ground truth at scale on the tensor cores (knnm_bf.cuh).

Builds the config-2 distribution at n points (default 1,000,000, d=128,
integers in [0, 255]), times ``brute_force_graph(k=20)`` (n x n Gram tiles on
tcgen05 kind::i8, exact integer distances), then checks a sample of rows
against the exact fp64 SIMT kernel (bf_variant 0) and a few rows against the
CPU oracle.  Usage: python tools/bf_groundtruth.py [--n N] [--k K] [--out F]"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--k", type=int, default=20)
    ap.add_argument("--sample", type=int, default=1000)
    ap.add_argument("--oracle-rows", type=int, default=8)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch

    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200.engine import get_engine

    ds = km.generate_int_gmm(a.n, 128, 1000, 20.0, seed=7)
    eng = get_engine(0)
    # warm-up (library load, dataset upload, kernel attributes)
    km.brute_force_graph(ds, km.Metric.L2, a.k, member_ids=np.arange(4096))
    torch.cuda.synchronize()
    eng.reset_stats() if hasattr(eng, "reset_stats") else None
    t0 = time.perf_counter()
    g = km.brute_force_graph(ds, km.Metric.L2, a.k)
    t1 = time.perf_counter()
    route = eng.bf_route()
    rng = np.random.default_rng(0)
    rows = np.sort(rng.choice(a.n, a.sample, replace=False))
    eng.set_bf_variant(0)
    try:
        eng.set_dataset(ds.vectors, 1)
        eng.begin(np.arange(a.n, dtype=np.int64), np.zeros(a.n, dtype=np.int8), a.k)
        t2 = time.perf_counter()
        sid, sd = eng.bf_topk(a.k, rows=rows, exclude_self=True)
        t3 = time.perf_counter()
    finally:
        eng.set_bf_variant(-1)
    same = bool(np.array_equal(g.ids[rows], sid) and np.array_equal(g.dists[rows], sd))
    ok_oracle = None
    if a.oracle_rows:
        from oracle import oracle as O

        ok_oracle = True
        for r in rows[: a.oracle_rows]:
            d = O.pair_dists(ds.vectors, np.full(a.n, r, np.int32), np.arange(a.n, dtype=np.int32), 1)
            d[r] = np.inf
            order = np.lexsort((np.arange(a.n), d))[: a.k]
            ok_oracle &= bool(np.array_equal(g.ids[r], order) and np.array_equal(g.dists[r], d[order]))
    rec = {
        "n": a.n, "d": 128, "k": a.k, "route": "tcgen05 kind::i8" if route == 1 else "simt",
        "seconds": t1 - t0, "pairs": a.n * a.n, "gram_tops": 2.0 * a.n * a.n * 128 / (t1 - t0) / 1e12,
        "sample_rows": a.sample, "sample_equal_to_simt_fp64": same,
        "simt_seconds_for_sample": t3 - t2, "simt_projected_full_seconds": (t3 - t2) * a.n / a.sample,
        "oracle_rows_equal": ok_oracle, "oracle_rows": a.oracle_rows,
    }
    print(json.dumps(rec))
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
