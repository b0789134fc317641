"""Golden-vector cases: seeded input definitions shared by the generator
(make_golden.py, runs the reference) and the tests (oracle / CUDA path).

Shapes and value distributions follow BASELINE.json's configs at sizes the
CPU oracle finishes in seconds; config 1 is at full size.
"""

from __future__ import annotations

import numpy as np

CASES = {
    # BASELINE config 1 at full size: 2 x 5,000 points, d=32 U[0,1), k=20,
    # 10 iterations, min_update_fraction 0
    "c1_full": dict(op="smerge", data="uniform", n=10000, d=32, data_seed=1, metric=1, k=20,
                    split="halves", g_seed=1, h_seed=2, merge_seed=3,
                    mp=dict(max_iters=10, min_update_fraction=0.0)),
    # config-2 shape: integer GMM, d=128, k=20 (fp32-exact data)
    "c2_small": dict(op="smerge", data="intgmm", n=4000, d=128, centres=50, data_seed=7, metric=1,
                     k=20, split="perm", split_seed=1, g_seed=1, h_seed=2, merge_seed=3),
    # config-3 shape: J-Merge, d=960 GMM in [0,1]
    "c3_small": dict(op="jmerge", data="unitgmm", n=1600, d=960, centres=20, data_seed=7, metric=1,
                     k=20, split="perm", split_seed=2, g_seed=1, h_seed=2, merge_seed=5),
    # config-4 shape: cosine, unit-normalised GMM, d=100, k=40
    "c4_small": dict(op="smerge", data="sphere", n=3000, d=100, centres=40, data_seed=7, metric=2,
                     k=40, split="perm", split_seed=3, g_seed=1, h_seed=2, merge_seed=3),
    # L1 metric, J-Merge on uniform data
    "l1_jmerge": dict(op="jmerge", data="uniform", n=1500, d=6, data_seed=4, metric=0, k=8,
                      split="perm", split_seed=4, g_seed=1, h_seed=2, merge_seed=6),
    # NN-Descent (MODE_ALL), the builder of every config's subgraphs
    "nnd_uniform": dict(op="nnd", data="uniform", n=3000, d=16, data_seed=5, metric=1, k=12,
                        split="perm", split_seed=5, g_seed=9),
    # kept-ratio edge cases (test_merge.py:127-143)
    "r0": dict(op="smerge", data="uniform", n=500, d=4, data_seed=11, metric=1, k=10,
               split="perm", split_seed=4, g_seed=1, h_seed=2, merge_seed=5, mp=dict(r=0.0)),
    "r1": dict(op="smerge", data="uniform", n=500, d=4, data_seed=11, metric=1, k=10,
               split="perm", split_seed=4, g_seed=1, h_seed=2, merge_seed=5, mp=dict(r=1.0)),
    # singleton side, k1 = k-1 (test_merge.py:47-61)
    "singleton": dict(op="smerge", data="uniform", n=500, d=4, data_seed=11, metric=1, k=10,
                      split="last1", inputs="bruteforce", merge_seed=4, mp=dict(r=0.9)),
    # empty raw set round trip (test_merge.py:147-152)
    "jmerge_empty": dict(op="jmerge", data="uniform", n=500, d=4, data_seed=11, metric=1, k=8,
                         split="all", inputs="bruteforce", raw="empty", merge_seed=1),
    # exact 6-point known answer (test_merge.py:19-34)
    "six_points": dict(op="smerge", data="six", n=6, d=2, metric=1, k=2, split="first3",
                       inputs="bruteforce", merge_seed=0),
    # tiny hoods with short lists, r=0.3 (k1 rounding) and max_iters cut
    "tiny_r03": dict(op="smerge", data="uniform", n=60, d=3, data_seed=2, metric=1, k=4,
                     split="perm", split_seed=7, g_seed=3, h_seed=4, merge_seed=8,
                     mp=dict(r=0.3, max_iters=3)),
}


def make_data(spec) -> np.ndarray:
    kind = spec["data"]
    n, d = spec["n"], spec["d"]
    if kind == "six":
        return np.array([[0.0, 0.0], [1.0, 0.2], [0.4, 0.9],
                         [5.0, 5.0], [6.0, 5.2], [5.4, 5.9]], dtype=np.float32)
    rng = np.random.default_rng(spec.get("data_seed", 0))
    if kind == "uniform":  # core.py:200-205 generate_uniform
        return rng.random((n, d), dtype=np.float32)
    if kind == "intgmm":
        c = rng.uniform(0.0, 255.0, size=(spec["centres"], d)).astype(np.float32)
        x = c[rng.integers(0, spec["centres"], size=n)] + rng.standard_normal((n, d), dtype=np.float32) * np.float32(20.0)
        return np.rint(np.clip(x, 0.0, 255.0)).astype(np.float32)
    if kind == "unitgmm":
        c = rng.uniform(0.0, 1.0, size=(spec["centres"], d)).astype(np.float32)
        x = c[rng.integers(0, spec["centres"], size=n)] + rng.standard_normal((n, d), dtype=np.float32) * np.float32(0.05)
        return np.clip(x, 0.0, 1.0).astype(np.float32)
    if kind == "sphere":
        c = rng.standard_normal((spec["centres"], d)).astype(np.float32)
        x = c[rng.integers(0, spec["centres"], size=n)] + rng.standard_normal((n, d), dtype=np.float32) * np.float32(0.3)
        return (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)
    raise ValueError(kind)


def split(spec):
    n = spec["n"]
    how = spec["split"]
    if how == "halves":
        return np.arange(n // 2, dtype=np.int64), np.arange(n // 2, n, dtype=np.int64)
    if how == "perm":  # test_merge.py:11-15 split_ids
        rng = np.random.default_rng(spec["split_seed"])
        perm = rng.permutation(n)
        n1 = int(round(n * 0.5))
        return np.sort(perm[:n1]), np.sort(perm[n1:])
    if how == "last1":
        return np.arange(n - 1, dtype=np.int64), np.array([n - 1], dtype=np.int64)
    if how == "first3":
        return np.array([0, 1, 2], dtype=np.int64), np.array([3, 4, 5], dtype=np.int64)
    if how == "all":
        return np.arange(n, dtype=np.int64), np.array([], dtype=np.int64)
    raise ValueError(how)
