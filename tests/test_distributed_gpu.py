"""Sharded (multi-rank) merges on one GPU: P virtual ranks in one process
(LoopbackComm), each with its own engine context, run the full id-sharded
protocol -- per-rank reverse/hoods/join, all-to-all of reference-order slot
blocks, per-owner apply, all-gather -- and must be bit-identical to the
single-GPU merge (and so to the reference)."""

import numpy as np
import pytest

from conftest import split_ids

pytestmark = pytest.mark.gpu


def _engines(world):
    from paper_1908_00814_b200.engine import Engine

    return {r: Engine(0) for r in range(world)}


@pytest.mark.parametrize("world", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["intgmm", "uniform"])
def test_sharded_s_merge_bit_identical(oracle, world, kind):
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import distributed as D

    n = 3000
    ds = (km.generate_int_gmm(n, 128, n_centres=30, seed=3) if kind == "intgmm"
          else km.generate_uniform(n, 16, seed=3))
    s1, s2 = split_ids(n, seed=2)
    g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=12), 1, member_ids=s1)
    h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=12), 2, member_ids=s2)
    mp = km.MergeParams(k=12, seed=5)
    c1 = km.DistanceCounter()
    want, rep_w = km.s_merge(ds, g, h, mp, counter=c1, return_report=True)
    c2 = km.DistanceCounter()
    got, rep_g = D.s_merge_sharded(ds, g, h, mp, D.LoopbackComm(world), _engines(world),
                                   counter=c2, return_report=True)
    assert np.array_equal(got.ids, want.ids)
    assert np.array_equal(got.dists, want.dists)
    assert np.array_equal(got.sizes, want.sizes)
    assert c1.count == c2.count
    assert [(r.pairs, r.updates, r.phi) for r in rep_g.rounds] == \
        [(r.pairs, r.updates, r.phi) for r in rep_w.rounds]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_j_merge_bit_identical(oracle, world):
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import distributed as D

    ds = km.generate_sphere_gmm(2500, 100, n_centres=20, seed=4)
    s1, s2 = split_ids(2500, seed=8)
    g = km.nn_descent(ds, km.Metric.COSINE, km.DescentParams(k=16), 1, member_ids=s1)
    mp = km.MergeParams(k=16, seed=7)
    want, rep_w = km.j_merge(ds, g, s2, mp, return_report=True)
    got, rep_g = D.j_merge_sharded(ds, g, s2, mp, D.LoopbackComm(world), _engines(world),
                                   return_report=True)
    assert np.array_equal(got.ids, want.ids)
    assert np.array_equal(got.dists, want.dists)
    assert [(r.pairs, r.updates, r.phi) for r in rep_g.rounds] == \
        [(r.pairs, r.updates, r.phi) for r in rep_w.rounds]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_rho_sampling_bit_identical(oracle, world):
    """rho = 0.5 sampling is deterministic per (round seed, row): every rank
    samples all rows identically, so sharded == single-GPU."""
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import distributed as D

    n = 3000
    ds = km.generate_int_gmm(n, 128, n_centres=30, seed=5)
    s1, s2 = split_ids(n, seed=3)
    g = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=16), 1, member_ids=s1)
    h = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=16), 2, member_ids=s2)
    mp = km.MergeParams(k=16, seed=9, rho=0.5)
    want, rep_w = km.s_merge(ds, g, h, mp, return_report=True)
    got, rep_g = D.s_merge_sharded(ds, g, h, mp, D.LoopbackComm(world), _engines(world),
                                   return_report=True)
    assert np.array_equal(got.ids, want.ids)
    assert np.array_equal(got.dists, want.dists)
    assert [(r.pairs, r.updates, r.phi) for r in rep_g.rounds] == \
        [(r.pairs, r.updates, r.phi) for r in rep_w.rounds]


@pytest.mark.parametrize("seed", range(12))
def test_sharded_random_cases(seed):
    """Random shapes / metrics / r / rho / world sizes: sharded == single GPU."""
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import distributed as D

    rng = np.random.default_rng(500 + seed)
    world = int(rng.integers(2, 5))
    n = int(rng.integers(400, 3000))
    kind = ["uniform", "intgmm", "sphere"][rng.integers(0, 3)]
    d = int(rng.choice([4, 16, 64, 100]))
    metric = km.Metric.COSINE if kind == "sphere" else km.Metric(int(rng.integers(0, 2)))
    k = int(rng.integers(4, 24))
    ds = (km.generate_uniform(n, d, seed=seed) if kind == "uniform"
          else km.generate_int_gmm(n, d, n_centres=12, seed=seed) if kind == "intgmm"
          else km.generate_sphere_gmm(n, d, n_centres=12, seed=seed))
    s1, s2 = split_ids(n, seed=seed + 1)
    mp = km.MergeParams(k=k, r=float(rng.choice([0.0, 0.5, 1.0])), seed=seed,
                        rho=float(rng.choice([1.0, 0.5])))
    g = km.nn_descent(ds, metric, km.DescentParams(k=k), 1, member_ids=s1)
    if rng.integers(0, 2):
        h = km.nn_descent(ds, metric, km.DescentParams(k=k), 2, member_ids=s2)
        want, rw = km.s_merge(ds, g, h, mp, return_report=True)
        got, rg = D.s_merge_sharded(ds, g, h, mp, D.LoopbackComm(world), _engines(world),
                                    return_report=True)
    else:
        want, rw = km.j_merge(ds, g, s2, mp, return_report=True)
        got, rg = D.j_merge_sharded(ds, g, s2, mp, D.LoopbackComm(world), _engines(world),
                                    return_report=True)
    assert np.array_equal(got.ids, want.ids)
    assert np.array_equal(got.dists, want.dists)
    assert np.array_equal(got.sizes, want.sizes)
    assert [(r.pairs, r.updates, r.phi) for r in rg.rounds] == \
        [(r.pairs, r.updates, r.phi) for r in rw.rounds]


@pytest.mark.parametrize("kind,metric", [("intgmm", "l2"), ("uniform", "l2"), ("sphere", "cos")])
def test_compacted_exchange_bit_identical(oracle, kind, metric):
    """Exchanging only the written slots (knnm_local_compact) gives the same
    merge as exchanging whole slot blocks, with less traffic."""
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import distributed as D

    n = 3000
    ds = {"intgmm": lambda: km.generate_int_gmm(n, 128, n_centres=30, seed=6),
          "uniform": lambda: km.generate_uniform(n, 24, seed=6),
          "sphere": lambda: km.generate_sphere_gmm(n, 100, n_centres=20, seed=6)}[kind]()
    m = km.Metric.L2 if metric == "l2" else km.Metric.COSINE
    s1, s2 = split_ids(n, seed=4)
    g = km.nn_descent(ds, m, km.DescentParams(k=12), 1, member_ids=s1)
    h = km.nn_descent(ds, m, km.DescentParams(k=12), 2, member_ids=s2)
    mp = km.MergeParams(k=12, seed=3)
    want = km.s_merge(ds, g, h, mp)
    out = {}
    for compact in (False, True):
        tr = {}
        got = D.s_merge_sharded(ds, g, h, mp, D.LoopbackComm(3), _engines(3), compact=compact,
                                traffic=tr)
        assert np.array_equal(got.ids, want.ids)
        assert np.array_equal(got.dists, want.dists)
        assert np.array_equal(got.sizes, want.sizes)
        out[compact] = sum(tr.values())
    assert 0 < out[True] < out[False]
    # j_merge over the compacted exchange
    wj = km.j_merge(ds, g, s2, mp)
    gj = D.j_merge_sharded(ds, g, s2, mp, D.LoopbackComm(2), _engines(2))
    assert np.array_equal(gj.ids, wj.ids) and np.array_equal(gj.dists, wj.dists)
