"""Randomised parity sweep: seeded random shapes, metrics, data kinds, kept
fractions r, sample rates rho and operations, each bit-exact against the
CPU oracle (graphs, per-round reports, distance counts)."""

import os

import numpy as np
import pytest

from conftest import split_ids

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = ["uniform", "intgmm", "sphere", "unitgmm"][rng.integers(0, 4)]
    metric = 2 if kind == "sphere" else int(rng.integers(0, 2))
    n = int(rng.integers(120, 3000))
    d = int(rng.choice([1, 3, 8, 17, 32, 64, 100, 130]))
    k = int(rng.integers(2, min(41, n // 4)))
    r = float(rng.choice([0.0, 0.3, 0.5, 1.0]))
    rho = float(rng.choice([1.0, 1.0, 0.5]))
    op = ["s_merge", "j_merge", "nn_descent"][rng.integers(0, 3)]
    return dict(kind=kind, metric=metric, n=n, d=d, k=k, r=r, rho=rho, op=op, seed=seed)


def _data(km, c):
    n, d, s = c["n"], c["d"], c["seed"] + 77
    if c["kind"] == "uniform":
        return km.generate_uniform(n, d, seed=s)
    if c["kind"] == "intgmm":
        return km.generate_int_gmm(n, d, n_centres=10, seed=s)
    if c["kind"] == "unitgmm":
        return km.generate_unit_gmm(n, d, n_centres=10, seed=s)
    return km.generate_sphere_gmm(n, d, n_centres=10, seed=s)


def _graph(km, og):
    g = km.KnnGraph(og.member_ids, og.k, og.metric)
    g.ids, g.dists, g.sizes = og.ids.copy(), og.dists.copy(), og.sizes.copy()
    return g


# KNNM_SWEEP_OFFSET shifts the 64 seeds (extra sweeps without new code)
_OFF = int(os.environ.get("KNNM_SWEEP_OFFSET", "0"))


@pytest.mark.parametrize("seed", range(_OFF, _OFF + 64))
def test_random_case_matches_oracle(oracle, seed):
    import paper_1908_00814_b200 as km

    c = _case(seed)
    ds = _data(km, c)
    n, k, metric, rho = c["n"], c["k"], c["metric"], c["rho"]
    s1, s2 = split_ids(n, seed=seed + 5)
    if c["op"] == "nn_descent":
        g, rep = km.nn_descent(ds, metric, km.DescentParams(k=k, rho=rho), 3, member_ids=s1,
                               return_report=True)
        og, orep, _ = oracle.nn_descent(ds.vectors, metric, k, 3, member_ids=s1, rho=rho)
    else:
        og1, _, _ = oracle.nn_descent(ds.vectors, metric, k, 1, member_ids=s1)
        mp = km.MergeParams(k=k, r=c["r"], seed=seed, rho=rho)
        cnt = km.DistanceCounter()
        if c["op"] == "s_merge":
            og2, _, _ = oracle.nn_descent(ds.vectors, metric, k, 2, member_ids=s2)
            g, rep = km.s_merge(ds, _graph(km, og1), _graph(km, og2), mp, counter=cnt, return_report=True)
            og, orep, ocount = oracle.s_merge(ds.vectors, og1, og2, k, r=c["r"], seed=seed, rho=rho)
        else:
            g, rep = km.j_merge(ds, _graph(km, og1), s2, mp, counter=cnt, return_report=True)
            og, orep, ocount = oracle.j_merge(ds.vectors, og1, s2, k, r=c["r"], seed=seed, rho=rho)
        assert cnt.count == ocount, c
    assert np.array_equal(np.asarray(g.member_ids), np.asarray(og.member_ids)), c
    assert np.array_equal(g.sizes, og.sizes), c
    assert np.array_equal(g.ids, og.ids), c
    assert np.array_equal(g.dists, og.dists), c
    got = [(x.iteration, x.pairs, x.updates, x.phi, x.distance_count) for x in rep.rounds]
    want = [(x.iteration, x.pairs, x.updates, x.phi, x.distance_count) for x in orep.rounds]
    assert got == want, c
