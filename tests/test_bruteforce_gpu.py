"""GPU exact brute force (construct.py:273-348) vs the CPU oracle's
restatement of bf_graph_dense / bf_queries_dense, bit-exact."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("metric,kind", [(1, "uniform"), (2, "sphere"), (0, "uniform"), (1, "intgmm")])
def test_brute_force_graph_matches_oracle(oracle, metric, kind):
    import paper_1908_00814_b200 as km

    ds = {"uniform": lambda: km.generate_uniform(700, 9, seed=3),
          "sphere": lambda: km.generate_sphere_gmm(700, 20, n_centres=7, seed=3),
          "intgmm": lambda: km.generate_int_gmm(700, 32, n_centres=5, seed=3)}[kind]()
    members = np.sort(np.random.default_rng(1).choice(700, 500, replace=False))
    c = km.DistanceCounter()
    g = km.brute_force_graph(ds, metric, 10, member_ids=members, counter=c)
    og = oracle.brute_force_graph(ds.vectors, metric, 10, member_ids=members)
    assert np.array_equal(g.ids, og.ids)
    assert np.array_equal(g.dists, og.dists)
    assert np.array_equal(g.sizes, og.sizes)
    assert c.count == 500 * 499 // 2
    g.validate()


def test_brute_force_queries_matches_reference_semantics(oracle):
    import paper_1908_00814_b200 as km

    ds = km.generate_uniform(3000, 12, seed=5)
    q = km.Dataset.from_dense(km.generate_uniform(40, 12, seed=6).vectors)
    ids, dists = km.brute_force_queries(ds, km.Metric.L2, q, 15)
    assert ids.dtype == np.int64
    for t in range(q.n):
        d = oracle.pair_dists(ds.vectors, np.full(ds.n, 0, np.int32), np.arange(ds.n, dtype=np.int32), 1)
        d = np.array([oracle.dense_dist(q.vectors[t], ds.vectors[i], 1) for i in range(ds.n)])
        order = np.lexsort((np.arange(ds.n), d))[:15]
        assert np.array_equal(ids[t], order)
        assert np.array_equal(dists[t], d[order])
