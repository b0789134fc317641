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


# -- tensor-core route (tcgen05 kind::i8 Gram tiles; knnm_bf.cuh) -----------
# Certified u8 data (integers in [0, 255], L2): exact integer distances, so
# the lists must equal the oracle's bf_graph_dense bit for bit.  Shapes cover
# rows shorter than one 128-byte K block (TMA zero fill), two K blocks with a
# ragged tail, candidate counts that are not multiples of the 256-row tile,
# query counts that are not multiples of the 128-query block, data slices
# (few queries), k up to 32, and heavy distance ties (few distinct points).

TC_CASES = [
    # n, d, members, k, centres
    (700, 32, 500, 10, 5),
    (3000, 128, 2900, 20, 40),
    (1200, 200, 1100, 32, 10),
    (300, 128, 129, 1, 3),
    (2600, 64, 2600, 16, 2),
]


@pytest.mark.parametrize("n,d,m,k,cent", TC_CASES)
def test_tensor_core_brute_force_graph_matches_oracle(oracle, n, d, m, k, cent):
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200.engine import get_engine

    ds = km.generate_int_gmm(n, d, n_centres=cent, seed=n + d)
    if cent == 2:  # many exact duplicates: ties broken by id
        ds = km.Dataset.from_dense(np.repeat(ds.vectors[:50], n // 50 + 1, axis=0)[:n].copy())
    members = np.sort(np.random.default_rng(k).choice(n, m, replace=False))
    c = km.DistanceCounter()
    g = km.brute_force_graph(ds, km.Metric.L2, k, member_ids=members, counter=c)
    assert get_engine(None).bf_route() == 1, "certified u8 data must take the tensor-core route"
    og = oracle.brute_force_graph(ds.vectors, 1, k, member_ids=members)
    assert np.array_equal(g.ids, og.ids)
    assert np.array_equal(g.dists, og.dists)
    assert np.array_equal(g.sizes, og.sizes)
    assert c.count == m * (m - 1) // 2


def test_tensor_core_queries_and_fallback(oracle):
    """Vector queries: integer queries take the tensor cores, fractional ones
    the exact SIMT kernel; both equal the reference order (dist, id)."""
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200.engine import get_engine

    ds = km.generate_int_gmm(5000, 128, n_centres=30, seed=2)
    qi = km.generate_int_gmm(333, 128, n_centres=30, seed=3).vectors
    qf = qi + np.float32(0.25)
    eng = get_engine(None)
    for q, route in ((qi, 1), (qf, 0)):
        ids, dists = km.brute_force_queries(ds, km.Metric.L2, km.Dataset.from_dense(q), 20)
        assert eng.bf_route() == route
        for t in range(0, q.shape[0], 37):
            d = oracle.pair_dists(np.vstack([ds.vectors, q[t:t + 1]]), np.full(ds.n, ds.n, np.int32),
                                  np.arange(ds.n, dtype=np.int32), 1)
            order = np.lexsort((np.arange(ds.n), d))[:20]
            assert np.array_equal(ids[t], order)
            assert np.array_equal(dists[t], d[order])
    # forcing the SIMT kernel gives the same lists on certified data
    eng.set_bf_variant(0)
    try:
        ids0, d0 = km.brute_force_queries(ds, km.Metric.L2, km.Dataset.from_dense(qi), 20)
    finally:
        eng.set_bf_variant(-1)
    ids1, d1 = km.brute_force_queries(ds, km.Metric.L2, km.Dataset.from_dense(qi), 20)
    assert np.array_equal(ids0, ids1) and np.array_equal(d0, d1)


def test_brute_force_graph_on_pair_matches_reference_order(oracle):
    """on_pair (construct.py:296-312): every pair (i < j), j-major, with the
    exact scalar distance; the graph equals the fast route's."""
    import paper_1908_00814_b200 as km

    ds = km.generate_uniform(90, 7, seed=4)
    members = np.arange(3, 90, 1)
    got = []
    c = km.DistanceCounter()
    g = km.brute_force_graph(ds, km.Metric.L2, 6, member_ids=members, counter=c,
                             on_pair=lambda a, b, d: got.append((a, b, d)))
    want = [(int(members[i]), int(members[j]), oracle.dense_dist(ds.vectors[members[i]], ds.vectors[members[j]], 1))
            for j in range(members.size) for i in range(j)]
    assert got == want
    assert c.count == len(want)
    g2 = km.brute_force_graph(ds, km.Metric.L2, 6, member_ids=members)
    assert np.array_equal(g.ids, g2.ids) and np.array_equal(g.dists, g2.dists)
