"""Host-side logic of the drop-in package (no GPU needed)."""

import numpy as np
import pytest

import paper_1908_00814_b200 as km
from paper_1908_00814_b200 import merge as M


def test_merge_params_validation():
    with pytest.raises(ValueError, match="r must be"):
        km.MergeParams(k=8, r=1.5)
    with pytest.raises(ValueError, match="k must be"):
        km.MergeParams(k=1)
    assert km.MergeParams(k=20, r=0.5).k1 == 10
    assert km.MergeParams(k=10, r=0.25).k1 == 2  # banker's rounding like the reference
    assert km.MergeParams(k=4, r=0.3).k1 == 1


@pytest.mark.parametrize("seed", range(5))
def test_merge_members_matches_union1d(seed):
    rng = np.random.default_rng(seed)
    perm = rng.permutation(1000 + seed * 17)
    a, b = np.sort(perm[:400]), np.sort(perm[400:])
    u, ra, rb = M._merge_members(a, b)
    assert np.array_equal(u, np.union1d(a, b))
    assert np.array_equal(ra, np.searchsorted(u, a))
    assert np.array_equal(rb, np.searchsorted(u, b))
    assert not M._overlaps(a, b)
    assert M._overlaps(a, np.sort(np.concatenate((b[:3], a[:1]))))


def test_check_merge_inputs_messages():
    ds = km.generate_uniform(50, 3, seed=1)
    g = km.KnnGraph(np.arange(25), 4, km.Metric.L2)
    h = km.KnnGraph(np.arange(20, 50), 4, km.Metric.L2)
    with pytest.raises(ValueError, match="disjoint"):
        M._check_merge_inputs(ds, g, h.member_ids, km.MergeParams(k=4), h)
    h2 = km.KnnGraph(np.arange(25, 50), 4, km.Metric.L2)
    with pytest.raises(ValueError, match="params.k"):
        M._check_merge_inputs(ds, g, h2.member_ids, km.MergeParams(k=6), h2)
    with pytest.raises(ValueError, match="outside"):
        M._check_merge_inputs(ds, g, np.array([60]), km.MergeParams(k=4), None)


def test_split_and_validate(oracle):
    vec = km.generate_uniform(300, 4, seed=3).vectors
    og = oracle.brute_force_graph(vec, 1, 8)
    g = km.KnnGraph.from_arrays(og.member_ids, 8, km.Metric.L2, og.ids, og.dists, og.sizes)
    g.validate()
    parts = km.split(g, 3)
    assert parts.head.k == 3 and parts.tail.k == 5
    assert np.array_equal(np.concatenate([parts.head.ids, parts.tail.ids], axis=1), g.ids)
    parts.head.validate()


def test_scalar_distance_bit_identical_to_oracle(oracle):
    rng = np.random.default_rng(0)
    c = km.DistanceCounter()
    for metric in (0, 1, 2):
        for _ in range(50):
            a = rng.standard_normal(37).astype(np.float32)
            b = rng.standard_normal(37).astype(np.float32)
            assert km.distance(metric, a, b, c) == oracle.dense_dist(a, b, metric)
    assert c.count == 150
    z = np.zeros(4, dtype=np.float32)
    assert km.distance(km.Metric.COSINE, z, z, c) == 0.0
    assert km.distance(km.Metric.COSINE, z, np.ones(4, np.float32), c) == 1.0
    assert km.distance(km.Metric.L2, np.array([0, 0], np.float32), np.array([3, 4], np.float32), c) == 25.0


def test_update_nn_spec():
    nl = km.NeighborList(3, owner=0)
    assert km.update_nn(nl, 5, 2.0)
    assert km.update_nn(nl, 4, 2.0)  # tie: smaller id first
    assert nl.ids() == [4, 5]
    assert not km.update_nn(nl, 5, 1.0)  # duplicate id
    assert km.update_nn(nl, 7, 3.0)
    assert not km.update_nn(nl, 8, 3.0)  # full and not strictly closer
    assert km.update_nn(nl, 9, 0.5)
    assert nl.ids() == [9, 4, 5]


def test_recall_helpers():
    truth = [[1, 2, 3], [4, 5, 6]]
    assert km.recall_at_k([[1, 2, 9], [6, 5, 4]], truth, 3) == 5 / 6
    assert km.recall_at_k_arrays(np.array([[1, 2, 9], [6, 5, 4]]), np.array(truth), 3) == 5 / 6
    assert km.scanning_rate(45, 10) == 1.0


def test_generators_shapes_and_certificates():
    ds = km.generate_int_gmm(500, 128, n_centres=10, seed=1)
    assert ds.vectors.dtype == np.float32 and np.all(ds.vectors == np.rint(ds.vectors))
    assert ds.vectors.min() >= 0 and ds.vectors.max() <= 255
    s = km.generate_sphere_gmm(200, 100, n_centres=5, seed=1)
    assert np.allclose(np.linalg.norm(s.vectors, axis=1), 1.0, atol=1e-5)
    u = km.generate_unit_gmm(100, 960, n_centres=5, seed=1)
    assert u.vectors.min() >= 0 and u.vectors.max() <= 1


def test_pcg_state_handoff_matches_numpy():
    """_pcg_consume advances numpy's PCG64 exactly as next_uint32 calls do."""
    from paper_1908_00814_b200.engine import _pcg_consume

    for seed in range(6):
        a = np.random.default_rng(seed)
        a.integers(0, 5, size=seed)  # vary the half-buffer
        b = np.random.default_rng(seed)
        b.integers(0, 5, size=seed)
        st = b.bit_generator.state
        n = 17 + seed
        a.integers(0, 2**32 - 1, size=n, dtype=np.uint64)  # one next_uint32 per draw (no rejection at 2^32-1)
        _pcg_consume(b, st, n)
        assert a.bit_generator.state == b.bit_generator.state


@pytest.mark.parametrize("n,k", [(1_000_000, 20), (500, 10), (12000, 300), (60, 40), (20001, 800)])
def test_native_sample_distinct_rows_matches_numpy(n, k):
    """Native Generator.choice restatement == the reference's per-row
    sample_distinct loop (core.py:222-230), values and final rng state."""
    from paper_1908_00814_b200.core import sample_distinct, sample_distinct_rows

    rows = np.random.default_rng(9).choice(n, size=min(n, 300), replace=False).astype(np.int32)
    a = np.random.default_rng(n + k)
    a.integers(0, 3, size=1)
    b = np.random.default_rng(n + k)
    b.integers(0, 3, size=1)
    want = np.stack([sample_distinct(a, n, k, exclude=int(r)) for r in rows])
    got = sample_distinct_rows(b, n, k, rows)
    assert np.array_equal(got, want)
    assert a.bit_generator.state == b.bit_generator.state


@pytest.mark.parametrize("a,b", [([1, 3, 5], [2, 3, 9]), ([], [4, 5]), ([7], []), ([1, 2], [3, 4]),
                                 ([3, 4], [1, 2]), ([], [])])
def test_native_merge_members(a, b):
    """Union + rows (np.union1d + searchsorted, merge.py:217-221) and the
    shared-id flag from the native linear merge."""
    from paper_1908_00814_b200.merge import _merge_members

    a = np.array(a, dtype=np.int64)
    b = np.array(b, dtype=np.int64)
    u, ra, rb, shared = _merge_members(a, b, with_overlap=True)
    want = np.union1d(a, b)
    assert np.array_equal(u, want)
    assert np.array_equal(ra, np.searchsorted(want, a))
    assert np.array_equal(rb, np.searchsorted(want, b))
    assert shared == bool(np.intersect1d(a, b).size)


def test_native_merge_members_large():
    from paper_1908_00814_b200.merge import _merge_members

    perm = np.random.default_rng(3).permutation(200_000)
    a, b = np.sort(perm[:90_000]).astype(np.int64), np.sort(perm[90_000:]).astype(np.int64)
    u, ra, rb = _merge_members(a, b)
    assert np.array_equal(u, np.union1d(a, b))
    assert np.array_equal(u[ra], a) and np.array_equal(u[rb], b)


@pytest.mark.parametrize("n,split,shared", [(200_000, 90_000, False), (300_001, 1, False),
                                            (150_000, 149_999, False), (200_000, 100_000, True)])
def test_native_merge_members_parallel_labels(n, split, shared):
    """The merge-path split over host threads (inputs >= 64K ids) gives the
    serial result, plus the merge labels (1 = from b); a shared id falls
    back to the serial tie semantics."""
    from paper_1908_00814_b200.merge import _merge_members

    perm = np.random.default_rng(n + split).permutation(n)
    a, b = np.sort(perm[:split]).astype(np.int64), np.sort(perm[split:]).astype(np.int64)
    if shared:
        b = np.sort(np.concatenate((b, a[[5, len(a) // 2]])))
    labs = []
    u, ra, rb, sh = _merge_members(a, b, with_overlap=True, labels_out=labs)
    want = np.union1d(a, b)
    assert sh == shared
    assert np.array_equal(u, want)
    assert np.array_equal(ra, np.searchsorted(want, a))
    assert np.array_equal(rb, np.searchsorted(want, b))
    if not shared:
        lab = np.zeros(want.size, dtype=np.int8)
        lab[rb] = 1
        assert len(labs) == 1 and np.array_equal(labs[0], lab)
    else:
        assert labs == []


@pytest.mark.parametrize("n,k,nrows,pre", [(1_000_000, 20, 6000, 1), (1_000_000, 20, 6000, 2),
                                           (8000, 40, 5000, 0), (3_000_000_000, 20, 4500, 3),
                                           (70_000, 1, 4200, 1)])
def test_parallel_sample_distinct_rows_matches_numpy(n, k, nrows, pre):
    """The parallel path of the per-row choice loop (>= 4096 rows: PCG64
    words by jump-ahead, rejection scan, rows on threads) == numpy's
    sequential per-row Generator.choice, values and final state; covers
    both half-buffer states, Floyd and tail-shuffle rows, rows without an
    exclusion and populations near 2^32 (frequent Lemire rejections)."""
    from paper_1908_00814_b200.core import sample_distinct, sample_distinct_rows

    g = np.random.default_rng(n % 997)
    rows = g.integers(-1, min(n, 2**31 - 1), size=nrows).astype(np.int32)
    a = np.random.default_rng(nrows + k)
    a.integers(0, 3, size=pre)
    b = np.random.default_rng(nrows + k)
    b.integers(0, 3, size=pre)
    want = np.stack([sample_distinct(a, n, k, exclude=int(r)) for r in rows])
    got = sample_distinct_rows(b, n, k, rows)
    assert np.array_equal(got, want)
    assert a.bit_generator.state == b.bit_generator.state


def test_from_arrays_flags_materialise_on_access():
    """KnnGraph.from_arrays without flags: all False, created on first access
    (reference layout, graph.py:96); explicit flags and assignment are kept."""
    import paper_1908_00814_b200 as km

    ids = np.arange(12, dtype=np.int32).reshape(4, 3)
    dists = np.arange(12, dtype=np.float64).reshape(4, 3)
    sizes = np.full(4, 3, dtype=np.int32)
    g = km.KnnGraph.from_arrays(np.arange(4), 3, km.Metric.L2, ids, dists, sizes)
    assert g._flags is None
    assert g.flags.shape == (4, 3) and g.flags.dtype == np.bool_ and not g.flags.any()
    assert g.flags is g.flags  # one array, not a fresh one per access
    g.flags[1, 2] = True
    assert g.flags[1, 2]
    h = g.with_capacity(5)
    assert h.flags.shape == (4, 5) and h.flags[1, 2] and h.flags.sum() == 1
    f = np.ones((4, 3), dtype=np.bool_)
    g2 = km.KnnGraph.from_arrays(np.arange(4), 3, km.Metric.L2, ids, dists, sizes, flags=f)
    assert g2.flags is f
    g2.flags = ~f
    assert not g2.flags.any()
