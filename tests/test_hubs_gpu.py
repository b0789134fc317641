"""Hub rows: data built so that a few points are the nearest neighbour of
hundreds of others (in-degree above the warp paths' limits: reverse
segments sorted by a block, memberships ranked by the sorted / block paths),
bit-exact against the CPU oracle on the u8 tensor-core route (integer data)
and on the exact route."""

import numpy as np
import pytest

from conftest import split_ids

pytestmark = pytest.mark.gpu


def _hub_data(shells, d=256, step=20, seed=0, jitter=False):
    """Hubs at integer points in [60, 195]^d; around hub h, shell points
    h +- step * e_i (axis directions, 2d of them at most): every shell point
    is `step` from its hub and step * sqrt(2) from its shell mates, so the
    hub is everyone's nearest neighbour."""
    rng = np.random.default_rng(seed)
    pts = []
    for size in shells:
        h = rng.integers(60, 196, size=d).astype(np.float32)
        pts.append(h)
        dirs = rng.permutation(2 * d)[:size]
        for q in dirs:
            p = h.copy()
            p[q % d] += step if q < d else -step
            pts.append(p)
    v = np.stack(pts).astype(np.float32)
    if jitter:  # non-integer data: the exact (fp64) route
        v = v + rng.random(v.shape, dtype=np.float32) * 0.25
    return v[rng.permutation(v.shape[0])]


def _graph(km, og):
    g = km.KnnGraph(og.member_ids, og.k, og.metric)
    g.ids, g.dists, g.sizes = og.ids.copy(), og.dists.copy(), og.sizes.copy()
    return g


@pytest.mark.parametrize("jitter", [False, True])
@pytest.mark.parametrize("op", ["s_merge", "j_merge", "nn_descent"])
def test_hub_rows_match_oracle(oracle, jitter, op):
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200.engine import get_engine

    eng = get_engine()
    eng.reset_stats()
    v = _hub_data([40, 130, 300, 400, 512, 31, 12], jitter=jitter, seed=3)
    ds = km.Dataset.from_dense(v)
    n, k = v.shape[0], 12
    s1, s2 = split_ids(n, seed=4)
    if op == "nn_descent":  # over all points: whole shells around each hub
        allm = np.arange(n, dtype=np.int64)
        g, rep = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=k), 3, member_ids=allm,
                               return_report=True)
        og, orep, _ = oracle.nn_descent(v, 1, k, 3, member_ids=allm)
    else:
        og1, _, _ = oracle.nn_descent(v, 1, k, 1, member_ids=s1)
        mp = km.MergeParams(k=k, seed=7)
        cnt = km.DistanceCounter()
        if op == "s_merge":
            og2, _, _ = oracle.nn_descent(v, 1, k, 2, member_ids=s2)
            g, rep = km.s_merge(ds, _graph(km, og1), _graph(km, og2), mp, counter=cnt,
                                return_report=True)
            og, orep, ocount = oracle.s_merge(v, og1, og2, k, seed=7)
        else:
            g, rep = km.j_merge(ds, _graph(km, og1), s2, mp, counter=cnt, return_report=True)
            og, orep, ocount = oracle.j_merge(v, og1, s2, k, seed=7)
        assert cnt.count == ocount
    assert np.array_equal(g.ids, og.ids)
    assert np.array_equal(g.dists, og.dists)
    assert np.array_equal(g.sizes, og.sizes)
    got = [(x.iteration, x.pairs, x.updates, x.phi, x.distance_count) for x in rep.rounds]
    want = [(x.iteration, x.pairs, x.updates, x.phi, x.distance_count) for x in orep.rounds]
    assert got == want
    # the data does what it is for: some row is the nearest neighbour of > 64
    # others, and the block paths (reverse segments > 256, > 256 memberships)
    # ran
    indeg = np.bincount(np.asarray(og.ids)[:, 0][np.asarray(og.sizes) > 0], minlength=og.n)
    assert indeg.max() > 64
    st = eng.stats()
    assert st["heavy_rev_rows"] > 0 and st["seg_hub_rows"] > 0, \
        {key: st[key] for key in ("heavy_rev_rows", "seg_hub_rows", "pairs", "rounds")}
