"""GPU parity: the CUDA path through the C-ABI against the CPU oracle.

Bit-exact on ids, dists, sizes, the distance counter and every per-round
report field (pairs, updates, phi), because the oracle restates the
reference arithmetic exactly and the device path replays the reference's
per-row insertion order.
"""

import numpy as np
import pytest

from conftest import split_ids

pytestmark = pytest.mark.gpu


def _km():
    import paper_1908_00814_b200 as km

    return km


def _same_graph(a, b):
    assert np.array_equal(np.asarray(a.member_ids), np.asarray(b.member_ids))
    assert np.array_equal(a.sizes, b.sizes)
    assert np.array_equal(a.ids, b.ids)
    assert np.array_equal(a.dists, b.dists)


def _same_report(rep, orep):
    assert rep.phi_initial == orep.phi_initial
    got = [(r.iteration, r.pairs, r.updates, r.phi, r.distance_count) for r in rep.rounds]
    want = [(r.iteration, r.pairs, r.updates, r.phi, r.distance_count) for r in orep.rounds]
    assert got == want
    assert rep.converged == orep.converged


CASES = [
    # n, d, k, metric, data kind
    (600, 4, 8, 1, "uniform"),
    (3000, 16, 10, 1, "uniform"),
    (2000, 12, 12, 2, "uniform"),
    (4000, 32, 20, 1, "uniform"),
    (3000, 8, 40, 1, "uniform"),
    (6000, 128, 20, 1, "intgmm"),
    (3000, 100, 40, 2, "sphere"),
    (2000, 960, 20, 1, "unitgmm"),
    (1500, 5, 6, 0, "uniform"),
    (5000, 100, 40, 1, "intgmm"),
    (2500, 70, 16, 0, "uniform"),  # L1, non-certified, ragged 32-dim blocks
    (1500, 400, 10, 2, "sphere"),  # d > 384: exact evaluation deferred to the apply
    (1500, 420, 12, 0, "uniform"),
]


def _data(km, n, d, kind, seed):
    if kind == "uniform":
        return km.generate_uniform(n, d, seed=seed)
    if kind == "intgmm":
        return km.generate_int_gmm(n, d, n_centres=50, seed=seed)
    if kind == "unitgmm":
        return km.generate_unit_gmm(n, d, n_centres=20, seed=seed)
    return km.generate_sphere_gmm(n, d, n_centres=40, seed=seed)


@pytest.mark.parametrize("n,d,k,metric,kind", CASES)
def test_nn_descent_matches_oracle(oracle, n, d, k, metric, kind):
    km = _km()
    ds = _data(km, n, d, kind, seed=n + d)
    s1, _ = split_ids(n, seed=1)
    g, rep = km.nn_descent(ds, metric, km.DescentParams(k=k), 1, member_ids=s1,
                           return_report=True)
    og, orep, ocount = oracle.nn_descent(ds.vectors, metric, k, 1, member_ids=s1)
    _same_graph(g, og)
    _same_report(rep, orep)


@pytest.mark.parametrize("n,d,k,metric,kind", CASES)
def test_s_merge_matches_oracle(oracle, n, d, k, metric, kind):
    km = _km()
    ds = _data(km, n, d, kind, seed=n + d)
    s1, s2 = split_ids(n, seed=2)
    g, _, _ = oracle.nn_descent(ds.vectors, metric, k, 1, member_ids=s1)
    h, _, _ = oracle.nn_descent(ds.vectors, metric, k, 2, member_ids=s2)
    gg = _to_graph(km, g)
    hh = _to_graph(km, h)
    c = km.DistanceCounter()
    u, rep = km.s_merge(ds, gg, hh, km.MergeParams(k=k, seed=3), counter=c, return_report=True)
    ou, orep, ocount = oracle.s_merge(ds.vectors, g, h, k, seed=3)
    _same_graph(u, ou)
    _same_report(rep, orep)
    assert c.count == ocount


@pytest.mark.parametrize("n,d,k,metric,kind", CASES)
def test_j_merge_matches_oracle(oracle, n, d, k, metric, kind):
    km = _km()
    ds = _data(km, n, d, kind, seed=n + d)
    s1, s2 = split_ids(n, seed=4)
    g, _, _ = oracle.nn_descent(ds.vectors, metric, k, 1, member_ids=s1)
    c = km.DistanceCounter()
    u, rep = km.j_merge(ds, _to_graph(km, g), s2, km.MergeParams(k=k, seed=5), counter=c,
                        return_report=True)
    ou, orep, ocount = oracle.j_merge(ds.vectors, g, s2, k, seed=5)
    _same_graph(u, ou)
    _same_report(rep, orep)
    assert c.count == ocount


def _to_graph(km, og):
    g = km.KnnGraph(og.member_ids, og.k, og.metric)
    g.ids = og.ids.copy()
    g.dists = og.dists.copy()
    g.sizes = og.sizes.copy()
    return g


@pytest.mark.parametrize("variant", [0, 1, 2, 4])
@pytest.mark.parametrize("n,d,k,metric,kind", [CASES[1], CASES[5], CASES[6], CASES[8]])
def test_join_variants_agree(oracle, variant, n, d, k, metric, kind):
    """Both local-join routes (fp64-every-pair / fp32-screen tiled) are
    bit-identical to the oracle."""
    km = _km()
    from paper_1908_00814_b200.engine import get_engine

    eng = get_engine()
    ds = _data(km, n, d, kind, seed=n + d + 1)
    s1, s2 = split_ids(n, seed=7)
    g, _, _ = oracle.nn_descent(ds.vectors, metric, k, 1, member_ids=s1)
    h, _, _ = oracle.nn_descent(ds.vectors, metric, k, 2, member_ids=s2)
    eng.set_join_variant(variant)
    try:
        u, rep = km.s_merge(ds, _to_graph(km, g), _to_graph(km, h), km.MergeParams(k=k, seed=9),
                            return_report=True)
    finally:
        eng.set_join_variant(-1)
    ou, orep, _ = oracle.s_merge(ds.vectors, g, h, k, seed=9)
    _same_graph(u, ou)
    _same_report(rep, orep)


def test_certificate_detection():
    km = _km()
    from paper_1908_00814_b200.engine import get_engine

    eng = get_engine()
    eng.set_dataset(km.generate_int_gmm(1000, 128, n_centres=10, seed=1).vectors, 1)
    assert eng.info()["cert"] and eng.info()["cert_dot"]
    eng.set_dataset(km.generate_int_gmm(1000, 256, n_centres=10, seed=1).vectors, 1)
    assert eng.info()["cert"] and not eng.info()["cert_dot"]  # 2*d*255^2 >= 2^24
    eng.set_dataset(km.generate_uniform(1000, 16, seed=1).vectors, 1)
    assert not eng.info()["cert"]
    eng.set_dataset(km.generate_int_gmm(1000, 128, n_centres=10, seed=1).vectors, 2)
    assert not eng.info()["cert"]  # cosine is never certified


@pytest.mark.parametrize("u8", [True, False])
def test_tensor_core_routes_u8_and_fp16(oracle, u8):
    """Integer data in [0,255]: the u8 (s32 MMA) and fp16 (f32 MMA) tensor-core
    routes are both bit-identical to the oracle."""
    km = _km()
    from paper_1908_00814_b200.engine import get_engine

    eng = get_engine()
    ds = km.generate_int_gmm(5000, 128, n_centres=40, seed=21)
    s1, s2 = split_ids(5000, seed=3)
    g, _, _ = oracle.nn_descent(ds.vectors, 1, 20, 1, member_ids=s1)
    h, _, _ = oracle.nn_descent(ds.vectors, 1, 20, 2, member_ids=s2)
    eng.set_u8(u8)
    try:
        u, rep = km.s_merge(ds, _to_graph(km, g), _to_graph(km, h), km.MergeParams(k=20, seed=4),
                            return_report=True)
        info = eng.info()
    finally:
        eng.set_u8(True)
    assert info["cert_dot"] and info["cert_u8"] == u8
    ou, orep, _ = oracle.s_merge(ds.vectors, g, h, 20, seed=4)
    _same_graph(u, ou)
    _same_report(rep, orep)


RHO_CASES = [
    # n, d, k, metric, data kind  (certified u8 route, non-certified fp32, cosine)
    (4000, 128, 20, 1, "intgmm"),
    (3000, 16, 12, 1, "uniform"),
    (3000, 100, 20, 2, "sphere"),
]


@pytest.mark.parametrize("rho", [0.5, 0.3])
@pytest.mark.parametrize("n,d,k,metric,kind", RHO_CASES)
def test_rho_sampling_matches_oracle(oracle, rho, n, d, k, metric, kind):
    """rho < 1 (classic NN-Descent sampling; no reference counterpart): the
    device path equals the oracle's restatement bit for bit (nn_descent,
    s_merge and j_merge), and rho = 1 stays the reference."""
    km = _km()
    ds = _data(km, n, d, kind, seed=n + d + 1)
    s1, s2 = split_ids(n, seed=6)
    g, rep = km.nn_descent(ds, metric, km.DescentParams(k=k, rho=rho), 1, member_ids=s1,
                           return_report=True)
    og, orep, _ = oracle.nn_descent(ds.vectors, metric, k, 1, member_ids=s1, rho=rho)
    _same_graph(g, og)
    _same_report(rep, orep)
    h, _, _ = oracle.nn_descent(ds.vectors, metric, k, 2, member_ids=s2, rho=rho)
    c = km.DistanceCounter()
    u, rep = km.s_merge(ds, _to_graph(km, og), _to_graph(km, h), km.MergeParams(k=k, seed=3, rho=rho),
                        counter=c, return_report=True)
    ou, orep, ocount = oracle.s_merge(ds.vectors, og, h, k, seed=3, rho=rho)
    _same_graph(u, ou)
    _same_report(rep, orep)
    assert c.count == ocount
    u, rep = km.j_merge(ds, _to_graph(km, og), s2, km.MergeParams(k=k, seed=5, rho=rho),
                        return_report=True)
    ou, orep, _ = oracle.j_merge(ds.vectors, og, s2, k, seed=5, rho=rho)
    _same_graph(u, ou)
    _same_report(rep, orep)


def test_rho_validation():
    km = _km()
    with pytest.raises(ValueError):
        km.MergeParams(k=10, rho=0.0)
    with pytest.raises(ValueError):
        km.DescentParams(k=10, rho=1.5)


def test_staged_host_transfers_large(oracle):
    """Host arrays above the 8 MB staging threshold in both directions (the
    dataset upload and the exported dists go through the pinned double
    buffer, several chunks each) -- results stay bit-identical."""
    km = _km()
    n, d, k = 60000, 40, 20  # vectors 9.6 MB, exported dists 9.6 MB
    ds = km.generate_uniform(n, d, seed=11)
    assert ds.vectors.nbytes > 8 << 20 and n * k * 8 > 8 << 20
    s1, s2 = split_ids(n, seed=12)
    g, _, _ = oracle.nn_descent(ds.vectors, 1, k, 1, member_ids=s1, max_iters=3)
    h, _, _ = oracle.nn_descent(ds.vectors, 1, k, 2, member_ids=s2, max_iters=3)
    mp = km.MergeParams(k=k, seed=3, max_iters=3)
    u = km.s_merge(ds, _to_graph(km, g), _to_graph(km, h), mp)
    ou, _, _ = oracle.s_merge(ds.vectors, g, h, k, seed=3, max_iters=3)
    _same_graph(u, ou)


@pytest.mark.parametrize("n,d,k,metric,kind", [
    (3000, 16, 64, 1, "intgmm"),   # W = 2k = 128 = MAX_W: u8 tensor-core route, 4 position blocks
    (2500, 12, 64, 1, "uniform"),  # same width on the non-certified tiled route
    (1200, 1, 8, 1, "uniform"),    # d = 1 (padded rows)
])
def test_limits_match_oracle(oracle, n, d, k, metric, kind):
    km = _km()
    ds = _data(km, n, d, kind, seed=n + d + 7)
    s1, s2 = split_ids(n, seed=13)
    g, _, _ = oracle.nn_descent(ds.vectors, metric, k, 1, member_ids=s1)
    h, _, _ = oracle.nn_descent(ds.vectors, metric, k, 2, member_ids=s2)
    c = km.DistanceCounter()
    u, rep = km.s_merge(ds, _to_graph(km, g), _to_graph(km, h), km.MergeParams(k=k, seed=3),
                        counter=c, return_report=True)
    ou, orep, ocount = oracle.s_merge(ds.vectors, g, h, k, seed=3)
    _same_graph(u, ou)
    _same_report(rep, orep)
    assert c.count == ocount
    gg, rep = km.nn_descent(ds, metric, km.DescentParams(k=k), 4, member_ids=s1, return_report=True)
    og, orep, _ = oracle.nn_descent(ds.vectors, metric, k, 4, member_ids=s1)
    _same_graph(gg, og)
    _same_report(rep, orep)


@pytest.mark.parametrize("d,k,metric,kind", [(960, 40, 1, "unitgmm"), (784, 40, 1, "uniform"),
                                             (960, 30, 2, "sphere")])
def test_long_rows_large_k_match_oracle(oracle, d, k, metric, kind):
    """Hoods whose whole rows exceed shared memory (4 W dp > 200 KB, e.g.
    GIST d=960 with k >= 27) take the d-chunked lazy join: bit-exact."""
    km = _km()
    n = 1200
    ds = _data(km, n, d, kind, seed=d + k)
    s1, s2 = split_ids(n, seed=3)
    g, _, _ = oracle.nn_descent(ds.vectors, metric, k, 1, member_ids=s1)
    h, _, _ = oracle.nn_descent(ds.vectors, metric, k, 2, member_ids=s2)
    c = km.DistanceCounter()
    u, rep = km.s_merge(ds, _to_graph(km, g), _to_graph(km, h), km.MergeParams(k=k, seed=3),
                        counter=c, return_report=True)
    ou, orep, ocount = oracle.s_merge(ds.vectors, g, h, k, seed=3)
    _same_graph(u, ou)
    _same_report(rep, orep)
    assert c.count == ocount
    gg, grep = km.nn_descent(ds, metric, km.DescentParams(k=k), 1, member_ids=s1,
                             return_report=True)
    _same_graph(gg, g)


def test_dataset_cache_sees_in_place_edits(oracle):
    """The device copy of Dataset.vectors is keyed on content: editing a
    writeable array in place between merges re-uploads it (a stale copy would
    give the old distances)."""
    km = _km()
    n, d, k = 1500, 16, 10
    vec = np.random.default_rng(5).random((n, d), dtype=np.float32)
    ds = km.Dataset.from_dense(vec)
    s1, s2 = split_ids(n, seed=2)
    g, _, _ = oracle.nn_descent(vec, 1, k, 1, member_ids=s1)
    km.j_merge(ds, _to_graph(km, g), s2, km.MergeParams(k=k, seed=1))
    vec[s2] *= 0.5  # in place: same object, new content
    g2, _, _ = oracle.nn_descent(vec, 1, k, 1, member_ids=s1)
    u = km.j_merge(ds, _to_graph(km, g2), s2, km.MergeParams(k=k, seed=1))
    ou, _, _ = oracle.j_merge(vec, g2, s2, k, seed=1)
    _same_graph(u, ou)
    # a read-only generated dataset is trusted by identity
    ro = km.generate_uniform(500, 8, seed=1)
    assert not ro.vectors.flags.writeable


def test_merge_rear_wider_tail_truncates(oracle):
    """merge_rear with rear lists wider than k keeps the k best (graph.py:259-280)."""
    km = _km()
    n, d = 800, 8
    ds = _data(km, n, d, "uniform", seed=3)
    ids = np.arange(n, dtype=np.int64)
    u = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=8), 1, member_ids=ids)
    wide = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=12), 2, member_ids=ids)
    narrow = km.KnnGraph(wide.member_ids, 8, km.Metric.L2)
    narrow.ids = wide.ids[:, :8].copy()
    narrow.dists = wide.dists[:, :8].copy()
    narrow.sizes = np.minimum(wide.sizes, 8).astype(np.int32)
    a = km.merge_rear(u, wide)
    b = km.merge_rear(u, narrow)
    _same_graph(a, b)


@pytest.mark.parametrize("variant", [-1, 1])
@pytest.mark.parametrize("n,d,k,kind,scale", [(2000, 960, 20, "unitgmm", 1.0), (1500, 960, 40, "unitgmm", 1.0),
                                              (1500, 784, 40, "uniform", 1.0), (1500, 500, 12, "uniform", 300.0),
                                              (1200, 1000, 8, "uniform", 1e-3)])
def test_tc_lazy_join_matches_oracle(oracle, variant, n, d, k, kind, scale):
    """Long non-certified L2 rows: the tcgen05 route (u8 limb products of a
    24-bit fixed-point image, rigorous lower bounds, exact values in the
    apply) and the fp32 chunked route are both bit-identical to the oracle,
    for data scaled so the fixed point's exponent moves."""
    km = _km()
    from paper_1908_00814_b200.engine import get_engine

    eng = get_engine()
    ds0 = _data(km, n, d, kind, seed=d + k + 11)
    vec = (ds0.vectors * np.float32(scale)).astype(np.float32)
    ds = km.Dataset.from_dense(vec)
    s1, s2 = split_ids(n, seed=6)
    g, _, _ = oracle.nn_descent(vec, 1, k, 1, member_ids=s1)
    eng.set_join_variant(variant)
    eng.reset_stats()
    try:
        c = km.DistanceCounter()
        u, rep = km.j_merge(ds, _to_graph(km, g), s2, km.MergeParams(k=k, seed=5), counter=c,
                            return_report=True)
        launches = eng.stats()["tc_join_launches"]
    finally:
        eng.set_join_variant(-1)
    ou, orep, ocount = oracle.j_merge(vec, g, s2, k, seed=5)
    _same_graph(u, ou)
    _same_report(rep, orep)
    assert c.count == ocount
    assert (launches > 0) == (variant == -1 and 2 * k <= 80)
