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


# ---------------------------------------------------------------------------
# hood-chunked rounds (candidate budget exceeded), sharded vs the oracle,
# the config-5 tree, and real multi-process TorchComm
# ---------------------------------------------------------------------------

def _og(km, og):
    g = km.KnnGraph(og.member_ids, og.k, og.metric)
    g.ids, g.dists, g.sizes = og.ids.copy(), og.dists.copy(), og.sizes.copy()
    return g


def _same(u, ou):
    assert np.array_equal(np.asarray(u.member_ids), np.asarray(ou.member_ids))
    assert np.array_equal(u.sizes, ou.sizes)
    assert np.array_equal(u.ids, ou.ids)
    assert np.array_equal(u.dists, ou.dists)


def _same_rep(rep, orep):
    assert rep.phi_initial == orep.phi_initial
    assert [(r.iteration, r.pairs, r.updates, r.phi, r.distance_count) for r in rep.rounds] == \
        [(r.iteration, r.pairs, r.updates, r.phi, r.distance_count) for r in orep.rounds]


# round 1 of these cases has ~10^5 admissible pairs: 200 KB of 12-byte slot
# budget forces ~8-20 hood chunks in the first rounds
_SMALL_BUDGET = 200_000


@pytest.mark.parametrize("kind,metric,k", [("intgmm", 1, 16), ("uniform", 1, 12),
                                           ("sphere", 2, 20), ("unitgmm", 1, 10)])
def test_chunked_rounds_match_oracle(oracle, kind, metric, k):
    """Rounds whose 2P slots exceed the candidate budget run in ascending
    hood chunks (knnm.cu plan_chunks / join_chunk): bit-exact vs the oracle,
    with at least three chunks in the first round."""
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200.engine import get_engine

    n = 3000
    d = {"intgmm": 128, "uniform": 16, "sphere": 100, "unitgmm": 960}[kind]
    ds = {"intgmm": lambda: km.generate_int_gmm(n, d, n_centres=30, seed=21),
          "uniform": lambda: km.generate_uniform(n, d, seed=21),
          "sphere": lambda: km.generate_sphere_gmm(n, d, n_centres=20, seed=21),
          "unitgmm": lambda: km.generate_unit_gmm(n, d, n_centres=20, seed=21)}[kind]()
    s1, s2 = split_ids(n, seed=5)
    g, _, _ = oracle.nn_descent(ds.vectors, metric, k, 1, member_ids=s1)
    h, _, _ = oracle.nn_descent(ds.vectors, metric, k, 2, member_ids=s2)
    eng = get_engine()
    eng.set_cand_budget(_SMALL_BUDGET)
    eng.reset_stats()
    try:
        c = km.DistanceCounter()
        u, rep = km.s_merge(ds, _og(km, g), _og(km, h), km.MergeParams(k=k, seed=3), counter=c,
                            return_report=True)
        st = eng.stats()
        cj = km.DistanceCounter()
        uj, repj = km.j_merge(ds, _og(km, g), s2, km.MergeParams(k=k, seed=4), counter=cj,
                              return_report=True)
    finally:
        eng.set_cand_budget(0)
    assert st["join_redos"] >= 1
    assert st["join_launches"] >= st["rounds"] + 2  # >= 3 chunks in some round
    ou, orep, ocount = oracle.s_merge(ds.vectors, g, h, k, seed=3)
    _same(u, ou)
    _same_rep(rep, orep)
    assert c.count == ocount
    oj, orepj, ocj = oracle.j_merge(ds.vectors, g, s2, k, seed=4)
    _same(uj, oj)
    _same_rep(repj, orepj)
    assert cj.count == ocj


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("budget", [0, _SMALL_BUDGET])
def test_sharded_matches_oracle(oracle, world, budget):
    """Sharded S-Merge and J-Merge compared with the oracle directly (not only
    with the single-GPU path), with and without hood chunks on every rank."""
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import distributed as D

    n = 3000
    ds = km.generate_int_gmm(n, 64, n_centres=25, seed=17)
    s1, s2 = split_ids(n, seed=9)
    g, _, _ = oracle.nn_descent(ds.vectors, 1, 14, 1, member_ids=s1)
    h, _, _ = oracle.nn_descent(ds.vectors, 1, 14, 2, member_ids=s2)
    engines = _engines(world)
    for e in engines.values():
        e.set_cand_budget(budget)
    c = km.DistanceCounter()
    u, rep = D.s_merge_sharded(ds, _og(km, g), _og(km, h), km.MergeParams(k=14, seed=6),
                               D.LoopbackComm(world), engines, counter=c, return_report=True)
    ou, orep, ocount = oracle.s_merge(ds.vectors, g, h, 14, seed=6)
    _same(u, ou)
    _same_rep(rep, orep)
    assert c.count == ocount
    cj = km.DistanceCounter()
    uj, repj = D.j_merge_sharded(ds, _og(km, g), s2, km.MergeParams(k=14, seed=8),
                                 D.LoopbackComm(world), engines, counter=cj, return_report=True)
    oj, orepj, ocj = oracle.j_merge(ds.vectors, g, s2, 14, seed=8)
    _same(uj, oj)
    _same_rep(repj, orepj)
    assert cj.count == ocj


def _tree_inputs(km, world, per, d=32, k=12):
    ds = km.generate_int_gmm(world * per, d, n_centres=40, seed=31)
    sets = [np.arange(r * per, (r + 1) * per, dtype=np.int64) for r in range(world)]
    graphs = [km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=k), 100 + r, member_ids=sets[r])
              for r in range(world)]
    return ds, sets, graphs


@pytest.mark.parametrize("world", [2, 4, 8])
def test_tree_merge_loopback_matches_sequential(world):
    """Config 5's tree with P virtual ranks (one engine each, LoopbackComm per
    group) equals the sequential single-GPU tree of s_merge calls, bit for bit."""
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import distributed as D

    ds, sets, graphs = _tree_inputs(km, world, 700)
    mp = km.MergeParams(k=12, seed=2)
    engines = _engines(world)
    final, log = D.tree_merge(ds, {r: graphs[r] for r in range(world)}, sets, mp, world,
                              lambda level, ranks: D.LoopbackComm(len(ranks)), engines)
    cur = list(graphs)
    counts = []
    while len(cur) > 1:
        nxt = []
        for i in range(0, len(cur), 2):
            c = km.DistanceCounter()
            nxt.append(km.s_merge(ds, cur[i], cur[i + 1], mp, counter=c))
            counts.append(c.count)
        cur = nxt
    want = cur[0]
    for r in range(world):
        got = final[r]
        assert np.array_equal(np.asarray(got.ids.cpu()), want.ids)
        assert np.array_equal(np.asarray(got.dists.cpu()), want.dists)
        assert np.array_equal(np.asarray(got.sizes.cpu()), want.sizes)
    assert [c.count for _, _, c in log] == counts


def _mp_worker(rank, world, port, q, task):
    import os

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1908_00814_b200 as km
        from paper_1908_00814_b200 import distributed as D
        from paper_1908_00814_b200.engine import Engine

        eng = Engine(0)
        if task == "merge":
            from oracle import oracle as O

            n = 2400
            ds = km.generate_int_gmm(n, 48, n_centres=20, seed=41)
            rng = np.random.default_rng(3)
            perm = rng.permutation(n)
            s1, s2 = np.sort(perm[: n // 2]), np.sort(perm[n // 2:])
            g, _, _ = O.nn_descent(ds.vectors, 1, 12, 1, member_ids=s1)
            h, _, _ = O.nn_descent(ds.vectors, 1, 12, 2, member_ids=s2)
            comm = D.TorchComm()
            eng.set_cand_budget(60_000 if rank == 0 else 0)  # chunks on rank 0 only
            c = km.DistanceCounter()
            u, rep = D.s_merge_sharded(ds, _og(km, g), _og(km, h), km.MergeParams(k=12, seed=5),
                                       comm, {rank: eng}, counter=c, return_report=True)
            ou, orep, ocount = O.s_merge(ds.vectors, g, h, 12, seed=5)
            ok = (np.array_equal(u.ids, ou.ids) and np.array_equal(u.dists, ou.dists)
                  and np.array_equal(u.sizes, ou.sizes) and c.count == ocount
                  and [(r.pairs, r.updates, r.phi) for r in rep.rounds]
                  == [(r.pairs, r.updates, r.phi) for r in orep.rounds])
            uj = D.j_merge_sharded(ds, _og(km, g), s2, km.MergeParams(k=12, seed=7), comm,
                                   {rank: eng})
            oj, _, _ = O.j_merge(ds.vectors, g, s2, 12, seed=7)
            ok = ok and np.array_equal(uj.ids, oj.ids) and np.array_equal(uj.dists, oj.dists)
        else:  # tree over new_group sub-communicators, one subgraph per rank
            per = 600
            ds, sets, _ = None, None, None
            ds = km.generate_int_gmm(world * per, 32, n_centres=40, seed=31)
            sets = [np.arange(r * per, (r + 1) * per, dtype=np.int64) for r in range(world)]
            mine = km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=12), 100 + rank,
                                 member_ids=sets[rank])
            groups = {tuple(m): dist.new_group(m) for _, m in D.tree_groups(world)}

            def group_comm(level, ranks):
                return D.TorchComm(groups[tuple(ranks)]) if rank in ranks else None

            mp = km.MergeParams(k=12, seed=2)
            final, log = D.tree_merge(ds, {rank: mine}, sets, mp, world, group_comm, {rank: eng})
            lo, hi = final[rank].shard
            # the sequential single-GPU tree, computed on every rank
            cur = [km.nn_descent(ds, km.Metric.L2, km.DescentParams(k=12), 100 + r,
                                 member_ids=sets[r]) for r in range(world)]
            while len(cur) > 1:
                cur = [km.s_merge(ds, cur[i], cur[i + 1], mp) for i in range(0, len(cur), 2)]
            got = final[rank]
            ok = (lo, hi) == (rank * per, (rank + 1) * per)
            ok = ok and np.array_equal(got.ids[lo:hi].cpu().numpy(), cur[0].ids[lo:hi])
            ok = ok and np.array_equal(got.dists[lo:hi].cpu().numpy(), cur[0].dists[lo:hi])
            ok = ok and np.array_equal(got.sizes[lo:hi].cpu().numpy(), cur[0].sizes[lo:hi])
        q.put((rank, bool(ok), ""))
    except Exception as exc:  # report, do not hang the parent
        import traceback

        q.put((rank, False, traceback.format_exc()[-2000:]))
    finally:
        dist.destroy_process_group()


def _run_mp(world, task):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_mp_worker, args=(r, world, port, q, task)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert ok, (rank, err)
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.timeout(900)
def test_torchcomm_processes_match_oracle():
    """s_merge_sharded / j_merge_sharded through TorchComm in two processes
    (each its own engine on cuda:0; gloo with host-staged tensors), chunked
    rounds on one rank only: bit-exact vs the oracle."""
    _run_mp(2, "merge")


@pytest.mark.timeout(900)
def test_tree_merge_processes_new_group():
    """Config 5's tree across 4 processes with torch new_group
    sub-communicators and no re-sharding: each rank's rows of the final graph
    equal the sequential single-GPU tree."""
    _run_mp(4, "tree")
