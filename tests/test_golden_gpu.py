"""CUDA path vs golden vectors produced by the reference itself: merged
graph, distance count, BuildReport and the end-of-round state of every
iteration (replay contract of SURVEY.md §6.3), bit-exact."""

import hashlib

import numpy as np
import pytest

from golden_check import GOLDEN, h_graph, inputs, report_list

pytestmark = pytest.mark.gpu


def _graph(km, og):
    return km.KnnGraph.from_arrays(og.member_ids, og.k, km.Metric(og.metric), og.ids.copy(),
                                   og.dists.copy(), og.sizes.copy())


def _state_hash(eng):
    ids, dists, flags, sizes = eng.state()
    h = hashlib.sha256()
    for a in (ids, dists, flags.astype(np.uint8), sizes):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


@pytest.mark.parametrize("variant", [-1, 0, 1])
@pytest.mark.parametrize("name", sorted(GOLDEN["cases"]))
def test_cuda_matches_reference(oracle, name, variant):
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import construct
    from paper_1908_00814_b200.engine import get_engine

    rec = GOLDEN["cases"][name]
    spec = rec["spec"]
    vec, g, h, s1, s2 = inputs(oracle, name)
    ds = km.Dataset.from_dense(vec, validate=False)
    k, metric = spec["k"], spec["metric"]
    states = []
    eng = get_engine()
    eng.set_join_variant(variant)
    construct.ROUND_HOOK = lambda e: states.append(_state_hash(e))
    try:
        c = km.DistanceCounter()
        if spec["op"] == "nnd":
            u, rep = km.nn_descent(ds, metric, km.DescentParams(k=k), spec["g_seed"],
                                   member_ids=s1, counter=c, return_report=True)
        else:
            mp = km.MergeParams(k=k, seed=spec["merge_seed"], **spec.get("mp", {}))
            if spec["op"] == "smerge":
                u, rep = km.s_merge(ds, _graph(km, g), _graph(km, h), mp, counter=c,
                                    return_report=True)
            else:
                raw = s2 if spec.get("raw", "s2") == "s2" else np.array([], dtype=np.int64)
                u, rep = km.j_merge(ds, _graph(km, g), raw, mp, counter=c, return_report=True)
    finally:
        construct.ROUND_HOOK = None
        eng.set_join_variant(-1)
    assert h_graph(u.ids, u.dists, u.sizes) == rec["out"]
    assert c.count == rec["count"]
    assert rep.phi_initial == rec["report"]["phi_initial"]
    assert report_list(rep) == rec["report"]["rounds"]
    assert rep.converged == rec["report"]["converged"]
    assert states == rec["states"]
