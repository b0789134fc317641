"""CPU oracle pinned against golden vectors produced by the reference itself
(tests/golden/make_golden.py): input subgraphs, merged graph, distance
count, the full BuildReport and every end-of-round state hash."""

import numpy as np
import pytest

from golden_check import GOLDEN, h_graph, inputs, report_list


@pytest.mark.parametrize("name", sorted(GOLDEN["cases"]))
def test_oracle_matches_reference(oracle, name):
    rec = GOLDEN["cases"][name]
    spec = rec["spec"]
    vec, g, h, s1, s2 = inputs(oracle, name)
    trace = []
    k, metric = spec["k"], spec["metric"]
    mp = spec.get("mp", {})
    if spec["op"] == "nnd":
        u, rep, count = oracle.nn_descent(vec, metric, k, spec["g_seed"], member_ids=s1, trace=trace)
    else:
        assert h_graph(g.ids, g.dists, g.sizes) == rec["g"], "input subgraph G differs"
        if spec["op"] == "smerge":
            assert h_graph(h.ids, h.dists, h.sizes) == rec["h"], "input subgraph H differs"
            u, rep, count = oracle.s_merge(vec, g, h, k, seed=spec["merge_seed"], trace=trace, **mp)
        else:
            raw = s2 if spec.get("raw", "s2") == "s2" else np.array([], dtype=np.int64)
            u, rep, count = oracle.j_merge(vec, g, raw, k, seed=spec["merge_seed"], trace=trace, **mp)
    assert h_graph(u.ids, u.dists, u.sizes) == rec["out"]
    assert count == rec["count"]
    assert rep.phi_initial == rec["report"]["phi_initial"]
    assert report_list(rep) == rec["report"]["rounds"]
    assert rep.converged == rec["report"]["converged"]
    assert [t["state"] for t in trace] == rec["states"]
    if "arrays" in rec:
        assert u.ids.tolist() == rec["arrays"]["ids"]
        assert u.dists.tolist() == rec["arrays"]["dists"]
