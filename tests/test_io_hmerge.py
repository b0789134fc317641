"""KNNG graph files + member-id ivecs (CPU, byte-identical to files written
by the reference) and H-Merge on the GPU (bit-identical to the reference's
h_merge: output graph, layer snapshots, per-stage reports, distance count)."""

import hashlib
import json
import os
import sys

import numpy as np
import pytest

from golden_check import h_graph

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import cases as C  # noqa: E402

with open(os.path.join(HERE, "golden", "golden_extra.json")) as f:
    EXTRA = json.load(f)


def test_knng_files_byte_identical_to_reference(oracle, tmp_path):
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import io as kio

    vec = C.make_data(dict(data="uniform", n=300, d=5, data_seed=2))
    og, _, _ = oracle.nn_descent(vec, 1, 6, 3, member_ids=np.arange(0, 300, 2))
    assert h_graph(og.ids, og.dists, og.sizes) == EXTRA["knng"]["graph"]
    g = km.KnnGraph.from_arrays(og.member_ids, 6, km.Metric.L2, og.ids, og.dists, og.sizes)
    kio.save_graph(tmp_path / "g.knng", g)
    kio.save_member_ids(tmp_path / "g.ids", g.member_ids)
    assert hashlib.sha256((tmp_path / "g.knng").read_bytes()).hexdigest() == EXTRA["knng"]["file_sha256"]
    assert hashlib.sha256((tmp_path / "g.ids").read_bytes()).hexdigest() == EXTRA["knng"]["ids_sha256"]
    back = kio.load_graph(tmp_path / "g.knng", member_ids=kio.load_member_ids(tmp_path / "g.ids"))
    assert np.array_equal(back.ids, g.ids) and np.array_equal(back.sizes, g.sizes)
    assert np.array_equal(back.dists, np.where(g.ids >= 0, g.dists.astype(np.float32), np.inf))
    kio.write_fvecs(tmp_path / "x.fvecs", vec)
    assert np.array_equal(kio.read_fvecs(tmp_path / "x.fvecs"), vec)
    kio.save_member_ids(tmp_path / "e.ids", np.array([], dtype=np.int64))
    assert kio.load_member_ids(tmp_path / "e.ids").size == 0
    with pytest.raises(ValueError):
        (tmp_path / "bad").write_bytes(b"XXXX" + bytes(12))
        kio.load_graph(tmp_path / "bad")


@pytest.mark.gpu
def test_h_merge_bit_identical_to_reference():
    import paper_1908_00814_b200 as km
    from golden_check import report_list

    rec = EXTRA["hmerge"]
    ds = km.Dataset.from_dense(C.make_data(dict(data="uniform", n=2000, d=4, data_seed=13)), validate=False)
    c = km.DistanceCounter()
    graph, hier, reps = km.h_merge(ds, km.Metric.L2, km.MergeParams(k=10, seed=4), counter=c,
                                   return_report=True)
    hier.validate(2000)
    assert hier.layer_sizes == rec["layer_sizes"]
    assert h_graph(graph.ids, graph.dists, graph.sizes) == rec["out"]
    assert [h_graph(l.graph.ids, l.graph.dists, l.graph.sizes) for l in hier.layers] == rec["layers"]
    assert c.count == rec["count"]
    for (name, rep), (gname, grep) in zip(reps, rec["reports"]):
        assert name == gname
        assert rep.phi_initial == grep["phi_initial"]
        assert report_list(rep) == grep["rounds"]
