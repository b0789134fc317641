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


@pytest.mark.gpu
def test_h_merge_snapshot_dir_byte_identical_to_reference(tmp_path):
    """snapshot_dir (reference merge.py:457-467, io.py:201-248): every layer
    file and the manifest hash-equal to the reference's; intermediates are
    dropped from memory and read back lazily; load_hierarchy round-trips."""
    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import io as kio

    rec = EXTRA["hmerge"]
    ds = km.Dataset.from_dense(C.make_data(dict(data="uniform", n=2000, d=4, data_seed=13)), validate=False)
    graph, hier = km.h_merge(ds, km.Metric.L2, km.MergeParams(k=10, seed=4), snapshot_dir=str(tmp_path))
    got = {f: hashlib.sha256((tmp_path / f).read_bytes()).hexdigest() for f in sorted(os.listdir(tmp_path))}
    assert got == rec["snapshot_sha256"]
    assert all(l.graph is None for l in hier.layers[:-1]) and hier.layers[-1].graph is graph
    back = kio.load_hierarchy(str(tmp_path))
    assert back.layer_sizes == rec["layer_sizes"] and back.k == 10 and back.metric == km.Metric.L2
    back.validate(2000)
    for t in range(len(back.layers)):
        a, b = hier.layer_graph(t), back.layer_graph(t)
        assert np.array_equal(a.ids, b.ids) and np.array_equal(a.sizes, b.sizes)


def test_hierarchy_manifest_round_trip(tmp_path):
    """save_hierarchy / load_hierarchy on CPU-built layers (no GPU): files
    named as the reference's, eager and lazy loads agree."""
    import json

    import paper_1908_00814_b200 as km
    from paper_1908_00814_b200 import io as kio

    rng = np.random.default_rng(0)
    layers = []
    for m in (8, 20):
        ids = np.sort(rng.choice(20, size=m, replace=False)).astype(np.int64)
        k = 3
        nb = np.stack([rng.choice(m, size=k, replace=False) for _ in range(m)]).astype(np.int32)
        dd = np.sort(rng.random((m, k)), axis=1)
        g = km.KnnGraph.from_arrays(ids, k, km.Metric.L2, nb, dd, np.full(m, k, np.int32))
        layers.append(km.HierarchyLayer(ids, g))
    h = km.Hierarchy(layers=layers, k=3, metric=km.Metric.L2)
    kio.save_hierarchy(str(tmp_path), h)
    man = json.loads((tmp_path / "manifest.json").read_text())
    assert man["layer_sizes"] == [8, 20] and man["metric"] == "L2"
    assert [e["graph"] for e in man["layers"]] == ["layer_0.knng", "layer_1.knng"]
    lazy, eager = kio.load_hierarchy(str(tmp_path)), kio.load_hierarchy(str(tmp_path), lazy=False)
    assert lazy.layers[0].graph is None and eager.layers[0].graph is not None
    for t in range(2):
        a, b = lazy.layer_graph(t), h.layer_graph(t)
        assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dists, b.dists.astype(np.float32))
    lazy.validate(20)
    assert km.doubling_layer_sizes(200, 10) == [64, 128, 200]
    assert km.doubling_layer_sizes(50, 60) == [50]
