"""On-disk formats of merge inputs and outputs (reference io.py:27-145).

* fvecs / ivecs (texmex): per record, a little-endian int32 dimension
  followed by that many float32 / int32 values.
* KNNG graph files: b"KNNG", then n, k, metric tag as little-endian uint32,
  then n*k (int32 id, float32 dist) records; short lists are padded with
  (-1, +inf).  Distances are stored in float32 (as the reference does), so a
  save/load round trip keeps ids exactly and dists to float32 precision.
* member-id files: one ivecs record holding the ascending global ids (an
  empty set is an empty file).
"""

from __future__ import annotations

import struct

import numpy as np

from .core import Dataset, Metric
from .graph import KnnGraph

GRAPH_MAGIC = b"KNNG"
_RECORD = np.dtype([("id", "<i4"), ("dist", "<f4")])


def _write_vecs(path, mat: np.ndarray, dtype: str) -> None:
    mat = np.ascontiguousarray(mat, dtype=dtype)
    if mat.ndim != 2:
        raise ValueError("expected a 2-D array")
    n, d = mat.shape
    buf = np.empty((n, d + 1), dtype="<i4")
    buf[:, 0] = d
    buf[:, 1:] = mat.view("<i4")
    buf.tofile(path)


def _read_vecs(path, kind: str) -> np.ndarray:
    raw = np.fromfile(path, dtype="<i4")
    if raw.size == 0:
        return np.empty((0, 0), dtype=np.float32 if kind == "f" else np.int32)
    d = int(raw[0])
    if d <= 0 or raw.size % (d + 1):
        raise ValueError(f"{path} is not a valid {kind}vecs file")
    mat = raw.reshape(-1, d + 1)
    if np.any(mat[:, 0] != d):
        raise ValueError(f"{path} has inconsistent record dimensions")
    body = np.ascontiguousarray(mat[:, 1:])
    return body.view("<f4").astype(np.float32) if kind == "f" else body.astype(np.int32)


def write_fvecs(path, vectors) -> None:
    _write_vecs(path, vectors, "<f4")


def read_fvecs(path) -> np.ndarray:
    return _read_vecs(path, "f")


def write_ivecs(path, rows) -> None:
    _write_vecs(path, rows, "<i4")


def read_ivecs(path) -> np.ndarray:
    return _read_vecs(path, "i")


def load_dataset(path, metric: Metric) -> Dataset:
    """Dense fvecs dataset (the merge path is dense-only)."""
    if not Metric(metric).for_dense:
        raise ValueError("only dense (fvecs) datasets are supported on the merge path")
    return Dataset.from_dense(read_fvecs(path))


def save_graph(path, graph: KnnGraph) -> None:
    ids = np.asarray(graph.ids if isinstance(graph.ids, np.ndarray) else graph.ids.cpu().numpy())
    dists = np.asarray(graph.dists if isinstance(graph.dists, np.ndarray) else graph.dists.cpu().numpy())
    rec = np.empty(ids.shape, dtype=_RECORD)
    rec["id"] = ids
    rec["dist"] = dists.astype(np.float32)
    with open(path, "wb") as fh:
        fh.write(GRAPH_MAGIC)
        fh.write(struct.pack("<III", graph.n, graph.k, int(graph.metric)))
        rec.tofile(fh)


def load_graph(path, member_ids=None) -> KnnGraph:
    with open(path, "rb") as fh:
        if fh.read(4) != GRAPH_MAGIC:
            raise ValueError(f"{path} is not a graph file")
        n, k, tag = struct.unpack("<III", fh.read(12))
        rec = np.fromfile(fh, dtype=_RECORD, count=n * k)
    if rec.size != n * k:
        raise ValueError(f"{path} is truncated")
    rec = rec.reshape(n, k)
    gids = np.arange(n, dtype=np.int64) if member_ids is None else np.asarray(member_ids, np.int64)
    if gids.shape[0] != n:
        raise ValueError("member id list does not match the stored graph")
    ids = rec["id"].astype(np.int32)
    dists = rec["dist"].astype(np.float64)
    dists[ids < 0] = np.inf
    sizes = (ids >= 0).sum(axis=1).astype(np.int32)
    return KnnGraph.from_arrays(gids, k, Metric(tag), ids, dists, sizes)


def save_member_ids(path, member_ids) -> None:
    ids = np.asarray(member_ids, dtype=np.int64).reshape(1, -1)
    if ids.size == 0:
        open(path, "wb").close()
        return
    write_ivecs(path, ids)


def load_member_ids(path) -> np.ndarray:
    return read_ivecs(path).reshape(-1).astype(np.int64)


# -- hierarchy directories (reference io.py:201-271) --------------------------
# One directory per hierarchy: per layer ``layer_<t>.knng`` (graph),
# ``layer_<t>.ids.ivecs`` (ascending member ids) and, when a diversified
# adjacency exists, ``layer_<t>.kadj`` (not produced on this path), plus a
# ``manifest.json`` naming them -- the same names and JSON layout as the
# reference, so either package reads the other's directories.


def _layer_files(t: int) -> dict:
    return {"graph": f"layer_{t}.knng", "ids": f"layer_{t}.ids.ivecs", "adjacency": f"layer_{t}.kadj"}


def save_hierarchy_layer(directory, hierarchy, index: int) -> None:
    """Write layer ``index``'s member ids and (if held) its graph; the
    layer's ``path`` then points at the graph file."""
    import os

    os.makedirs(directory, exist_ok=True)
    layer = hierarchy.layers[index]
    files = _layer_files(index)
    save_member_ids(os.path.join(directory, files["ids"]), layer.member_ids)
    if layer.graph is not None:
        layer.path = os.path.join(directory, files["graph"])
        save_graph(layer.path, layer.graph)
    if layer.adjacency is not None:
        raise ValueError("diversified adjacency layers are not supported on the merge path")


def save_hierarchy_manifest(directory, hierarchy) -> None:
    import json
    import os

    os.makedirs(directory, exist_ok=True)
    entries = []
    for t, layer in enumerate(hierarchy.layers):
        files = _layer_files(t)
        entries.append({"size": int(layer.size), "ids": files["ids"], "graph": files["graph"],
                        "adjacency": files["adjacency"] if layer.adjacency is not None else None})
    manifest = {"k": int(hierarchy.k), "metric": Metric(hierarchy.metric).name,
                "layer_sizes": [int(s) for s in hierarchy.layer_sizes], "layers": entries}
    with open(os.path.join(directory, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=2)


def save_hierarchy(directory, hierarchy) -> None:
    """Write every layer, reading dropped ones back from their files first."""
    for t, layer in enumerate(hierarchy.layers):
        dropped = layer.graph is None and layer.path is not None
        if dropped:
            layer.graph = hierarchy.layer_graph(t)
        save_hierarchy_layer(directory, hierarchy, t)
        if dropped:
            layer.graph = None
    save_hierarchy_manifest(directory, hierarchy)


def load_hierarchy(directory, lazy: bool = True):
    """A ``Hierarchy`` from a manifest directory; with ``lazy`` the graphs
    stay on disk until ``Hierarchy.layer_graph`` asks for them."""
    import json
    import os

    from .hierarchy import Hierarchy, HierarchyLayer

    with open(os.path.join(directory, "manifest.json")) as fh:
        manifest = json.load(fh)
    out = Hierarchy(layers=[], k=int(manifest["k"]), metric=Metric.from_name(manifest["metric"]))
    for entry in manifest["layers"]:
        layer = HierarchyLayer(member_ids=load_member_ids(os.path.join(directory, entry["ids"])))
        gpath = os.path.join(directory, entry["graph"])
        if os.path.exists(gpath):
            layer.path = gpath
            if not lazy:
                layer.graph = load_graph(gpath, member_ids=layer.member_ids)
        out.layers.append(layer)
    return out
