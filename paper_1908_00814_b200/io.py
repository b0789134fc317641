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
