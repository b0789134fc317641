"""Device engine: one libknnm context per CUDA device.

This is the host-side owner of the device state behind the reference's
round engine (construct.py:111-179) and merge glue (merge.py:195-338).  It
keeps the dataset resident in HBM across merges (tree merges and H-Merge
reuse it) and forwards each reference operator to its C-ABI replacement.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _lib
from ._lib import check, ptr


class Engine:
    def __init__(self, device: int = 0):
        self.device = int(device)
        lib = _lib.load()
        h = ctypes.c_void_p()
        check(lib.knnm_create(self.device, ctypes.byref(h)), "knnm_create")
        self._h = h
        self._lib = lib
        self._vectors = None  # host array currently resident on the device
        self._metric = None
        self.n = 0
        self.k = 0

    def close(self) -> None:
        if self._h is not None and self._h.value:
            self._lib.knnm_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- dataset -----------------------------------------------------------
    def set_dataset(self, vectors: np.ndarray, metric: int) -> None:
        """Upload Dataset.vectors once; re-used while the same array is passed."""
        if self._vectors is vectors and self._metric == int(metric):
            return
        v = np.ascontiguousarray(vectors, dtype=np.float32)
        if v.ndim != 2:
            raise ValueError("dense data must be a 2-D array")
        check(self._lib.knnm_set_dataset(self._h, ptr(v), v.shape[0], v.shape[1], int(metric)),
              "knnm_set_dataset")
        self._vectors = vectors
        self._metric = int(metric)

    # -- merge state -------------------------------------------------------
    def begin(self, union_gids: np.ndarray, labels: np.ndarray, k: int) -> None:
        ug = np.ascontiguousarray(union_gids, dtype=np.int64)
        lab = np.ascontiguousarray(labels, dtype=np.int8)
        check(self._lib.knnm_begin(self._h, ptr(ug), ug.shape[0], ptr(lab), int(k)), "knnm_begin")
        self.n = ug.shape[0]
        self.k = int(k)

    def load_graph(self, rows: np.ndarray, graph, k1: int) -> None:
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        gi = np.ascontiguousarray(graph.ids, dtype=np.int32)
        gd = np.ascontiguousarray(graph.dists, dtype=np.float64)
        gs = np.ascontiguousarray(graph.sizes, dtype=np.int32)
        check(self._lib.knnm_load_graph(self._h, ptr(rows), rows.shape[0], ptr(gi), ptr(gd),
                                        ptr(gs), int(graph.k), int(k1)), "knnm_load_graph")

    def insert_directed(self, rows: np.ndarray, nids: np.ndarray) -> int:
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        nids = np.ascontiguousarray(nids, dtype=np.int32)
        acc = ctypes.c_int64()
        check(self._lib.knnm_insert_directed(self._h, ptr(rows), ptr(nids), rows.shape[0],
                                             ctypes.byref(acc)), "knnm_insert_directed")
        return int(acc.value)

    def round(self, mode: int, rev_cap: int, seed: int):
        pairs = ctypes.c_int64()
        acc = ctypes.c_int64()
        check(self._lib.knnm_round(self._h, int(mode), int(rev_cap), ctypes.c_uint64(seed),
                                   ctypes.byref(pairs), ctypes.byref(acc)), "knnm_round")
        return int(pairs.value), int(acc.value)

    def phi(self) -> float:
        out = ctypes.c_double()
        check(self._lib.knnm_phi(self._h, ctypes.byref(out)), "knnm_phi")
        return float(out.value)

    def export(self, merge_rear: bool):
        ids = np.empty((self.n, self.k), dtype=np.int32)
        dists = np.empty((self.n, self.k), dtype=np.float64)
        sizes = np.empty(self.n, dtype=np.int32)
        check(self._lib.knnm_export(self._h, int(bool(merge_rear)), ptr(ids), ptr(dists),
                                    ptr(sizes)), "knnm_export")
        return ids, dists, sizes

    def state(self):
        ids = np.empty((self.n, self.k), dtype=np.int32)
        dists = np.empty((self.n, self.k), dtype=np.float64)
        flags = np.empty((self.n, self.k), dtype=np.uint8)
        sizes = np.empty(self.n, dtype=np.int32)
        check(self._lib.knnm_get_state(self._h, ptr(ids), ptr(dists), ptr(flags), ptr(sizes)),
              "knnm_get_state")
        return ids, dists, flags, sizes

    # -- on_pair capture ---------------------------------------------------
    def set_capture(self, on: bool) -> None:
        check(self._lib.knnm_set_capture(self._h, int(bool(on))), "knnm_set_capture")

    def fetch_captured(self):
        cnt = ctypes.c_int64()
        check(self._lib.knnm_capture_count(self._h, ctypes.byref(cnt)), "knnm_capture_count")
        m = int(cnt.value)
        pa = np.empty(m, dtype=np.int32)
        pb = np.empty(m, dtype=np.int32)
        pd = np.empty(m, dtype=np.float64)
        check(self._lib.knnm_capture_fetch(self._h, ptr(pa), ptr(pb), ptr(pd), m),
              "knnm_capture_fetch")
        return pa, pb, pd

    # -- instrumentation ---------------------------------------------------
    def set_profiling(self, on: bool) -> None:
        check(self._lib.knnm_set_profiling(self._h, int(bool(on))), "knnm_set_profiling")

    def stats(self) -> dict:
        s = _lib.KnnmStats()
        check(self._lib.knnm_get_stats(self._h, ctypes.byref(s)), "knnm_get_stats")
        return s.as_dict()

    def reset_stats(self) -> None:
        check(self._lib.knnm_reset_stats(self._h), "knnm_reset_stats")

    def sync(self) -> None:
        check(self._lib.knnm_sync(self._h), "knnm_sync")


_engines: dict[int, Engine] = {}
_lock = threading.Lock()


def default_device() -> int:
    env = os.environ.get("KNNM_DEVICE")
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0"))


def get_engine(device: int | None = None) -> Engine:
    """Process-wide engine for `device` (created on first use)."""
    dev = default_device() if device is None else int(device)
    with _lock:
        eng = _engines.get(dev)
        if eng is None:
            eng = Engine(dev)
            _engines[dev] = eng
        return eng
