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
        self._key = None      # (shape, metric) of the resident copy
        self._fp = None       # its content fingerprint
        self.pinned_outputs = False  # export into page-locked host buffers
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
        """Keep Dataset.vectors resident in HBM across merges.

        The device copy is re-used when the same read-only array is passed
        again (its whole base chain read-only, so it cannot change), or when
        the content fingerprint (knnm_fingerprint, host threads) equals the
        uploaded one -- an in-place edit of a writeable array is re-uploaded,
        never served stale.  ``invalidate()`` drops the copy explicitly."""
        v = np.ascontiguousarray(vectors, dtype=np.float32)
        if v.ndim != 2:
            raise ValueError("dense data must be a 2-D array")
        key = (v.shape, int(metric))
        if self._vectors is vectors and self._key == key and _frozen(vectors):
            return
        if self._vectors is not None and self._key == key:
            fp = fingerprint(v)
            if self._fp == fp:
                self._vectors = vectors
                return
            check(self._lib.knnm_set_dataset(self._h, ptr(v), v.shape[0], v.shape[1], int(metric)),
                  "knnm_set_dataset")
        else:
            # nothing comparable is resident: the upload happens anyway, so the
            # fingerprint (kept for the next call) runs beside it (both native
            # calls release the GIL)
            box = {}
            th = threading.Thread(target=lambda: box.setdefault("fp", fingerprint(v)))
            th.start()
            try:
                check(self._lib.knnm_set_dataset(self._h, ptr(v), v.shape[0], v.shape[1], int(metric)),
                      "knnm_set_dataset")
            finally:
                th.join()
            fp = box["fp"]
        self._vectors = vectors
        self._metric = int(metric)
        self._key = key
        self._fp = fp

    def invalidate(self) -> None:
        """Forget the resident dataset: the next set_dataset uploads."""
        self._vectors = None
        self._key = None
        self._fp = None

    # -- merge state -------------------------------------------------------
    def begin(self, union_gids: np.ndarray, labels: np.ndarray, k: int) -> None:
        ug = np.ascontiguousarray(union_gids, dtype=np.int64)
        lab = np.ascontiguousarray(labels, dtype=np.int8)
        check(self._lib.knnm_begin(self._h, ptr(ug), ug.shape[0], ptr(lab), int(k)), "knnm_begin")
        self.n = ug.shape[0]
        self.k = int(k)

    def load_graph(self, rows: np.ndarray, graph, k1: int) -> None:
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        if _is_cuda_tensor(graph.ids):
            # graph already resident in HBM (torch CUDA tensors): no host copy
            gi, gd, gs = graph.ids, graph.dists, graph.sizes
            for t, dt in ((gi, "int32"), (gd, "float64"), (gs, "int32")):
                if not (_is_cuda_tensor(t) and t.is_contiguous() and str(t.dtype).endswith(dt)):
                    raise ValueError("device graph arrays must be contiguous CUDA tensors "
                                     "(ids int32, dists float64, sizes int32)")
            self.wait_torch()  # the tensors may still be in flight on torch's stream
            check(self._lib.knnm_load_graph_dev(
                self._h, ptr(rows), rows.shape[0], ctypes.c_void_p(gi.data_ptr()),
                ctypes.c_void_p(gd.data_ptr()), ctypes.c_void_p(gs.data_ptr()), int(graph.k),
                int(k1)), "knnm_load_graph_dev")
            return
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

    def insert_rows(self, rows: np.ndarray, count: int, nids: np.ndarray) -> int:
        """Directed inserts with targets np.repeat(rows, count), expanded on device."""
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        nids = np.ascontiguousarray(nids, dtype=np.int32)
        if nids.shape[0] != rows.shape[0] * int(count):
            raise ValueError("nids must hold len(rows) * count entries")
        acc = ctypes.c_int64()
        check(self._lib.knnm_insert_rows(self._h, ptr(rows), rows.shape[0], int(count), ptr(nids),
                                         ctypes.byref(acc)), "knnm_insert_rows")
        return int(acc.value)

    # -- random-append draw matrix (merge.py:146-163) ------------------------
    def _bad(self, n):
        return np.empty(max(int(n), 1), dtype=np.int64)

    def draws_load(self, cand: np.ndarray) -> np.ndarray:
        cand = np.ascontiguousarray(cand, dtype=np.int64)
        bad = self._bad(cand.shape[0])
        nb = ctypes.c_int64()
        check(self._lib.knnm_draws_load(self._h, ptr(cand), cand.shape[0], cand.shape[1],
                                        ptr(bad), ctypes.byref(nb)), "knnm_draws_load")
        return bad[: nb.value].copy()

    def draws_replace(self, rows: np.ndarray, vals: np.ndarray) -> np.ndarray:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        vals = np.ascontiguousarray(vals, dtype=np.int64)
        bad = self._bad(rows.shape[0])
        nb = ctypes.c_int64()
        check(self._lib.knnm_draws_replace(self._h, ptr(rows), rows.shape[0], ptr(vals), ptr(bad),
                                           ctypes.byref(nb)), "knnm_draws_replace")
        return bad[: nb.value].copy()

    def draws_gen(self, rng, m: int, nrows: int, t: int) -> np.ndarray:
        """rng.integers(0, m, size=(nrows, t)) generated on the device (same
        values, same resulting generator state); returns the bad rows."""
        st, arr, has, uint = _pcg_split(rng)
        bad = self._bad(nrows)
        nb = ctypes.c_int64()
        used = ctypes.c_int64()
        check(self._lib.knnm_draws_gen(self._h, ptr(arr), int(has), ctypes.c_uint32(uint), int(m),
                                       int(nrows), int(t), ctypes.byref(used), ptr(bad),
                                       ctypes.byref(nb)), "knnm_draws_gen")
        _pcg_consume(rng, st, int(used.value))
        return bad[: nb.value].copy()

    def draws_regen(self, rng, m: int, rows: np.ndarray) -> np.ndarray:
        """cand[rows] = rng.integers(0, m, size=(len(rows), t)) on the device."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        st, arr, has, uint = _pcg_split(rng)
        bad = self._bad(rows.shape[0])
        nb = ctypes.c_int64()
        used = ctypes.c_int64()
        check(self._lib.knnm_draws_regen(self._h, ptr(arr), int(has), ctypes.c_uint32(uint), int(m),
                                         ptr(rows), rows.shape[0], ctypes.byref(used), ptr(bad),
                                         ctypes.byref(nb)), "knnm_draws_regen")
        _pcg_consume(rng, st, int(used.value))
        return bad[: nb.value].copy()

    def draws_insert_range(self, rows: np.ndarray, pool: np.ndarray, r0: int, r1: int) -> int:
        """draws_insert for draw rows [r0, r1) only (sharded initialisation)."""
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        pool = np.ascontiguousarray(pool, dtype=np.int32)
        acc = ctypes.c_int64()
        check(self._lib.knnm_draws_insert_range(self._h, ptr(rows), ptr(pool), pool.shape[0],
                                                int(r0), int(r1), ctypes.byref(acc)),
              "knnm_draws_insert_range")
        return int(acc.value)

    def draws_insert(self, rows: np.ndarray, pool: np.ndarray) -> int:
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        pool = np.ascontiguousarray(pool, dtype=np.int32)
        acc = ctypes.c_int64()
        check(self._lib.knnm_draws_insert(self._h, ptr(rows), ptr(pool), pool.shape[0],
                                          ctypes.byref(acc)), "knnm_draws_insert")
        return int(acc.value)

    def set_sample(self, new_cap: int) -> None:
        """rho-sampling: new entries per row per round (0 = all, the reference)."""
        check(self._lib.knnm_set_sample(self._h, int(new_cap)), "knnm_set_sample")

    def round(self, mode: int, rev_cap: int, seed: int):
        pairs = ctypes.c_int64()
        acc = ctypes.c_int64()
        check(self._lib.knnm_round(self._h, int(mode), int(rev_cap), ctypes.c_uint64(seed),
                                   ctypes.byref(pairs), ctypes.byref(acc)), "knnm_round")
        return int(pairs.value), int(acc.value)

    def bf_topk(self, k: int, queries: np.ndarray | None = None, rows: np.ndarray | None = None,
                exclude_self: bool = False):
        """Exact top-k by (fp64 distance, id) against the current union (or
        the whole dataset when no merge is active)."""
        if (queries is None) == (rows is None):
            raise ValueError("pass exactly one of queries / rows")
        if queries is not None:
            q = np.ascontiguousarray(queries, dtype=np.float32)
            nq, qp, rp = q.shape[0], ptr(q), None
        else:
            r = np.ascontiguousarray(rows, dtype=np.int64)
            nq, qp, rp = r.shape[0], None, ptr(r)
        ids = np.empty((nq, k), dtype=np.int32)
        dists = np.empty((nq, k), dtype=np.float64)
        check(self._lib.knnm_bf_topk(self._h, qp, rp, nq, int(k), int(bool(exclude_self)), ptr(ids),
                                     ptr(dists)), "knnm_bf_topk")
        return ids, dists

    def phi(self) -> float:
        out = ctypes.c_double()
        check(self._lib.knnm_phi(self._h, ctypes.byref(out)), "knnm_phi")
        return float(out.value)

    PHI_SLOTS = 64  # KNNM_PHI_SLOTS

    def phi_async(self, slot: int) -> None:
        """Start phi of the current lists on a side stream (knnm_phi_async)."""
        check(self._lib.knnm_phi_async(self._h, int(slot) % self.PHI_SLOTS), "knnm_phi_async")

    def phi_fetch(self, slot: int) -> float:
        out = ctypes.c_double()
        check(self._lib.knnm_phi_fetch(self._h, int(slot) % self.PHI_SLOTS, ctypes.byref(out)),
              "knnm_phi_fetch")
        return float(out.value)

    def export(self, merge_rear: bool, on_device: bool = False):
        if on_device:
            import torch

            dev = torch.device("cuda", self.device)
            ids = torch.empty((self.n, self.k), dtype=torch.int32, device=dev)
            dists = torch.empty((self.n, self.k), dtype=torch.float64, device=dev)
            sizes = torch.empty(self.n, dtype=torch.int32, device=dev)
            self.wait_torch()  # fresh allocations: no pending torch reads of them
            check(self._lib.knnm_export_dev(self._h, int(bool(merge_rear)),
                                            ctypes.c_void_p(ids.data_ptr()),
                                            ctypes.c_void_p(dists.data_ptr()),
                                            ctypes.c_void_p(sizes.data_ptr())), "knnm_export_dev")
            self.signal_torch()  # torch work on the outputs runs after the export
            return ids, dists, sizes
        ids = _host_empty((self.n, self.k), np.int32, self.pinned_outputs)
        dists = _host_empty((self.n, self.k), np.float64, self.pinned_outputs)
        sizes = _host_empty((self.n,), np.int32, self.pinned_outputs)
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

    def set_cand_budget(self, nbytes: int) -> None:
        """Candidate-slot budget (bytes; 0 = default 40 GiB).  Rounds whose
        slots exceed it run in hood chunks (a small value forces that path)."""
        check(self._lib.knnm_set_cand_budget(self._h, int(nbytes)), "knnm_set_cand_budget")

    def wait_torch(self) -> None:
        """Order the engine's stream after work queued on torch's current
        stream of this device (tensors torch produced that the engine reads)."""
        import torch

        s = torch.cuda.current_stream(self.device)
        check(self._lib.knnm_wait_stream(self._h, ctypes.c_void_p(s.cuda_stream)), "knnm_wait_stream")

    def signal_torch(self) -> None:
        """Order torch's current stream after the engine's queued work."""
        import torch

        s = torch.cuda.current_stream(self.device)
        check(self._lib.knnm_signal_stream(self._h, ctypes.c_void_p(s.cuda_stream)),
              "knnm_signal_stream")

    def pair_dists(self, pa: np.ndarray, pb: np.ndarray) -> np.ndarray:
        """Exact reference distances of union-row pairs (pair_dists_dense)."""
        a = np.ascontiguousarray(pa, dtype=np.int32)
        b = np.ascontiguousarray(pb, dtype=np.int32)
        out = np.empty(a.shape[0], dtype=np.float64)
        check(self._lib.knnm_pair_dists(self._h, ptr(a), ptr(b), a.shape[0], ptr(out)), "knnm_pair_dists")
        return out

    def set_bf_variant(self, variant: int) -> None:
        """Brute-force route: -1 auto, 0 exact SIMT, 1 tensor cores (tcgen05)."""
        check(self._lib.knnm_set_bf_variant(self._h, int(variant)), "knnm_set_bf_variant")

    def bf_route(self) -> int:
        """Route of the last bf_topk call: 0 SIMT, 1 tensor cores."""
        r = ctypes.c_int32(0)
        check(self._lib.knnm_bf_route(self._h, ctypes.byref(r)), "knnm_bf_route")
        return int(r.value)

    def set_join_variant(self, variant: int) -> None:
        """-1 auto, 0 exact fp64 route, 1 tiled / chunked fp32-screen route, 2 tensor-core
        route (mma.sync, certified data), 3 tcgen05 lazy route (fixed-point bounds)."""
        check(self._lib.knnm_set_join_variant(self._h, int(variant)), "knnm_set_join_variant")

    def set_locality(self, iters: int) -> None:
        """Label-propagation rounds for the hood locality order (0 = id order)."""
        check(self._lib.knnm_set_locality(self._h, int(iters)), "knnm_set_locality")

    def info(self) -> dict:
        cert = ctypes.c_int32()
        dp = ctypes.c_int32()
        check(self._lib.knnm_get_info(self._h, ctypes.byref(cert), ctypes.byref(dp)), "knnm_get_info")
        return {"cert": bool(cert.value & 1), "cert_dot": bool(cert.value & 2),
                "cert_u8": bool(cert.value & 4), "dp": int(dp.value)}

    def set_u8(self, on: bool) -> None:
        """Enable/disable the u8 integer tensor-core route (next set_dataset)."""
        check(self._lib.knnm_set_u8(self._h, int(bool(on))), "knnm_set_u8")
        self.invalidate()

    # -- instrumentation ---------------------------------------------------
    def set_profiling(self, on: bool) -> None:
        check(self._lib.knnm_set_profiling(self._h, int(bool(on))), "knnm_set_profiling")

    def stats(self) -> dict:
        s = _lib.KnnmStats()
        check(self._lib.knnm_get_stats(self._h, ctypes.byref(s)), "knnm_get_stats")
        return s.as_dict()

    def reset_stats(self) -> None:
        check(self._lib.knnm_reset_stats(self._h), "knnm_reset_stats")

    def mark(self, slot: int) -> None:
        check(self._lib.knnm_mark(self._h, int(slot)), "knnm_mark")

    def elapsed_ms(self, a: int, b: int) -> float:
        out = ctypes.c_double()
        check(self._lib.knnm_elapsed(self._h, int(a), int(b), ctypes.byref(out)), "knnm_elapsed")
        return float(out.value)

    def sync(self) -> None:
        check(self._lib.knnm_sync(self._h), "knnm_sync")


# --- numpy PCG64 state hand-off (numpy/random/src/pcg64/pcg64.h) ----------
_M64 = (1 << 64) - 1
_M128 = (1 << 128) - 1
_PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645


def _pcg_split(rng):
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("device draws need a PCG64 generator (np.random.default_rng)")
    s, inc = st["state"]["state"], st["state"]["inc"]
    arr = np.array([s >> 64, s & _M64, inc >> 64, inc & _M64], dtype=np.uint64)
    return st, arr, st["has_uint32"], st["uinteger"]


def _pcg_advance(s, inc, delta):
    """pcg_advance_lcg_128: the LCG state after `delta` steps."""
    acc_mult, acc_plus, cur_mult, cur_plus = 1, 0, _PCG_MULT, inc
    while delta > 0:
        if delta & 1:
            acc_mult = (acc_mult * cur_mult) & _M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & _M128
        cur_plus = ((cur_mult + 1) * cur_plus) & _M128
        cur_mult = (cur_mult * cur_mult) & _M128
        delta >>= 1
    return (acc_mult * s + acc_plus) & _M128


def _pcg_out(s):
    x = ((s >> 64) ^ s) & _M64
    r = s >> 122
    return ((x >> r) | (x << ((64 - r) & 63))) & _M64


def _pcg_consume(rng, st, used):
    """Advance rng exactly as `used` next_uint32 calls would."""
    s, inc = st["state"]["state"], st["state"]["inc"]
    has, uint = st["has_uint32"], st["uinteger"]
    if used <= 0:
        return
    if has:
        used -= 1
        has = 0
    outs = (used + 1) // 2
    if outs:
        s = _pcg_advance(s, inc, outs)
        uint = _pcg_out(s) >> 32
        has = used % 2
    new = dict(st)
    new["state"] = {"state": s, "inc": inc}
    new["has_uint32"] = has
    new["uinteger"] = uint
    rng.bit_generator.state = new


def _host_empty(shape, dtype, pinned: bool) -> np.ndarray:
    if not pinned:
        return np.empty(shape, dtype=dtype)
    import torch

    tdt = {np.int32: torch.int32, np.float64: torch.float64}[dtype]
    return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()


def pinned_copy(a: np.ndarray) -> np.ndarray:
    """A page-locked copy of a host array (DMA at full PCIe speed)."""
    import torch

    t = torch.empty(a.shape, dtype=torch.from_numpy(np.empty(0, dtype=a.dtype)).dtype, pin_memory=True)
    out = t.numpy()
    out[...] = a
    return out


def fingerprint(a: np.ndarray) -> int:
    """Content fingerprint of a C-contiguous host array (knnm_fingerprint)."""
    a = np.ascontiguousarray(a)
    out = ctypes.c_uint64()
    check(_lib.load().knnm_fingerprint(ptr(a), a.nbytes, ctypes.byref(out)), "knnm_fingerprint")
    return int(out.value)


def _frozen(a) -> bool:
    """True when no writeable array can alias ``a``: it and every base it
    views are read-only numpy arrays (numpy refuses to make a view of a
    read-only base writeable)."""
    x = a
    while isinstance(x, np.ndarray):
        if x.flags.writeable:
            return False
        x = x.base
    return x is None


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "data_ptr") and getattr(x, "is_cuda", False)


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
