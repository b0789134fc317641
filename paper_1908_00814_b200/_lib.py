"""ctypes binding of libknnm.so (include/knnm.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_1908_00814_b200.build``).  There is no fallback: if the
library or a CUDA device is missing, every engine call raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# KNNM_LIB: alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("KNNM_LIB") or os.path.join(_HERE, "libknnm.so")

KNNM_OK = 0
_ERRORS = {
    -1: "CUDA failure",
    -2: "invalid argument",
    -3: "call out of order",
    -4: "device out of memory",
    -5: "input exceeds a supported bound",
}

# Every symbol declared in include/knnm.h, with (restype, argtypes).
P = ctypes.c_void_p
I32 = ctypes.c_int32
I64 = ctypes.c_int64
U64 = ctypes.c_uint64
PI64 = ctypes.POINTER(ctypes.c_int64)
PDBL = ctypes.POINTER(ctypes.c_double)


class KnnmStats(ctypes.Structure):
    _fields_ = [
        ("join_ms", ctypes.c_double),
        ("reverse_ms", ctypes.c_double),
        ("assemble_ms", ctypes.c_double),
        ("update_ms", ctypes.c_double),
        ("other_ms", ctypes.c_double),
        ("join_launches", I64),
        ("pairs", I64),
        ("init_evals", I64),
        ("members", I64),
        ("candidates", I64),
        ("accepted", I64),
        ("rounds", I64),
        ("exact_evals", I64),
        ("launches", I64),
        ("h2d_bytes", I64),
        ("join_redos", I64),
        ("d2h_bytes", I64),
        ("join_kernel_ms", ctypes.c_double),
        ("written_slots", I64),
        ("join_row_bytes", I64),
        ("heavy_rev_rows", I64),
        ("seg_hub_rows", I64),
        ("apply_rows_in", I64),
        ("apply_rows_out", I64),
        ("apply_kernel_ms", ctypes.c_double),
        ("active_hoods", I64),
        ("bf_tc_launches", I64),
        ("lazy_batches", I64),
        ("tc_join_launches", I64),
        ("dense_join_launches", I64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


SIGNATURES = {
    "knnm_last_error": (ctypes.c_char_p, []),
    "knnm_version": (ctypes.c_int, []),
    "knnm_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(P)]),
    "knnm_destroy": (ctypes.c_int, [P]),
    "knnm_set_dataset": (ctypes.c_int, [P, P, I64, I32, I32]),
    "knnm_fingerprint": (ctypes.c_int, [P, I64, ctypes.POINTER(U64)]),
    "knnm_begin": (ctypes.c_int, [P, P, I64, P, I32]),
    "knnm_load_graph": (ctypes.c_int, [P, P, I64, P, P, P, I32, I32]),
    "knnm_load_graph_dev": (ctypes.c_int, [P, P, I64, P, P, P, I32, I32]),
    "knnm_insert_directed": (ctypes.c_int, [P, P, P, I64, PI64]),
    "knnm_insert_rows": (ctypes.c_int, [P, P, I64, I32, P, PI64]),
    "knnm_draws_load": (ctypes.c_int, [P, P, I64, I32, P, PI64]),
    "knnm_draws_replace": (ctypes.c_int, [P, P, I64, P, P, PI64]),
    "knnm_draws_insert": (ctypes.c_int, [P, P, P, I64, PI64]),
    "knnm_draws_insert_range": (ctypes.c_int, [P, P, P, I64, I64, I64, PI64]),
    "knnm_draws_gen": (ctypes.c_int, [P, P, I32, ctypes.c_uint32, U64, I64, I32, PI64, P, PI64]),
    "knnm_draws_regen": (ctypes.c_int, [P, P, I32, ctypes.c_uint32, U64, P, I64, PI64, P, PI64]),
    "knnm_merge_members": (ctypes.c_int, [P, I64, P, I64, P, P, P, ctypes.POINTER(I64),
                                          ctypes.POINTER(I32), P]),
    "knnm_sample_distinct_rows": (ctypes.c_int, [P, ctypes.POINTER(I32), ctypes.POINTER(ctypes.c_uint32),
                                                 I64, I32, P, I64, P]),
    "knnm_round": (ctypes.c_int, [P, I32, I32, U64, PI64, PI64]),
    "knnm_set_shard": (ctypes.c_int, [P, I64, I64]),
    "knnm_round_local": (ctypes.c_int, [P, I32, I32, U64, PI64]),
    "knnm_local_chunks": (ctypes.c_int, [P, ctypes.POINTER(I32)]),
    "knnm_local_join": (ctypes.c_int, [P, I32]),
    "knnm_set_cand_budget": (ctypes.c_int, [P, I64]),
    "knnm_wait_stream": (ctypes.c_int, [P, P]),
    "knnm_signal_stream": (ctypes.c_int, [P, P]),
    "knnm_local_views": (ctypes.c_int, [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P)]),
    "knnm_local_compact": (ctypes.c_int, [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P),
                                          ctypes.POINTER(ctypes.c_int64)]),
    "knnm_round_apply": (ctypes.c_int, [P, I32, P, P, P, P, PI64]),
    "knnm_pack_rows": (ctypes.c_int, [P, I32, ctypes.POINTER(P), ctypes.POINTER(ctypes.c_int64),
                                      ctypes.POINTER(I32)]),
    "knnm_unpack_rows": (ctypes.c_int, [P, P, I64]),
    "knnm_state_views": (ctypes.c_int, [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P)]),
    "knnm_bf_topk": (ctypes.c_int, [P, P, P, I64, I32, I32, P, P]),
    "knnm_set_bf_variant": (ctypes.c_int, [P, I32]),
    "knnm_pair_dists": (ctypes.c_int, [P, P, P, I64, P]),
    "knnm_bf_route": (ctypes.c_int, [P, P]),
    "knnm_phi": (ctypes.c_int, [P, PDBL]),
    "knnm_phi_async": (ctypes.c_int, [P, I32]),
    "knnm_phi_fetch": (ctypes.c_int, [P, I32, PDBL]),
    "knnm_export": (ctypes.c_int, [P, I32, P, P, P]),
    "knnm_export_dev": (ctypes.c_int, [P, I32, P, P, P]),
    "knnm_get_state": (ctypes.c_int, [P, P, P, P, P]),
    "knnm_set_capture": (ctypes.c_int, [P, I32]),
    "knnm_capture_count": (ctypes.c_int, [P, PI64]),
    "knnm_capture_fetch": (ctypes.c_int, [P, P, P, P, I64]),
    "knnm_set_join_variant": (ctypes.c_int, [P, I32]),
    "knnm_set_sample": (ctypes.c_int, [P, I32]),
    "knnm_set_locality": (ctypes.c_int, [P, I32]),
    "knnm_set_u8": (ctypes.c_int, [P, I32]),
    "knnm_get_info": (ctypes.c_int, [P, ctypes.POINTER(I32), ctypes.POINTER(I32)]),
    "knnm_set_profiling": (ctypes.c_int, [P, I32]),
    "knnm_get_stats": (ctypes.c_int, [P, ctypes.POINTER(KnnmStats)]),
    "knnm_reset_stats": (ctypes.c_int, [P]),
    "knnm_mark": (ctypes.c_int, [P, I32]),
    "knnm_elapsed": (ctypes.c_int, [P, I32, I32, PDBL]),
    "knnm_sync": (ctypes.c_int, [P]),
}

_lib = None


class KnnmError(RuntimeError):
    """A CUDA-side failure reported by libknnm.so."""


def load():
    """Load libknnm.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise KnnmError(
                f"{LIB_PATH} is missing; build it with __graft_entry__.build() "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(code: int, what: str) -> None:
    if code != KNNM_OK:
        msg = load().knnm_last_error().decode(errors="replace")
        kind = _ERRORS.get(code, f"error {code}")
        if code == -2:
            raise ValueError(f"{what}: {kind}: {msg}")
        raise KnnmError(f"{what}: {kind}: {msg}")


def ptr(a: np.ndarray):
    if not a.flags.c_contiguous:
        raise ValueError("array must be C-contiguous")
    return a.ctypes.data_as(ctypes.c_void_p)
