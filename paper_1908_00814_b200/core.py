"""Datasets, metric tags, distance counting and seeded generators.

Host-side mirror of the reference's ``core.py`` (pkg/src/knnmerge/core.py)
restricted to the dense path the merge hot path uses: same class names,
argument meaning and error behaviour, so code written against the
reference works unchanged.  Distances on the hot path are computed by the
CUDA engine; ``distance`` here is the public scalar utility.
"""

from __future__ import annotations

import threading
from enum import IntEnum

import numpy as np

TAG_L1 = 0
TAG_L2 = 1
TAG_COSINE = 2
TAG_JACCARD = 3


class Metric(IntEnum):
    """Distance metric tag (core.py:28-51). L2 is squared euclidean."""

    L1 = TAG_L1
    L2 = TAG_L2
    COSINE = TAG_COSINE
    JACCARD = TAG_JACCARD

    @classmethod
    def from_name(cls, name: str) -> "Metric":
        try:
            return cls[name.upper()]
        except KeyError:
            raise ValueError(f"unknown metric {name!r}") from None

    @property
    def for_dense(self) -> bool:
        return self is not Metric.JACCARD

    def check_kind(self, kind: str) -> None:
        if self.for_dense and kind != "dense":
            raise ValueError(f"{self.name} requires a dense dataset, got {kind}")
        if not self.for_dense and kind != "sparse":
            raise ValueError(f"{self.name} requires a sparse dataset, got {kind}")


class DistanceCounter:
    """Monotone, lock-protected tally of metric evaluations (core.py:54-76)."""

    def __init__(self) -> None:
        self._count = 0
        self._lock = threading.Lock()

    @property
    def count(self) -> int:
        return self._count

    def add(self, n: int = 1) -> None:
        if n < 0:
            raise ValueError("counter is monotone; cannot add a negative tally")
        with self._lock:
            self._count += int(n)

    def __repr__(self) -> str:
        return f"DistanceCounter(count={self._count})"


class Dataset:
    """Dense records addressed by contiguous ids 0..n-1 (core.py:79-172).

    ``vectors`` is a C-contiguous float32 (n, d) array.  Datasets are
    immutable after construction; the engine keeps one device copy per
    Dataset and re-uses it across merges.
    """

    def __init__(self, kind, n, d, vectors=None, indptr=None, items=None):
        self.kind = kind
        self.n = int(n)
        self.d = int(d)
        self.vectors = vectors
        self.indptr = indptr
        self.items = items

    @classmethod
    def from_dense(cls, vectors, validate: bool = True) -> "Dataset":
        vectors = np.ascontiguousarray(vectors, dtype=np.float32)
        if vectors.ndim != 2:
            raise ValueError("dense data must be a 2-D array")
        ds = cls("dense", vectors.shape[0], vectors.shape[1], vectors=vectors)
        if validate:
            ds.validate()
        return ds

    def validate(self) -> None:
        if self.kind != "dense":
            raise ValueError("only dense datasets are supported on the merge path")
        if self.vectors.shape != (self.n, self.d):
            raise ValueError("dense shape mismatch")
        if not np.all(np.isfinite(self.vectors)):
            raise ValueError("dense records must be finite")

    def record(self, i: int):
        return self.vectors[i]

    def take(self, ids) -> "Dataset":
        ids = np.asarray(ids, dtype=np.int64)
        return Dataset("dense", ids.shape[0], self.d,
                       vectors=np.ascontiguousarray(self.vectors[ids]))

    def __len__(self) -> int:
        return self.n

    def __repr__(self) -> str:
        return f"Dataset(kind={self.kind!r}, n={self.n}, d={self.d})"


def distance(metric: Metric, a, b, counter: DistanceCounter) -> float:
    """metric(a, b) with the reference's arithmetic (core.py:175-197,
    _kernels.py:43-80): fp64 accumulation in index order.  ``np.cumsum`` is
    a strictly sequential left fold, so the value is bit-identical."""
    metric = Metric(metric)
    if not metric.for_dense:
        raise ValueError("only dense metrics are supported")
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    if a.ndim != 1 or b.ndim != 1:
        raise ValueError("dense records must be 1-D vectors")
    if a.shape[0] != b.shape[0]:
        raise ValueError(f"dimension mismatch: {a.shape[0]} vs {b.shape[0]}")
    x = a.astype(np.float64)
    y = b.astype(np.float64)
    if a.shape[0] == 0:
        d = 0.0 if metric != Metric.COSINE else 0.0
    elif metric == Metric.L2:
        df = x - y
        d = float(np.cumsum(df * df)[-1])
    elif metric == Metric.L1:
        d = float(np.cumsum(np.abs(x - y))[-1])
    else:
        dot = float(np.cumsum(x * y)[-1])
        na = float(np.cumsum(x * x)[-1])
        nb = float(np.cumsum(y * y)[-1])
        if na == 0.0 or nb == 0.0:
            d = 0.0 if na == nb else 1.0
        elif dot > 0.0 and dot * dot >= na * nb:
            d = 0.0
        else:
            d = 1.0 - dot / (np.sqrt(na) * np.sqrt(nb))
            d = 0.0 if d < 0.0 else float(d)
    counter.add(1)
    return d


def generate_uniform(n: int, d: int, seed: int) -> Dataset:
    """n x d, i.i.d. U[0,1) float32 from PCG64 (core.py:200-205)."""
    if n < 1 or d < 1:
        raise ValueError("n and d must be >= 1")
    rng = np.random.default_rng(seed)
    return _owned(rng.random((n, d), dtype=np.float32))


def sample_distinct(rng, n: int, k: int, exclude: int = -1) -> np.ndarray:
    """k distinct draws from 0..n-1, optionally excluding one value
    (core.py:222-230; same PCG64 call, so the same stream)."""
    pool = n - 1 if 0 <= exclude < n else n
    if k > pool:
        raise ValueError("not enough values to sample from")
    out = rng.choice(pool, size=k, replace=False).astype(np.int64)
    if 0 <= exclude < n:
        out[out >= exclude] += 1
    return out


def sample_distinct_rows(rng, n: int, k: int, exclude: np.ndarray) -> np.ndarray:
    """[sample_distinct(rng, n, k, exclude=e) for e in exclude] as an
    (len(exclude), k) int64 array, computed natively (libknnm.so) with the
    same PCG64 stream; rng ends in the identical state."""
    import ctypes

    from . import _lib
    from .engine import _pcg_split

    exclude = np.ascontiguousarray(exclude, dtype=np.int32)
    out = np.empty((exclude.shape[0], k), dtype=np.int64)
    st, arr, has, uint = _pcg_split(rng)
    h = ctypes.c_int32(int(has))
    u = ctypes.c_uint32(int(uint))
    _lib.check(_lib.load().knnm_sample_distinct_rows(_lib.ptr(arr), ctypes.byref(h), ctypes.byref(u),
                                                     int(n), int(k), _lib.ptr(exclude),
                                                     exclude.shape[0], _lib.ptr(out)),
               "knnm_sample_distinct_rows")
    new = dict(st)
    new["state"] = {"state": (int(arr[0]) << 64) | int(arr[1]), "inc": st["state"]["inc"]}
    new["has_uint32"] = int(h.value)
    new["uinteger"] = int(u.value)
    rng.bit_generator.state = new
    return out


# ---------------------------------------------------------------------------
# Synthetic stand-ins for the BASELINE.json configs.  The
# reference ships only generate_uniform; these restate the configs'
# distributions with PCG64 so every run is seeded and reproducible.
# ---------------------------------------------------------------------------


def _owned(x: np.ndarray) -> Dataset:
    """A Dataset over an array only it holds, made read-only: the engine
    then trusts its device copy by identity (no fingerprint per merge)."""
    x.flags.writeable = False
    return Dataset.from_dense(x, validate=False)


def _chunked_gmm(rng, n, d, centres, sigma, chunk=1 << 16):
    out = np.empty((n, d), dtype=np.float32)
    labels = rng.integers(0, centres.shape[0], size=n)
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        noise = rng.standard_normal((hi - lo, d), dtype=np.float32) * np.float32(sigma)
        out[lo:hi] = centres[labels[lo:hi]] + noise
    return out


def generate_int_gmm(n: int, d: int = 128, n_centres: int = 1000, sigma: float = 20.0,
                     seed: int = 7) -> Dataset:
    """Config 2/5 stand-in for SIFT: GMM with centres U[0,255]^d, sigma 20,
    clipped to [0, 255] and rounded to integers (exact in fp32)."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, 255.0, size=(n_centres, d)).astype(np.float32)
    x = _chunked_gmm(rng, n, d, centres, sigma)
    np.clip(x, 0.0, 255.0, out=x)
    np.rint(x, out=x)
    return _owned(x)


def generate_unit_gmm(n: int, d: int = 960, n_centres: int = 500, sigma: float = 0.05,
                      seed: int = 7) -> Dataset:
    """Config 3 stand-in for GIST: centres U[0,1]^d, sigma 0.05, clipped to [0,1]."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, 1.0, size=(n_centres, d)).astype(np.float32)
    x = _chunked_gmm(rng, n, d, centres, sigma)
    np.clip(x, 0.0, 1.0, out=x)
    return _owned(x)


def generate_sphere_gmm(n: int, d: int = 100, n_centres: int = 2000, sigma: float = 0.3,
                        seed: int = 7) -> Dataset:
    """Config 4 stand-in for GloVe (cosine): centres N(0, I), sigma 0.3,
    rows L2-normalised."""
    rng = np.random.default_rng(seed)
    centres = rng.standard_normal((n_centres, d)).astype(np.float32)
    x = _chunked_gmm(rng, n, d, centres, sigma)
    x /= np.linalg.norm(x, axis=1, keepdims=True).astype(np.float32)
    return _owned(x)
