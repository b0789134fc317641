"""Quality and cost metrics (reference evaluate.py:28-55)."""

from __future__ import annotations

import numpy as np

from .core import DistanceCounter


def _as_count(counter) -> int:
    if isinstance(counter, DistanceCounter):
        return counter.count
    return int(counter)


def recall_at_k(results, truth, k: int) -> float:
    """Mean per-list overlap of evaluated vs truth top-k ids (evaluate.py:28-48)."""
    if len(results) != len(truth):
        raise ValueError(f"misaligned lists: {len(results)} results vs {len(truth)} truth")
    if len(truth) == 0:
        raise ValueError("empty evaluation")
    hits = 0
    for got, want in zip(results, truth):
        want = [int(v) for v in want]
        if len(want) < k:
            raise ValueError("truth list shorter than k")
        hits += len(set(want[:k]).intersection(int(v) for v in got[:k]))
    return hits / (len(truth) * k)


def recall_at_k_arrays(got_ids: np.ndarray, truth_ids: np.ndarray, k: int) -> float:
    """Vectorised recall@k for (n, >=k) id arrays (same value as recall_at_k
    when rows hold distinct ids)."""
    g = np.asarray(got_ids)[:, :k]
    t = np.asarray(truth_ids)[:, :k]
    hits = 0
    for j in range(k):
        hits += int(np.sum((g == t[:, j:j + 1]).any(axis=1) & (t[:, j] >= 0)))
    return hits / (t.shape[0] * k)


def scanning_rate(counter, n: int) -> float:
    """Distance evaluations relative to one full pairwise pass (evaluate.py:51-55)."""
    if n < 2:
        raise ValueError("scanning rate needs n >= 2")
    return _as_count(counter) / (n * (n - 1) / 2.0)
