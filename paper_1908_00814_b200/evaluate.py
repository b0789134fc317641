"""Quality and cost metrics of a build (reference evaluate.py:28-55):
recall against exact ground truth and the scanning rate (distance
evaluations relative to one all-pairs pass)."""

from __future__ import annotations

import numpy as np

from .core import DistanceCounter


def _evals(counter) -> int:
    return counter.count if isinstance(counter, DistanceCounter) else int(counter)


def recall_at_k(results, truth, k: int) -> float:
    """Fraction of the true top-k ids found in each result's first k, over
    aligned sequences of id lists (evaluate.py:28-48; same errors)."""
    if len(results) != len(truth):
        raise ValueError(f"misaligned lists: {len(results)} results vs {len(truth)} truth")
    if len(truth) == 0:
        raise ValueError("empty evaluation")
    found = 0
    for got, want in zip(results, truth):
        if len(want) < k:
            raise ValueError("truth list shorter than k")
        top = {int(v) for v in list(want)[:k]}
        found += sum(1 for v in {int(x) for x in list(got)[:k]} if v in top)
    return found / (k * len(truth))


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
    """Evaluations / (n (n - 1) / 2) (evaluate.py:51-55)."""
    if n < 2:
        raise ValueError("scanning rate needs n >= 2")
    return _evals(counter) * 2.0 / (n * (n - 1))
