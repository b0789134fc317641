"""H-Merge: grow a graph by joint merges over an expanding random sample.

Reference behaviour: ``merge.py:74-122`` (``HierarchyLayer`` / ``Hierarchy``),
``merge.py:341-443`` (``doubling_layer_sizes`` / ``h_merge``),
``merge.py:446-467`` (first-stage descent, layer snapshots) and
``io.py:201-271`` (hierarchy directories).

Structure here: the whole schedule is resolved up front into a list of
``_Stage`` records (which members each stage adds and the seed it runs
with), then executed against the GPU ``nn_descent`` / ``j_merge``.  Layer
snapshots go through a ``_Sink`` that either keeps them in memory or writes
them to a directory (and drops intermediates from memory, as the reference
does).  The seeds come from one PCG64 stream in the reference's order --
permutation first, then one 63-bit draw per stage -- so graphs, layer
snapshots and reports are bit-identical to the reference's ``h_merge``.
"""

from __future__ import annotations

import dataclasses
import logging
import os
from dataclasses import dataclass, field

import numpy as np

from .construct import nn_descent
from .core import DistanceCounter, Metric
from .graph import KnnGraph
from .merge import MergeParams, j_merge

logger = logging.getLogger(__name__)

_SEED_HI = 2**63 - 1


@dataclass
class HierarchyLayer:
    """One layer: member ids plus its graph snapshot.  ``graph`` is None
    once the snapshot lives only on disk (``path``); ``adjacency`` is kept
    for API parity (the diversified layers are out of scope here)."""

    member_ids: np.ndarray
    graph: KnnGraph | None = None
    path: str | None = None
    adjacency: object | None = None

    @property
    def size(self) -> int:
        return int(self.member_ids.shape[0])


@dataclass
class Hierarchy:
    """Layers from the top (smallest sample) down to the full set."""

    layers: list = field(default_factory=list)
    k: int = 0
    metric: Metric = Metric.L2

    @property
    def layer_sizes(self) -> list:
        return [layer.size for layer in self.layers]

    def layer_graph(self, t: int) -> KnnGraph:
        """The layer's graph, read back from its file when it was dropped."""
        layer = self.layers[t]
        if layer.graph is not None:
            return layer.graph
        if layer.path is None:
            raise ValueError(f"layer {t} has neither a graph nor a file")
        from .io import load_graph

        return load_graph(layer.path, member_ids=layer.member_ids)

    def validate(self, n_total: int | None = None) -> None:
        sizes = np.asarray(self.layer_sizes)
        assert np.all(np.diff(sizes) > 0), "sizes not ascending"
        for t in range(len(self.layers) - 1):
            upper, lower = self.layers[t].member_ids, self.layers[t + 1].member_ids
            # both ascending: nested iff every upper id is found in lower
            at = np.searchsorted(lower, upper)
            ok = np.all(at < lower.shape[0]) and np.array_equal(lower[np.minimum(at, lower.shape[0] - 1)], upper)
            assert ok, "layer member sets are not nested"
        if n_total is not None:
            assert sizes.size and sizes[-1] == n_total, "bottom layer does not cover the dataset"


def doubling_layer_sizes(n: int, k: int, start: int = 64) -> list:
    """Layer sizes max(start, k+2) * 2^i, capped by n (reference merge.py:341-350)."""
    first = max(int(start), int(k) + 2)
    if first >= n:
        return [int(n)]
    count = 1
    while first << count < n:
        count += 1
    return [first << i for i in range(count)] + [int(n)]


@dataclass
class _Stage:
    """``members``: the ids this stage adds (the top sample for stage 0)."""

    kind: str  # "descent" | "jmerge"
    size: int
    members: np.ndarray
    seed: int

    @property
    def label(self) -> str:
        return "descent" if self.kind == "descent" else f"jmerge[{self.size}]"


def _check_sizes(sizes, n: int, k: int) -> list:
    sizes = [int(s) for s in sizes]
    if any(b <= a for a, b in zip(sizes, sizes[1:])):
        raise ValueError("layer sizes must be strictly ascending")
    if sizes[-1] != n:
        raise ValueError("the last layer size must equal the dataset size")
    if sizes[0] < k + 1:
        raise ValueError("the first layer must hold at least k+1 members")
    return sizes


def _plan(n: int, sizes: list, seed: int) -> list:
    """Stages of the schedule with the reference's draws: one permutation
    of [0, n), then a 63-bit seed per stage (merge.py:397-441, 446-454)."""
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)
    seeds = rng.integers(0, _SEED_HI, size=len(sizes))  # = one scalar draw per stage
    bounds = [0] + sizes
    stages = []
    for i, size in enumerate(sizes):
        block = np.sort(perm[bounds[i]:bounds[i + 1]])
        stages.append(_Stage("descent" if i == 0 else "jmerge", size, block, int(seeds[i])))
    return stages


class _Sink:
    """Where layer snapshots go: memory, or ``directory`` (reference
    ``_maybe_snapshot``, merge.py:457-467: intermediates are written and
    dropped, the bottom layer is written and kept; a manifest closes it)."""

    def __init__(self, hierarchy: Hierarchy, directory: str | None):
        self.h = hierarchy
        self.dir = directory

    def add(self, layer: HierarchyLayer, final: bool) -> None:
        self.h.layers.append(layer)
        if self.dir is None:
            return
        from .io import save_hierarchy_layer

        save_hierarchy_layer(self.dir, self.h, len(self.h.layers) - 1)
        if not final:
            layer.graph = None

    def close(self) -> None:
        if self.dir is not None:
            from .io import save_hierarchy_manifest

            save_hierarchy_manifest(self.dir, self.h)


def h_merge(dataset, metric: Metric, params: MergeParams, layer_sizes=None,
            counter: DistanceCounter | None = None, on_pair=None, snapshot_dir: str | None = None,
            return_report: bool = False, device: int | None = None):
    """Hierarchical construction (reference merge.py:353-443): NN-Descent on
    a random top sample, then one joint merge per layer, each adding the
    next block of the permutation.  Returns ``(graph, hierarchy)`` or, with
    ``return_report``, ``(graph, hierarchy, [(stage label, BuildReport)])``.
    Non-bottom layers keep ``k // 2`` entries per list; with
    ``snapshot_dir`` every layer is also written there (``io.load_hierarchy``
    reads it back) and intermediates are dropped from memory."""
    metric = Metric(metric)
    metric.check_kind(dataset.kind)
    n = dataset.n
    sizes = _check_sizes(doubling_layer_sizes(n, params.k) if layer_sizes is None else layer_sizes,
                         n, params.k)
    counter = DistanceCounter() if counter is None else counter
    if snapshot_dir is not None:
        os.makedirs(snapshot_dir, exist_ok=True)
    hierarchy = Hierarchy(layers=[], k=params.k, metric=metric)
    sink = _Sink(hierarchy, snapshot_dir)
    reports = []

    def descent(member_ids, seed):
        return nn_descent(dataset, metric, params.descent_params(), seed, member_ids=member_ids,
                          counter=counter, on_pair=on_pair, return_report=True, device=device)

    if len(sizes) == 1:
        # a one-layer schedule is a plain build over the whole set, seeded
        # with params.seed itself (no permutation is drawn)
        graph, rep = descent(None, params.seed)
        reports.append(("descent", rep))
        sink.add(HierarchyLayer(graph.member_ids.copy(), graph), final=True)
    else:
        keep = max(1, params.k // 2)
        graph = None
        for stage in _plan(n, sizes, params.seed):
            if stage.kind == "descent":
                graph, rep = descent(stage.members, stage.seed)
            else:
                sink.add(HierarchyLayer(graph.member_ids.copy(), graph.with_capacity(keep)), final=False)
                graph, rep = j_merge(dataset, graph, stage.members,
                                     dataclasses.replace(params, seed=stage.seed), counter=counter,
                                     on_pair=on_pair, return_report=True, device=device)
                logger.info("h_merge grew to %d members (dists=%d)", stage.size, counter.count)
            reports.append((stage.label, rep))
        sink.add(HierarchyLayer(graph.member_ids.copy(), graph), final=True)
    sink.close()
    return (graph, hierarchy, reports) if return_report else (graph, hierarchy)
