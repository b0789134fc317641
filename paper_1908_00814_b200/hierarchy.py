"""H-Merge: hierarchical construction by repeated joint merges (reference
merge.py:74-122, 341-454).  A pure caller of the GPU ``j_merge`` and
``nn_descent``; every draw follows the reference, so graphs and reports are
bit-identical to the reference's ``h_merge``."""

from __future__ import annotations

import dataclasses
import logging
from dataclasses import dataclass, field

import numpy as np

from .construct import nn_descent
from .core import DistanceCounter, Metric
from .graph import KnnGraph
from .merge import MergeParams, j_merge

logger = logging.getLogger(__name__)


@dataclass
class HierarchyLayer:
    """One layer: member ids and the (k/2-truncated) graph snapshot."""

    member_ids: np.ndarray
    graph: KnnGraph | None = None
    path: str | None = None
    adjacency: object | None = None

    @property
    def size(self) -> int:
        return self.member_ids.shape[0]


@dataclass
class Hierarchy:
    """Layers ordered top (smallest) to bottom (full set)."""

    layers: list = field(default_factory=list)
    k: int = 0
    metric: Metric = Metric.L2

    @property
    def layer_sizes(self) -> list:
        return [layer.size for layer in self.layers]

    def layer_graph(self, t: int) -> KnnGraph:
        layer = self.layers[t]
        if layer.graph is not None:
            return layer.graph
        if layer.path is None:
            raise ValueError(f"layer {t} has neither a graph nor a file")
        from .io import load_graph

        return load_graph(layer.path, member_ids=layer.member_ids)

    def validate(self, n_total: int | None = None) -> None:
        sizes = self.layer_sizes
        assert all(a < b for a, b in zip(sizes, sizes[1:])), "sizes not ascending"
        for upper, lower in zip(self.layers, self.layers[1:]):
            assert np.all(np.isin(upper.member_ids, lower.member_ids)), "layer member sets are not nested"
        if n_total is not None:
            assert sizes[-1] == n_total, "bottom layer does not cover the dataset"


def doubling_layer_sizes(n: int, k: int, start: int = 64) -> list:
    """Block sizes doubling from max(start, k+2) until they cover n (merge.py:341-350)."""
    first = max(start, k + 2)
    if first >= n:
        return [n]
    sizes = [first]
    while sizes[-1] * 2 < n:
        sizes.append(sizes[-1] * 2)
    sizes.append(n)
    return sizes


def h_merge(dataset, metric: Metric, params: MergeParams, layer_sizes=None,
            counter: DistanceCounter | None = None, on_pair=None, snapshot_dir: str | None = None,
            return_report: bool = False, device: int | None = None):
    """Grow a graph by joint merges over an expanding random sample
    (merge.py:353-443); returns (graph, hierarchy[, reports])."""
    if snapshot_dir is not None:
        raise NotImplementedError("layer snapshots to disk are not supported")
    metric = Metric(metric)
    metric.check_kind(dataset.kind)
    n = dataset.n
    if layer_sizes is None:
        layer_sizes = doubling_layer_sizes(n, params.k)
    layer_sizes = [int(s) for s in layer_sizes]
    if any(a >= b for a, b in zip(layer_sizes, layer_sizes[1:])):
        raise ValueError("layer sizes must be strictly ascending")
    if layer_sizes[-1] != n:
        raise ValueError("the last layer size must equal the dataset size")
    if layer_sizes[0] < params.k + 1:
        raise ValueError("the first layer must hold at least k+1 members")
    if counter is None:
        counter = DistanceCounter()
    rng = np.random.default_rng(params.seed)
    reports = []
    if len(layer_sizes) == 1:
        graph, rep = nn_descent(dataset, metric, params.descent_params(), params.seed,
                                counter=counter, on_pair=on_pair, return_report=True, device=device)
        reports.append(("descent", rep))
        hierarchy = Hierarchy(layers=[HierarchyLayer(graph.member_ids.copy(), graph)], k=params.k,
                              metric=metric)
        return (graph, hierarchy, reports) if return_report else (graph, hierarchy)

    perm = rng.permutation(n)
    top_ids = np.sort(perm[: layer_sizes[0]])
    seed = int(rng.integers(0, 2**63 - 1))  # nn_descent_stage (merge.py:446-454)
    graph, rep = nn_descent(dataset, metric, params.descent_params(), seed, member_ids=top_ids,
                            counter=counter, on_pair=on_pair, return_report=True, device=device)
    reports.append(("descent", rep))
    hierarchy = Hierarchy(layers=[], k=params.k, metric=metric)
    half = max(1, params.k // 2)
    for step, size in enumerate(layer_sizes[1:]):
        hierarchy.layers.append(HierarchyLayer(graph.member_ids.copy(), graph.with_capacity(half)))
        block = np.sort(perm[layer_sizes[step]:size])
        step_params = dataclasses.replace(params, seed=int(rng.integers(0, 2**63 - 1)))
        graph, rep = j_merge(dataset, graph, block, step_params, counter=counter, on_pair=on_pair,
                             return_report=True, device=device)
        reports.append((f"jmerge[{size}]", rep))
        logger.info("h_merge grew to %d members (dists=%d)", size, counter.count)
    hierarchy.layers.append(HierarchyLayer(graph.member_ids.copy(), graph))
    return (graph, hierarchy, reports) if return_report else (graph, hierarchy)
