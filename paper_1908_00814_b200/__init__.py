"""B200-native S-Merge / J-Merge for k-NN graphs (arXiv 1908.00814).

Drop-in for the reference package ``knnmerge`` on its merge hot path: the
same public names and signatures for ``s_merge``, ``j_merge``,
``nn_descent`` and the containers they exchange, backed by hand-written
sm_100a CUDA kernels in ``libknnm.so`` (see include/knnm.h).
"""

from .construct import (
    BuildReport,
    DescentParams,
    RoundStats,
    brute_force_graph,
    brute_force_queries,
    nn_descent,
)
from .core import (
    Dataset,
    DistanceCounter,
    Metric,
    distance,
    generate_int_gmm,
    generate_sphere_gmm,
    generate_uniform,
    generate_unit_gmm,
    sample_distinct,
)
from .evaluate import recall_at_k, recall_at_k_arrays, scanning_rate
from .graph import KnnGraph, Neighbor, NeighborList, SplitGraph, phi, split, update_nn
from .hierarchy import Hierarchy, HierarchyLayer, doubling_layer_sizes, h_merge
from .merge import MergeParams, j_merge, merge_rear, s_merge

__version__ = "0.1.0"

__all__ = [
    "BuildReport",
    "Dataset",
    "DescentParams",
    "DistanceCounter",
    "Hierarchy",
    "HierarchyLayer",
    "KnnGraph",
    "MergeParams",
    "Metric",
    "Neighbor",
    "NeighborList",
    "RoundStats",
    "brute_force_graph",
    "brute_force_queries",
    "SplitGraph",
    "distance",
    "doubling_layer_sizes",
    "h_merge",
    "generate_int_gmm",
    "generate_sphere_gmm",
    "generate_uniform",
    "generate_unit_gmm",
    "j_merge",
    "merge_rear",
    "nn_descent",
    "phi",
    "recall_at_k",
    "recall_at_k_arrays",
    "s_merge",
    "sample_distinct",
    "scanning_rate",
    "split",
    "update_nn",
]
