"""B200-native exact triangle counter (GPU forward algorithm, Polak arXiv:1503.00576).

Drop-in for the reference ``tricount`` hot path: the same entry points
(``preprocess``, ``count_triangles``, ``count_partitioned``, ``count_with_timings``,
``intersect_count``, ``PartitionPlan``, ``PhaseTimings``) over the same containers
(``EdgeArray``, ``OrientedGraph``), computed by hand-written sm_100a kernels in
libtcb200.so (include/tricount_b200.h).  There is no CPU fallback.
"""
from .count import (
    PartitionPlan,
    PhaseTimings,
    count_device,
    count_partitioned,
    count_triangles,
    count_with_timings,
    count_with_timings_device,
    default_workers,
    intersect_count,
    merge_work,
    preprocess_device,
    schedule_bytes,
    warm_kernel,
)
from .graph import (
    AsymmetricEdgeError,
    DegreeOrder,
    DuplicateEdgeError,
    EdgeArray,
    GraphValidationError,
    OrientedGraph,
    SelfLoopError,
    degrees_of,
    max_out_degree_bound,
    validate_edge_array,
    validate_oriented_graph,
)
from .metrics import CountOverflowError, InconsistentCountsError, transitivity, wedge_count
from .preprocess import build_node_array, orient_and_compact, preprocess, sort_edges, unzip

__version__ = "0.1.0"

__all__ = [
    "DegreeOrder", "EdgeArray", "OrientedGraph", "PartitionPlan", "PhaseTimings",
    "build_node_array", "count_device", "count_partitioned", "count_triangles",
    "count_with_timings", "count_with_timings_device", "default_workers", "degrees_of",
    "intersect_count", "max_out_degree_bound", "merge_work", "orient_and_compact",
    "preprocess", "preprocess_device", "schedule_bytes", "sort_edges", "unzip", "validate_oriented_graph",
    "warm_kernel", "AsymmetricEdgeError", "DuplicateEdgeError", "GraphValidationError",
    "SelfLoopError", "validate_edge_array", "CountOverflowError", "InconsistentCountsError",
    "transitivity", "wedge_count",
]
