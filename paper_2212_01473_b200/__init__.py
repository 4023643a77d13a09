"""B200-native maximal clique enumeration (the hot path of arXiv:2212.01473).

Drop-in for the reference ``mce`` package's path: graph load and ordering,
the enumerate/count entry points and the clique output format, with the
work done by hand-written sm_100a CUDA kernels in libmce_b200.so (C ABI in
include/mce_b200.h, bound with ctypes).  There is no CPU fallback.

    from paper_2212_01473_b200 import RunConfig, parse_edge_list, preprocess, run
    g = parse_edge_list(open("graph.txt"))
    g2, order, stats = preprocess(g)
    result = run(g2, stats, RunConfig())
    print(result.clique_count, result.report().load_ratio)
"""

from paper_2212_01473_b200._lib import CapacityError, MceError
from paper_2212_01473_b200.bk import (
    CliqueSink,
    RootTask,
    bk_basic,
    bk_pivot,
    first_level_root,
    first_level_roots,
    second_level_root,
    second_level_roots,
)
from paper_2212_01473_b200.graph import (
    DegeneracyOrder,
    EdgeListParseError,
    Graph,
    GraphStats,
    degeneracy_order,
    from_device_edges,
    from_edges,
    parse_edge_list,
    preprocess,
    reorder,
    stats,
)
from paper_2212_01473_b200.metrics import MetricsReport, WorkerMetrics, aggregate
from paper_2212_01473_b200.scheduler import (
    Backoff,
    RunConfig,
    RunResult,
    choose_induced_mode,
    run,
)

__version__ = "0.1.0"

__all__ = [
    "Backoff", "CapacityError", "CliqueSink", "DegeneracyOrder", "EdgeListParseError",
    "Graph", "GraphStats", "MceError", "MetricsReport", "RootTask", "RunConfig", "RunResult",
    "WorkerMetrics", "aggregate", "bk_basic", "bk_pivot", "choose_induced_mode",
    "degeneracy_order", "first_level_root", "first_level_roots", "from_device_edges",
    "from_edges", "parse_edge_list", "preprocess", "reorder", "run", "second_level_root",
    "second_level_roots", "stats",
]
