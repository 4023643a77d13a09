"""Clique sinks, subtree roots and the whole-graph enumerators
(reference mce/bk.py).

``CliqueSink`` and the root extractors are host-side data plumbing with the
reference's exact semantics.  ``bk_pivot`` / ``bk_basic`` enumerate through
the GPU engine (``scheduler.run``): the clique set of a graph does not
depend on the traversal, so they return the reference's count and cliques.
The brute-force ``oracle_enumerate`` of the reference is test
infrastructure and lives in ``oracle/`` (not in the product).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Iterator

import numpy as np

from paper_2212_01473_b200.graph import Graph


class CliqueSink:
    """Receives maximal cliques: always counts, optionally collects sorted
    tuples up to ``collect_limit`` (reference bk.py:23-58)."""

    __slots__ = ("collect_limit", "total", "collected")

    def __init__(self, collect_limit: int | None = None) -> None:
        self.collect_limit = collect_limit
        self.total = 0
        self.collected: list[tuple[int, ...]] = []

    @classmethod
    def counting(cls) -> "CliqueSink":
        return cls(collect_limit=None)

    @classmethod
    def collecting(cls, limit: int = 1 << 20) -> "CliqueSink":
        return cls(collect_limit=limit)

    def report(self, vertices: Iterable[int]) -> None:
        self.total += 1
        if self.collect_limit is not None and len(self.collected) < self.collect_limit:
            self.collected.append(tuple(sorted(int(v) for v in vertices)))

    def merge(self, other: "CliqueSink") -> None:
        self.total += other.total
        if self.collect_limit is not None:
            room = self.collect_limit - len(self.collected)
            if room > 0:
                self.collected.extend(other.collected[:room])

    def clique_set(self) -> set[tuple[int, ...]]:
        return set(self.collected)


@dataclass(frozen=True)
class RootTask:
    """Seed state of one independent subtree (reference bk.py:62-73)."""

    root_vertices: tuple[int, ...]
    P: np.ndarray
    X: np.ndarray
    origin_index: int


def first_level_root(g: Graph, v: int) -> RootTask:
    """Per-vertex root: P = later neighbours, X = earlier (bk.py:186-190)."""
    adj = g.neighbors(v)
    cut = int(np.searchsorted(adj, v))
    return RootTask((v,), adj[cut:].copy(), adj[:cut].copy(), origin_index=v)


def first_level_roots(g: Graph) -> Iterator[RootTask]:
    for v in range(g.num_vertices):
        yield first_level_root(g, v)


def second_level_root(g: Graph, edge_index: int) -> RootTask:
    """Per-edge root: common neighbours after / before the later endpoint
    (bk.py:198-204)."""
    u, v = (int(a) for a in g.edges()[edge_index])
    common = np.intersect1d(g.neighbors(u), g.neighbors(v), assume_unique=True)
    cut = int(np.searchsorted(common, max(u, v)))
    return RootTask((u, v), common[cut:].copy(), common[:cut].copy(), origin_index=edge_index)


def second_level_roots(g: Graph) -> Iterator[RootTask]:
    for e in range(len(g.edges())):
        yield second_level_root(g, e)


def _enumerate_whole_graph(g: Graph, sink: CliqueSink, metrics: dict | None) -> int:
    from paper_2212_01473_b200.graph import preprocess
    from paper_2212_01473_b200.scheduler import RunConfig, run

    if g.num_vertices == 0:
        if metrics is not None:
            metrics["nodes"] = 0
        return sink.total
    g2, order, st = preprocess(g)
    inner = CliqueSink(collect_limit=sink.collect_limit)
    res = run(g2, st, RunConfig(workers=0), sink=inner)
    inverse = np.argsort(order.position)
    sink.total += inner.total
    if sink.collect_limit is not None:
        room = sink.collect_limit - len(sink.collected)
        for c in inner.collected[:max(room, 0)]:
            sink.collected.append(tuple(sorted(int(inverse[v]) for v in c)))
    if metrics is not None:
        metrics["nodes"] = res.nodes_total
    return sink.total


ORACLE_MAX_VERTICES = 24


def adjacency_masks(g: Graph) -> list[int]:
    """Neighbourhood of every vertex as an int bit mask (reference bk.py:113-121)."""
    ro, ci = g.row_offsets, g.col_indices
    out = []
    for v in range(g.num_vertices):
        m = 0
        for u in ci[ro[v]:ro[v + 1]]:
            m |= 1 << int(u)
        out.append(m)
    return out


def oracle_enumerate(g: Graph) -> list[tuple[int, ...]]:
    """Maximal cliques by testing every vertex subset, for n <= 24 (reference
    bk.py:212-241): the independent check behind ``mce oracle-check``.  All
    2^n subsets at once as uint32 masks: a subset is a clique when every
    member's closed neighbourhood covers it, maximal when no outside vertex
    is adjacent to all of it."""
    n = g.num_vertices
    if n > ORACLE_MAX_VERTICES:
        raise ValueError(f"oracle limited to {ORACLE_MAX_VERTICES} vertices, got {n}")
    if n == 0:
        return []
    nbr = np.array(adjacency_masks(g), dtype=np.uint32)
    subsets = np.arange(1 << n, dtype=np.uint32)
    clique = np.ones(subsets.size, dtype=bool)
    grow = np.zeros(subsets.size, dtype=bool)
    for v in range(n):
        bit = np.uint32(1 << v)
        member = (subsets & bit) != 0
        closed = nbr[v] | bit
        clique &= ~member | ((subsets & ~closed) == 0)
        grow |= ~member & ((subsets & ~nbr[v]) == 0)
    keep = subsets[clique & ~grow & (subsets != 0)]
    return sorted(tuple(v for v in range(n) if (int(s) >> v) & 1) for s in keep)


def bk_pivot(g: Graph, sink: CliqueSink, metrics: dict | None = None) -> int:
    """All maximal cliques of ``g`` (reference bk.py:153-183) via the GPU
    engine; cliques are reported in ``g``'s labels.  ``metrics["nodes"]`` is
    the engine's pivoting traversal over the degeneracy-ordered subtrees --
    the reference's single whole-graph recursion pivots once more at the top
    and breaks ties by global id, so its total differs (both never exceed
    bk_basic's)."""
    return _enumerate_whole_graph(g, sink, metrics)


def bk_basic(g: Graph, sink: CliqueSink, metrics: dict | None = None) -> int:
    """Plain Bron-Kerbosch without pivoting (reference bk.py:124-150), on the GPU.

    The reference's recursion from (R = {}, P = V, X = {}) branches on every
    vertex in id order, so its first level IS the per-vertex subtree
    decomposition in the graph's own order: vertex v's subtree starts from
    P = N(v) & {u > v}, X = N(v) & {u < v}.  The engine runs exactly those
    subtrees (no degeneracy reordering) with ``pivot=False``, and the node
    total is the reference's: every subtree node plus the top-level call."""
    from paper_2212_01473_b200.graph import GraphStats
    from paper_2212_01473_b200.scheduler import RunConfig, run

    n = g.num_vertices
    if n == 0:
        if metrics is not None:
            metrics["nodes"] = 0
        return sink.total
    ro = g.row_offsets
    ci = g.col_indices
    later = int(max(ro[v + 1] - ro[v] - np.searchsorted(ci[ro[v]:ro[v + 1]], v, side="right")
                    for v in range(n)))
    st = GraphStats(n, len(ci) // 2, int(np.diff(ro).max()), later)
    res = run(g, st, RunConfig(workers=0, roots="l1", induced="ipx", worker_list=False),
              sink=sink, pivot=False)
    if metrics is not None:
        metrics["nodes"] = res.nodes_total + 1  # + the top-level call go([], V, {})
    return sink.total
