"""Graph ingestion, canonicalisation, statistics and degeneracy ordering.

Same API as the reference ``mce.graph`` (reference graph.py:1-243): a
canonical undirected simple graph in CSR form with strictly ascending
adjacency rows.  The difference is where the work happens: canonicalisation
(``from_edges``), degeneracy ordering and reordering run as CUDA kernels in
libmce_b200.so and the graph stays resident in HBM; the numpy CSR arrays of
the reference's dataclass are materialised only when host code reads them.

``degeneracy_order`` takes ``method``:

* ``"parallel"`` -- bucket peeling on the GPU: every vertex whose
  current degree is at most the peel level leaves in the same round, ranked
  by id.  A valid degeneracy ordering with exactly the reference's
  degeneracy ``d`` (so |P| <= d for every first-level root), but not the same
  permutation.
* ``"async"`` -- peeling without rounds inside a level: the claimed
  vertices' adjacency is a device-wide task queue, and a vertex is claimed
  (and given its position) the moment a decrement takes its degree to the
  level.  A valid degeneracy ordering with the reference's degeneracy, in a
  data-dependent order that can differ from run to run; the fastest method
  and the default.
* ``"exact"`` -- the reference's own order (minimum current degree, ties to
  the smallest id; graph.py:183-210), computed by a single-CTA kernel;
  positions are bit-identical to the reference.

Clique results never depend on the method: counts, size histograms and the
clique-set hash (over original labels) are identical; only traversal-tree
sizes differ.
"""

from __future__ import annotations

import ctypes
from typing import IO, Iterable

import numpy as np

from paper_2212_01473_b200 import _lib

ORDER_METHODS = {"parallel": 0, "exact": 1, "async": 2}


class EdgeListParseError(ValueError):
    """Malformed edge-list input; carries the 1-based line number
    (reference graph.py:19-24)."""

    def __init__(self, line_no: int, message: str) -> None:
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


class _DeviceGraph:
    """Owns one ``mce_graph*`` (device-resident CSR)."""

    __slots__ = ("handle",)

    def __init__(self, handle: ctypes.c_void_p) -> None:
        self.handle = handle

    def __del__(self) -> None:
        h, self.handle = self.handle, None
        if h and _lib._lib is not None:
            _lib._lib.mce_graph_free(h)

    def info(self) -> dict:
        vals = [ctypes.c_int64() for _ in range(5)]
        _lib.check(_lib.lib().mce_graph_info(self.handle, *[ctypes.byref(v) for v in vals]),
                   "mce_graph_info")
        n, nnz, maxdeg, later, earlier = (v.value for v in vals)
        return {"n": n, "nnz": nnz, "max_degree": maxdeg, "max_later": later,
                "max_earlier": earlier}


class Graph:
    """Undirected simple graph in CSR form (reference graph.py:28-82).

    ``row_offsets`` (n+1) and ``col_indices`` (2m, rows strictly ascending)
    are numpy views materialised on demand from the device copy; ``labels``
    (original vertex id of every vertex) is set on reordered graphs.
    """

    def __init__(self, num_vertices: int, row_offsets: np.ndarray | None = None,
                 col_indices: np.ndarray | None = None, edge_list: np.ndarray | None = None,
                 *, _device: _DeviceGraph | None = None, _labels: np.ndarray | None = None,
                 _device_labels: bool = False):
        self.num_vertices = int(num_vertices)
        self._ro = None if row_offsets is None else np.asarray(row_offsets, dtype=np.int64)
        self._ci = None if col_indices is None else np.asarray(col_indices, dtype=np.int64)
        self.edge_list = edge_list
        self._dev = _device
        self._labels = _labels
        self._device_labels = _device_labels
        self._info: dict | None = None
        # ordering method behind a reordered graph ("parallel" / "exact" are
        # deterministic, "async" is not); None for graphs not made by
        # preprocess/reorder.  Sharding across ranks checks it.
        self.order_method: str | None = None
        if self._dev is None and (self._ro is None or self._ci is None):
            raise ValueError("Graph needs CSR arrays or a device graph")

    # --- device / host residency ---------------------------------------
    @property
    def device(self) -> _DeviceGraph:
        """The device-resident copy (uploaded from the CSR arrays if needed)."""
        if self._dev is None:
            ro = np.ascontiguousarray(self._ro, dtype=np.int64)
            ci = np.ascontiguousarray(self._ci, dtype=np.int64)
            h = ctypes.c_void_p()
            _lib.check(_lib.lib().mce_graph_from_csr(_lib.ptr(ro), _lib.ptr(ci),
                                                     self.num_vertices, len(ci), 0, None,
                                                     ctypes.byref(h)), "mce_graph_from_csr")
            self._dev = _DeviceGraph(h)
        return self._dev

    def _materialize(self) -> None:
        info = self.device_info()
        ro = np.empty(self.num_vertices + 1, dtype=np.int64)
        ci = np.empty(info["nnz"], dtype=np.int64)
        _lib.check(_lib.lib().mce_graph_copy_csr(self._dev.handle, _lib.ptr(ro), _lib.ptr(ci),
                                                 None, None), "mce_graph_copy_csr")
        self._ro, self._ci = ro, ci

    def device_info(self) -> dict:
        if self._info is None:
            self._info = self.device.info()
        return self._info

    @property
    def row_offsets(self) -> np.ndarray:
        if self._ro is None:
            self._materialize()
        return self._ro

    @property
    def col_indices(self) -> np.ndarray:
        if self._ci is None:
            self._materialize()
        return self._ci

    @property
    def labels(self) -> np.ndarray | None:
        """Original label of every vertex (reordered graphs), else None.
        Copied from the device on first access when the relabel ran there."""
        if self._labels is None and self._device_labels:
            lab = np.empty(self.num_vertices, dtype=np.int64)
            _lib.check(_lib.lib().mce_graph_copy_csr(self._dev.handle, None, None, _lib.ptr(lab),
                                                     None), "mce_graph_copy_csr")
            self._labels = lab
        return self._labels

    # --- reference accessors ---------------------------------------------
    def neighbors(self, v: int) -> np.ndarray:
        ro = self.row_offsets
        return self.col_indices[ro[v]:ro[v + 1]]

    def degree(self, v: int) -> int:
        ro = self.row_offsets
        return int(ro[v + 1] - ro[v])

    @property
    def num_edges(self) -> int:
        if self._ci is not None:
            return len(self._ci) // 2
        return self.device_info()["nnz"] // 2

    def has_edge(self, u: int, v: int) -> bool:
        adj = self.neighbors(u)
        i = int(np.searchsorted(adj, v))
        return i < len(adj) and adj[i] == v

    def edges(self) -> np.ndarray:
        """All undirected edges as an (m, 2) array with u < v, cached."""
        if self.edge_list is None:
            ro, ci = self.row_offsets, self.col_indices
            src = np.repeat(np.arange(self.num_vertices, dtype=np.int64), np.diff(ro))
            keep = src < ci
            self.edge_list = np.column_stack((src[keep], ci[keep]))
        return self.edge_list

    def validate(self) -> None:
        """Check the CSR invariants (reference graph.py:66-82); raises ValueError."""
        ro, ci = self.row_offsets, self.col_indices
        n = self.num_vertices
        if len(ro) != n + 1 or ro[0] != 0 or ro[-1] != len(ci):
            raise ValueError("row_offsets inconsistent with col_indices")
        if np.any(np.diff(ro) < 0):
            raise ValueError("row_offsets not non-decreasing")
        src = np.repeat(np.arange(n, dtype=np.int64), np.diff(ro))
        if len(ci):
            if np.any(ci == src) or np.any(ci < 0) or np.any(ci >= n):
                raise ValueError("self-loop or out-of-range neighbour")
            same_row = src[1:] == src[:-1]
            if np.any(same_row & (ci[1:] <= ci[:-1])):
                raise ValueError("adjacency not strictly ascending")
        fwd = src * np.int64(max(n, 1)) + ci
        rev = ci * np.int64(max(n, 1)) + src
        if not np.array_equal(np.sort(fwd), np.sort(rev)):
            raise ValueError("adjacency not symmetric")

    def __repr__(self) -> str:
        return f"Graph(num_vertices={self.num_vertices}, num_edges={self.num_edges})"


class GraphStats:
    """Headline numbers: size, max degree, degeneracy (reference graph.py:86-92).

    ``max_degree`` / ``degeneracy`` may be resolved lazily (``preprocess``
    returns before the device has finished: they are read from the device
    graph's statistics on first access)."""

    __slots__ = ("n", "_m", "_max_degree", "_degeneracy", "_thunk")

    def __init__(self, n: int, m: int | None = None, max_degree: int | None = None,
                 degeneracy: int | None = None, _thunk=None) -> None:
        self.n = int(n)
        self._m = m
        self._max_degree = max_degree
        self._degeneracy = degeneracy
        self._thunk = _thunk

    def _resolve(self) -> None:
        m, md, d = self._thunk()
        self._m = int(m) if self._m is None else self._m
        self._max_degree = int(md) if self._max_degree is None else self._max_degree
        self._degeneracy = int(d) if self._degeneracy is None else self._degeneracy
        self._thunk = None

    @property
    def m(self) -> int:
        if self._m is None:
            self._resolve()
        return self._m

    @property
    def max_degree(self) -> int:
        if self._max_degree is None:
            self._resolve()
        return self._max_degree

    @property
    def degeneracy(self) -> int:
        if self._degeneracy is None:
            self._resolve()
        return self._degeneracy

    def __eq__(self, other) -> bool:
        return isinstance(other, GraphStats) and (self.n, self.m, self.max_degree, self.degeneracy) \
            == (other.n, other.m, other.max_degree, other.degeneracy)

    def __repr__(self) -> str:
        return (f"GraphStats(n={self.n}, m={self.m}, max_degree={self.max_degree}, "
                f"degeneracy={self.degeneracy})")


class DegeneracyOrder:
    """Permutation original id -> rank plus the degeneracy it realises
    (reference graph.py:96-100).  ``position`` may be produced lazily (by
    ``preprocess``, which keeps the permutation on the device)."""

    __slots__ = ("_position", "_degeneracy", "_thunk", "_dthunk", "method")

    def __init__(self, position: np.ndarray | None, degeneracy: int | None, _thunk=None,
                 _dthunk=None, method: str | None = None) -> None:
        self.method = method
        self._position = position
        self._degeneracy = None if degeneracy is None else int(degeneracy)
        self._thunk = _thunk
        self._dthunk = _dthunk

    @property
    def degeneracy(self) -> int:
        if self._degeneracy is None:
            self._degeneracy = int(self._dthunk())
            self._dthunk = None
        return self._degeneracy

    @property
    def position(self) -> np.ndarray:
        if self._position is None:
            self._position = self._thunk()
            self._thunk = None
        return self._position

    def __eq__(self, other) -> bool:
        return (isinstance(other, DegeneracyOrder) and self.degeneracy == other.degeneracy
                and np.array_equal(self.position, other.position))

    def __repr__(self) -> str:
        return f"DegeneracyOrder(n={len(self.position)}, degeneracy={self.degeneracy})"


def _from_device(n: int, h: ctypes.c_void_p, labels: np.ndarray | None = None) -> Graph:
    return Graph(n, _device=_DeviceGraph(h), _labels=labels)


def from_edges(edges: Iterable[tuple[int, int]] | np.ndarray, num_vertices: int) -> Graph:
    """Canonical graph from compacted vertex pairs, built on the GPU
    (reference graph.py:103-129): self-loops dropped, duplicates merged,
    both directions stored, rows ascending.  An int32 array is shipped as
    is (``mce_graph_from_edges32``: half the host->device bytes); anything
    else as int64, like the reference."""
    if isinstance(edges, np.ndarray) and edges.dtype == np.int32:
        arr = np.ascontiguousarray(edges.reshape(-1, 2))
        entry = "mce_graph_from_edges32"
    else:
        arr = np.ascontiguousarray(
            np.asarray(list(edges) if not isinstance(edges, np.ndarray) else edges,
                       dtype=np.int64).reshape(-1, 2))
        entry = "mce_graph_from_edges"
    h = ctypes.c_void_p()  # ids outside [0, n) are rejected on the device (ValueError)
    _lib.check(getattr(_lib.lib(), entry)(_lib.ptr(arr), len(arr), int(num_vertices), 0,
                                          None, ctypes.byref(h)), entry)
    return _from_device(num_vertices, h)


def from_device_edges(edges_dev, num_edges: int, num_vertices: int, stream=None) -> Graph:
    """Canonical graph from an edge buffer already in device memory
    (int64 or int32 pairs; e.g. a torch CUDA tensor or mce_gen_rmat output)."""
    h = ctypes.c_void_p()
    dt = getattr(edges_dev, "dtype", None)
    entry = "mce_graph_from_edges32" if str(dt) in ("torch.int32", "int32") else \
        "mce_graph_from_edges"
    _lib.check(getattr(_lib.lib(), entry)(_lib.ptr(edges_dev), int(num_edges),
                                          int(num_vertices), 1, stream, ctypes.byref(h)), entry)
    return _from_device(num_vertices, h)


_PARSE_MESSAGES = {
    1: "expected two integer tokens, got {!r}",
    2: "non-integer token in {!r}",
    3: "vertex id below base in {!r}",
}


def parse_edge_list(source: str | bytes | IO[str] | IO[bytes], base: int = 0,
                    symmetrize: bool = True) -> Graph:
    """Parse whitespace-separated edge-list text into a canonical graph
    (reference graph.py:132-180): '#'/'%' comments, a MatrixMarket header
    switches to 1-based ids and skips the size line, ids are compacted to
    [0, n), duplicates merge, self-loops drop, output always symmetric.

    The text is parsed on the GPU (``mce_graph_from_text``): lines are found
    by a device scan, classified and tokenised one thread per line; the
    first malformed line raises ``EdgeListParseError`` with its number, as
    in the reference's sequential loop."""
    del symmetrize  # canonical form is always undirected
    if base not in (0, 1):
        raise ValueError("base must be 0 or 1")
    if isinstance(source, str):
        data = source.encode()
    elif isinstance(source, (bytes, bytearray, memoryview)):
        data = bytes(source)
    else:
        raw = source.read()
        data = raw.encode() if isinstance(raw, str) else bytes(raw)
    h = ctypes.c_void_p()
    line = ctypes.c_int64(0)
    code = ctypes.c_int(0)
    n = ctypes.c_int64(0)
    rc = _lib.lib().mce_graph_from_text(data, len(data), int(base), 0, None, ctypes.byref(h),
                                        ctypes.byref(line), ctypes.byref(code), ctypes.byref(n))
    if rc == -2 and line.value > 0:
        text = data.split(b"\n")[line.value - 1].decode(errors="replace").strip()
        raise EdgeListParseError(line.value, _PARSE_MESSAGES[code.value].format(text))
    _lib.check(rc, "mce_graph_from_text")
    return _from_device(int(n.value), h)


def degeneracy_order(g: Graph, method: str = "async") -> DegeneracyOrder:
    """Degeneracy ordering on the GPU (reference graph.py:183-210); see the
    module docstring for ``method``."""
    if method not in ORDER_METHODS:
        raise ValueError(f"unknown ordering method {method!r}")
    n = g.num_vertices
    pos = np.empty(n, dtype=np.int64)
    d = ctypes.c_int64(0)
    if n:
        _lib.check(_lib.lib().mce_degeneracy_order(g.device.handle, ORDER_METHODS[method],
                                                   _lib.ptr(pos), 0, ctypes.byref(d), None),
                   "mce_degeneracy_order")
    return DegeneracyOrder(pos, int(d.value), method=method)


def reorder(g: Graph, order: DegeneracyOrder) -> Graph:
    """Relabel vertices by rank on the GPU (reference graph.py:213-224)."""
    pos = np.ascontiguousarray(order.position, dtype=np.int64)
    if len(pos) != g.num_vertices:
        raise ValueError("permutation length does not match vertex count")
    n = g.num_vertices
    if n == 0:
        return from_edges(np.empty((0, 2), dtype=np.int64), 0)
    h = ctypes.c_void_p()
    _lib.check(_lib.lib().mce_reorder(g.device.handle, _lib.ptr(pos), 0, None, ctypes.byref(h)),
               "mce_reorder")
    base = g.labels if g.labels is not None else np.arange(n, dtype=np.int64)
    labels = np.empty(n, dtype=np.int64)
    labels[pos] = base
    g2 = _from_device(n, h, labels)
    g2.order_method = order.method
    return g2


def stats(g: Graph, order: DegeneracyOrder) -> GraphStats:
    """Vertex/edge counts, maximum degree and the ordering's degeneracy."""
    if g.num_vertices == 0:
        return GraphStats(0, 0, 0, order.degeneracy)
    if g._ro is not None:
        max_degree = int(np.diff(g._ro).max())
    else:
        max_degree = g.device_info()["max_degree"]
    return GraphStats(n=g.num_vertices, m=g.num_edges, max_degree=max_degree,
                      degeneracy=order.degeneracy)


def preprocess(g: Graph, method: str = "async") -> tuple[Graph, DegeneracyOrder, GraphStats]:
    """Order, relabel and summarise in one step (reference graph.py:239-243).

    One device call (``mce_preprocess``): the permutation never leaves HBM;
    ``order.position`` is rebuilt from the reordered graph's labels only if
    host code reads it."""
    if method not in ORDER_METHODS:
        raise ValueError(f"unknown ordering method {method!r}")
    n = g.num_vertices
    if n == 0:
        order = DegeneracyOrder(np.empty(0, dtype=np.int64), 0, method=method)
        g2 = from_edges(np.empty((0, 2), dtype=np.int64), 0)
        g2.order_method = method
        return g2, order, stats(g2, order)
    h = ctypes.c_void_p()
    # no degeneracy out-parameter: the call returns once its work is queued;
    # the reordered graph's max later degree is the degeneracy
    _lib.check(_lib.lib().mce_preprocess(g.device.handle, ORDER_METHODS[method], None,
                                         None, ctypes.byref(h)), "mce_preprocess")
    g2 = Graph(n, _device=_DeviceGraph(h), _device_labels=True)
    g2.order_method = method
    base = g.labels

    def position() -> np.ndarray:
        # labels2[rank] = label(v)  =>  position[v] = rank of label(v)
        inv = np.empty(n, dtype=np.int64)
        inv[g2.labels] = np.arange(n, dtype=np.int64)
        return inv if base is None else inv[base]

    def device_stats() -> tuple[int, int, int]:
        info = g2.device_info()
        return info["nnz"] // 2, info["max_degree"], info["max_later"]

    order = DegeneracyOrder(None, None, _thunk=position, _dthunk=lambda: device_stats()[2],
                            method=method)
    st = GraphStats(n, _thunk=device_stats)
    return g2, order, st
