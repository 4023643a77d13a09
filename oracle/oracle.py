"""TEST INFRASTRUCTURE ONLY -- the CPU parity oracle for the MCE hot path.

A restatement of the reference ``mce`` package (a CPU Python implementation
of arXiv:2212.01473, mounted read-only at /root/reference/pkg) used to *check*
the CUDA engine in ``paper_2212_01473_b200`` and to time the reference
algorithm on host cores.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this module.  The product never does.

Graph canonicalisation / reordering is restated with numpy
(reference graph.py:103-129 ``from_edges`` and graph.py:213-224 ``reorder``);
degeneracy ordering and the Bron-Kerbosch traversal are restated in C
(``mce_oracle.c``, loaded via ctypes).  The restatement is pinned against the
reference itself by the vectors in ``tests/golden`` (made by
``tests/golden/make_golden.py`` importing /root/reference here).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmce_oracle.so")
HIST_MAX = 4096

MASK64 = (1 << 64) - 1
SIZE_SALT = 0xD1B54A32D192ED03


class _Result(ctypes.Structure):
    _fields_ = [
        ("cliques", ctypes.c_int64),
        ("nodes", ctypes.c_int64),
        ("hash", ctypes.c_uint64),
        ("max_size", ctypes.c_int64),
        ("hist", ctypes.c_int64 * HIST_MAX),
    ]


_lib = None


def build() -> str:
    """Compile the oracle library in-tree (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        p64 = ctypes.POINTER(ctypes.c_int64)
        L.mce_oracle_degeneracy_order.restype = ctypes.c_int64
        L.mce_oracle_degeneracy_order.argtypes = [ctypes.c_int64, p64, p64, p64]
        L.mce_oracle_enumerate.restype = ctypes.c_int
        L.mce_oracle_enumerate.argtypes = [
            ctypes.c_int64, p64, p64, ctypes.c_int, ctypes.c_int, ctypes.c_int64, p64,
            ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
            ctypes.POINTER(_Result), p64, ctypes.c_int64, p64,
        ]
        _lib = L
    return _lib


def _p64(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


# --- hashing (shared definition) -------------

def mix64(x):
    """splitmix64 finaliser on uint64 numpy arrays or python ints."""
    if isinstance(x, np.ndarray):
        with np.errstate(over="ignore"):
            x = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
            x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            return x ^ (x >> np.uint64(31))
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def clique_hash(labels) -> int:
    s = 0
    for v in labels:
        s = (s + mix64(int(v))) & MASK64
    return mix64((s + len(labels) * SIZE_SALT) & MASK64)


def summarize_cliques(cliques) -> dict:
    """count / size histogram / order-independent hash of an explicit clique list."""
    total = 0
    hist: dict[int, int] = {}
    h = 0
    for c in cliques:
        total += 1
        hist[len(c)] = hist.get(len(c), 0) + 1
        h = (h + clique_hash(c)) & MASK64
    return {"count": total, "hist": {int(k): int(v) for k, v in sorted(hist.items())},
            "hash": f"{h:016x}"}


# --- graph canonicalisation (restates graph.py:103-129, 221-232) ----------

def from_edges(edges, n: int) -> tuple[np.ndarray, np.ndarray]:
    """Canonical CSR (row_offsets, col_indices) from vertex pairs: loops
    dropped, duplicates merged, both directions present, rows ascending."""
    arr = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    ro = np.zeros(n + 1, dtype=np.int64)
    if arr.size == 0:
        return ro, np.empty(0, dtype=np.int64)
    lo = np.minimum(arr[:, 0], arr[:, 1])
    hi = np.maximum(arr[:, 0], arr[:, 1])
    keep = lo != hi
    key = np.unique(lo[keep] * np.int64(n) + hi[keep])
    a, b = key // n, key % n
    src = np.concatenate((a, b))
    dst = np.concatenate((b, a))
    order = np.argsort(src * np.int64(n) + dst, kind="stable")
    src, dst = src[order], dst[order]
    np.cumsum(np.bincount(src, minlength=n), out=ro[1:])
    return ro, np.ascontiguousarray(dst)


def upper_edges(ro: np.ndarray, ci: np.ndarray) -> np.ndarray:
    n = len(ro) - 1
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(ro))
    keep = src < ci
    return np.column_stack((src[keep], ci[keep]))


def degeneracy_order(ro: np.ndarray, ci: np.ndarray) -> tuple[np.ndarray, int]:
    n = len(ro) - 1
    pos = np.empty(n, dtype=np.int64)
    d = lib().mce_oracle_degeneracy_order(n, _p64(ro), _p64(ci), _p64(pos))
    return pos, int(d)


def reorder(ro: np.ndarray, ci: np.ndarray, position: np.ndarray):
    n = len(ro) - 1
    e = upper_edges(ro, ci)
    return from_edges(position[e], n)


def round_up_capacity(nbits: int) -> int:
    return max(1, -(-nbits // 64)) * 64


def enumerate_cliques(ro: np.ndarray, ci: np.ndarray, roots: str = "l1",
                      induced: str = "ipx", degeneracy: int | None = None,
                      labels: np.ndarray | None = None, root_begin: int = 0,
                      root_end: int = -1, root_stride: int = 1,
                      include_isolated: bool = True, threads: int = 0,
                      collect: int = 0) -> dict:
    """Run the restated traversal on a canonical, degeneracy-reordered CSR."""
    n = len(ro) - 1
    ro = np.ascontiguousarray(ro, dtype=np.int64)
    ci = np.ascontiguousarray(ci, dtype=np.int64)
    if degeneracy is None:
        later = ro[1:] - np.array([np.searchsorted(ci[ro[v]:ro[v + 1]], v) + ro[v]
                                   for v in range(n)], dtype=np.int64) if n else np.zeros(0)
        degeneracy = int(later.max()) if n else 0
    cap = round_up_capacity(max(degeneracy, 1))
    res = _Result()
    buf = np.zeros(max(collect, 1), dtype=np.int64) if collect else None
    used = np.zeros(1, dtype=np.int64)
    if labels is not None:
        labels = np.ascontiguousarray(labels, dtype=np.int64)
    rc = lib().mce_oracle_enumerate(
        n, _p64(ro), _p64(ci), 1 if roots == "l1" else 2, 1 if induced == "ipx" else 0,
        cap, _p64(labels), root_begin, root_end, root_stride, int(include_isolated),
        threads, ctypes.byref(res), _p64(buf), collect, _p64(used))
    if rc != 0:
        raise RuntimeError(f"oracle enumerate failed rc={rc}")
    hist = {s: int(res.hist[s]) for s in range(HIST_MAX) if res.hist[s]}
    out = {"count": int(res.cliques), "nodes": int(res.nodes), "hash": f"{res.hash:016x}",
           "hist": hist, "max_size": int(res.max_size)}
    if collect:
        cl = []
        i, end = 0, min(int(used[0]), collect)
        while i < end:
            s = int(buf[i])
            if i + 1 + s > end:
                break
            cl.append(tuple(sorted(int(x) for x in buf[i + 1:i + 1 + s])))
            i += 1 + s
        out["cliques"] = cl
    return out


def reference_pipeline(edges, n: int, roots: str = "l1", induced: str = "auto",
                       threads: int = 0, collect: int = 0, **kw) -> dict:
    """from_edges -> degeneracy order -> reorder -> enumerate, hashing cliques
    by their ORIGINAL labels (so results compare across orderings)."""
    ro, ci = from_edges(edges, n)
    pos, d = degeneracy_order(ro, ci)
    ro2, ci2 = reorder(ro, ci, pos)
    inv = np.empty(n, dtype=np.int64)
    inv[pos] = np.arange(n, dtype=np.int64)
    deg = np.diff(ro2)
    max_degree = int(deg.max()) if n else 0
    if induced == "auto":
        induced = "ip" if d > 0 and max_degree / d > 200.0 else "ipx"
    out = enumerate_cliques(ro2, ci2, roots=roots, induced=induced, degeneracy=d,
                            labels=inv, threads=threads, collect=collect, **kw)
    out.update({"n": n, "m": int(len(ci) // 2), "degeneracy": d, "max_degree": max_degree,
                "induced": induced, "roots": roots})
    return out


def bucket_peel_order(ro: np.ndarray, ci: np.ndarray) -> tuple[np.ndarray, int]:
    """The GPU's ``method="parallel"`` ordering restated in numpy (NOT the
    reference's; its exact order is ``degeneracy_order``): round-synchronous
    bucket peeling -- at level k every live vertex with current degree <= k
    leaves in the same round, ranked by id; an empty round raises k to
    max(k + 1, min live degree); the degeneracy is the largest level at which
    a round removed vertices."""
    n = len(ro) - 1
    deg = np.diff(ro).astype(np.int64)
    alive = np.ones(n, dtype=bool)
    pos = np.empty(n, dtype=np.int64)
    src = np.repeat(np.arange(n, dtype=np.int64), np.diff(ro))
    k = 0
    base = 0
    dmax = 0
    while base < n:
        take = alive & (deg <= k)
        if not take.any():
            k = max(k + 1, int(deg[alive].min()))
            continue
        ids = np.flatnonzero(take)
        pos[ids] = base + np.arange(len(ids))
        base += len(ids)
        dmax = max(dmax, k)
        alive &= ~take
        hit = take[src] & alive[ci]
        np.subtract.at(deg, ci[hit], 1)
    return pos, dmax
