"""Seed-deterministic synthetic graph generators (input synthesis, host side).

Mirrors the reference generator API (reference mce/generate.py:17-68:
``gnp``, ``moon_moser``, ``planted_skew``, ``write_edge_list``) -- the first
three consume numpy's PCG64 stream in exactly the reference's order, so the
same seed yields the same graph -- and adds the generators behind the five
BASELINE.json workloads:

* ``barabasi_albert(n, m)``   -- preferential attachment (Batagelj-Brandes copy model)
* ``rmat_edges(scale, ef)``   -- Graph500-style R-MAT/Kronecker with a counter-based RNG
                                 (the same stream as the CUDA generator in csrc/synth.cu)
* ``planted_cliques(n, ...)`` -- uniform random background + planted cliques

Generators return either a :class:`~paper_2212_01473_b200.graph.Graph` (reference
API) or, for the large workloads, a raw ``(m, 2)`` int64 edge array that feeds
``graph.from_edges`` (which canonicalises on the GPU).
"""

from __future__ import annotations

from typing import IO

import numpy as np

MASK64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)


# --- counter-based RNG (identical on host and device) --------------------

def mix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser, vectorised over uint64."""
    with np.errstate(over="ignore"):
        x = x.astype(np.uint64, copy=True) + GOLDEN
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def counter_u64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """64 random bits for counter ``idx`` of ``stream`` under ``seed``."""
    key = mix64(np.asarray([seed * 0x100 + stream], dtype=np.uint64))[0]
    return mix64(idx.astype(np.uint64) ^ key)


def counter_unit(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Uniform doubles in [0, 1) with 53 random bits."""
    return (counter_u64(seed, stream, idx) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


# --- reference-compatible generators --------------------------------------

def gnp(n: int, p: float, seed: int = 0):
    """Erdos-Renyi G(n, p) drawing the reference's PCG64 stream
    (reference generate.py:17-26: one uniform per pair (u, v>u), row-major)."""
    from paper_2212_01473_b200.graph import from_edges

    if n < 0 or not 0.0 <= p <= 1.0:
        raise ValueError("need n >= 0 and 0 <= p <= 1")
    return from_edges(gnp_edges(n, p, seed), n)


def gnp_edges(n: int, p: float, seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    out = []
    # the stream is consumed row by row; drawing rows in blocks keeps it identical
    u = 0
    while u < n:
        rows = []
        total = 0
        u_end = u
        while u_end < n and total < (1 << 22):
            total += n - u_end - 1
            u_end += 1
        draws = rng.random(total) < p
        off = 0
        for uu in range(u, u_end):
            k = n - uu - 1
            hits = np.flatnonzero(draws[off:off + k])
            if hits.size:
                rows.append(np.column_stack((np.full(hits.size, uu, dtype=np.int64),
                                             hits.astype(np.int64) + uu + 1)))
            off += k
        if rows:
            out.append(np.concatenate(rows))
        u = u_end
    return np.concatenate(out) if out else np.empty((0, 2), dtype=np.int64)


def moon_moser(parts: int):
    """Complete multipartite graph with ``parts`` parts of size 3 (3**parts
    maximal cliques); reference generate.py:29-38."""
    from paper_2212_01473_b200.graph import from_edges

    if parts < 1:
        raise ValueError("parts must be >= 1")
    n = 3 * parts
    u, v = np.triu_indices(n, k=1)
    keep = (u // 3) != (v // 3)
    return from_edges(np.column_stack((u[keep], v[keep])).astype(np.int64), n)


def planted_skew(n: int = 10_000, community: int = 40, p_in: float = 0.8,
                 background_degree: float = 4.0, seed: int = 0):
    """Sparse background plus one dense community, same stream as reference
    generate.py:41-62."""
    from paper_2212_01473_b200.graph import from_edges

    if community > n:
        raise ValueError("community larger than the graph")
    rng = np.random.default_rng(seed)
    p_bg = min(1.0, background_degree / max(n, 1))
    tri = n * (n - 1) // 2
    parts = []
    # background: row-major pairs, one uniform each
    done = 0
    u = 0
    while u < n:
        u_end, total = u, 0
        while u_end < n and total < (1 << 22):
            total += n - u_end - 1
            u_end += 1
        hits = np.flatnonzero(rng.random(total) < p_bg)
        if hits.size:
            # map flat offsets inside this row block back to (row, col)
            lens = n - np.arange(u, u_end, dtype=np.int64) - 1
            starts = np.concatenate(([0], np.cumsum(lens)[:-1]))
            rows = np.searchsorted(starts, hits, side="right") - 1
            cols = hits - starts[rows] + (u + rows) + 1
            parts.append(np.column_stack((u + rows, cols)))
        done += total
        u = u_end
    assert done == tri
    members = np.sort(rng.choice(n, size=community, replace=False))
    iu, ju = np.triu_indices(community, k=1)
    keep = rng.random(iu.size) < p_in
    parts.append(np.column_stack((members[iu[keep]], members[ju[keep]])).astype(np.int64))
    edges = np.concatenate(parts) if parts else np.empty((0, 2), dtype=np.int64)
    return from_edges(edges, n)


def write_edge_list(g, out: IO[str]) -> None:
    """Canonical edge-list text: one ``u v`` line per undirected edge (u < v)."""
    e = g.edges()
    if len(e):
        np.savetxt(out, e, fmt="%d")


# --- BASELINE.json workloads ------------------------------------------------

def barabasi_albert_edges(n: int, m: int, seed: int = 0) -> np.ndarray:
    """Preferential attachment via the Batagelj-Brandes copy model: edge j
    (source j // m) targets the endpoint stored at a uniformly random earlier
    slot of the endpoint array, i.e. a vertex chosen proportionally to degree.
    Copy chains are resolved by pointer jumping (vectorised)."""
    if n < 1 or m < 1:
        raise ValueError("need n >= 1 and m >= 1")
    E = n * m
    j = np.arange(E, dtype=np.int64)
    # slot 2j holds the source, slot 2j+1 copies slot r_j in [0, 2j]
    r = (counter_u64(seed, 1, j) % (2 * j + 1).astype(np.uint64)).astype(np.int64)
    ptr = r.copy()
    for _ in range(128):
        odd = (ptr & 1) == 1
        if not odd.any():
            break
        ptr[odd] = r[ptr[odd] >> 1]
    else:  # pragma: no cover - probability ~0
        raise RuntimeError("copy chains did not resolve")
    src = j // m
    dst = (ptr >> 1) // m
    return np.column_stack((src, dst))


RMAT_A, RMAT_B, RMAT_C = 0.57, 0.19, 0.19


def _scramble(x: np.ndarray, scale: int, seed: int) -> np.ndarray:
    """A bijection of [0, 2**scale) (odd multiply + xorshift rounds)."""
    mask = np.uint64((1 << scale) - 1)
    k1 = np.uint64((int(mix64(np.asarray([seed + 11], np.uint64))[0]) | 1))
    k2 = np.uint64((int(mix64(np.asarray([seed + 13], np.uint64))[0]) | 1))
    s1 = np.uint64(max(1, scale // 2))
    s2 = np.uint64(max(1, scale // 3))
    with np.errstate(over="ignore"):
        x = x.astype(np.uint64)
        x = (x * k1) & mask
        x ^= x >> s1
        x = (x * k2) & mask
        x ^= x >> s2
        x = (x * k1) & mask
    return x.astype(np.int64)


def rmat_edges(scale: int, edge_factor: int = 16, seed: int = 0,
               start: int = 0, count: int | None = None) -> np.ndarray:
    """R-MAT (a, b, c, d) = (0.57, 0.19, 0.19, 0.05) edges ``start ..
    start+count`` of ``edge_factor * 2**scale``, then a seeded vertex
    scramble.  Counter-based, so any slice can be produced independently and
    the CUDA generator (csrc/synth.cu) emits the identical stream."""
    total = edge_factor << scale
    if count is None:
        count = total - start
    e = np.arange(start, start + count, dtype=np.int64)
    u = np.zeros(count, dtype=np.int64)
    v = np.zeros(count, dtype=np.int64)
    ab, abc = RMAT_A + RMAT_B, RMAT_A + RMAT_B + RMAT_C
    for level in range(scale):
        r = counter_unit(seed, 2, e * scale + level)
        bit = np.int64(1) << np.int64(scale - 1 - level)
        u += np.where(r >= ab, bit, 0)
        v += np.where(((r >= RMAT_A) & (r < ab)) | (r >= abc), bit, 0)
    return np.column_stack((_scramble(u, scale, seed), _scramble(v, scale, seed)))


def planted_cliques_edges(n: int = 1_000_000, avg_degree: float = 20.0,
                          cliques: int = 1000, min_size: int = 30, max_size: int = 60,
                          seed: int = 0) -> np.ndarray:
    """Uniform random background with ``n * avg_degree / 2`` edge draws
    (an Erdos-Renyi G(n, M) up to duplicate draws) plus ``cliques`` planted
    cliques with sizes uniform in [min_size, max_size]."""
    M = int(round(n * avg_degree / 2))
    idx = np.arange(M, dtype=np.int64)
    a = (counter_u64(seed, 3, 2 * idx) % np.uint64(n)).astype(np.int64)
    b = (counter_u64(seed, 3, 2 * idx + 1) % np.uint64(n)).astype(np.int64)
    parts = [np.column_stack((a, b))]
    rng = np.random.default_rng(seed)
    sizes = rng.integers(min_size, max_size + 1, size=cliques)
    for s in sizes:
        members = rng.choice(n, size=int(s), replace=False)
        iu, ju = np.triu_indices(int(s), k=1)
        parts.append(np.column_stack((members[iu], members[ju])).astype(np.int64))
    return np.concatenate(parts)


WORKLOADS = {
    "er2k": "Erdos-Renyi G(n=2000, p=0.01) (reference gnp, seed 0)",
    "ba200k": "Barabasi-Albert n=200k, m=8",
    "rmat20": "RMAT scale-20, edge factor 16",
    "planted1m": "ER n=1M avg deg 20 + 1k planted cliques of size 30-60",
    "rmat24": "RMAT scale-24, edge factor 16",
}


def workload_edges(name: str, seed: int = 0) -> tuple[np.ndarray, int]:
    """Edge array and vertex count of one BASELINE.json workload (host numpy).
    rmat24 is best generated on the device (graph.rmat_device)."""
    if name == "er2k":
        return gnp_edges(2000, 0.01, seed), 2000
    if name == "ba200k":
        return barabasi_albert_edges(200_000, 8, seed), 200_000
    if name == "rmat20":
        return rmat_edges(20, 16, seed), 1 << 20
    if name == "planted1m":
        return planted_cliques_edges(1_000_000, 20.0, 1000, 30, 60, seed), 1_000_000
    if name == "rmat24":
        return rmat_edges(24, 16, seed), 1 << 24
    raise ValueError(f"unknown workload {name!r}")
