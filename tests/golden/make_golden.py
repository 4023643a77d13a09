"""Generate the golden vectors in tests/golden/ by running the REFERENCE itself.

This script imports the reference ``mce`` package from /root/reference/pkg/src
(read-only, present only in the build container) and records, for a set of
small and medium graphs, exactly what the reference computes:

  * the degeneracy ordering (``position``) and degeneracy,
  * per configuration (roots l1/l2 x induced ip/ipx): the clique count, the
    search-tree node total (reference node accounting, workers=1), the size
    histogram and the order-independent clique-set hash (over ORIGINAL labels),
  * for graphs small enough, the brute-force oracle's clique set.

The vectors are committed; tests never read /root/reference at run time.
Run:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from mce.bk import CliqueSink, oracle_enumerate  # noqa: E402  (reference)
from mce.generate import gnp, moon_moser, planted_skew  # noqa: E402  (reference)
from mce.graph import from_edges, preprocess  # noqa: E402  (reference)
from mce.scheduler import RunConfig, run  # noqa: E402  (reference)

from oracle.oracle import summarize_cliques  # noqa: E402  (hash definition only)

MODES = [("l1", "ipx"), ("l1", "ip"), ("l2", "ipx"), ("l2", "ip")]


def record(name: str, g, modes=MODES, brute: bool = False, collect: bool = True) -> dict:
    t0 = time.time()
    edges = [[int(u), int(v)] for u, v in g.edges()]
    g2, order, st = preprocess(g)
    inv = np.argsort(order.position)
    case = {
        "name": name,
        "n": int(g.num_vertices),
        "edges": edges,
        "m": int(st.m),
        "max_degree": int(st.max_degree),
        "degeneracy": int(st.degeneracy),
        "position": [int(x) for x in order.position],
        "runs": {},
    }
    if brute:
        case["brute_force"] = [list(c) for c in oracle_enumerate(g)]
    for roots, induced in modes:
        sink = CliqueSink.collecting(limit=1 << 30) if collect else CliqueSink.counting()
        res = run(g2, st, RunConfig(workers=1, roots=roots, induced=induced), sink=sink)
        entry = {
            "count": int(res.clique_count),
            "nodes": int(sum(w.nodes_visited for w in res.worker_metrics)),
        }
        if collect:
            orig = [tuple(sorted(int(inv[v]) for v in c)) for c in sink.collected]
            entry.update({k: v for k, v in summarize_cliques(orig).items() if k != "count"})
            assert len(orig) == res.clique_count
        case["runs"][f"{roots}-{induced}"] = entry
    print(f"{name}: n={case['n']} m={case['m']} d={case['degeneracy']} "
          f"count={next(iter(case['runs'].values()))['count']} ({time.time() - t0:.1f}s)")
    return case


def main() -> None:
    cases = []
    k4t = [(0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3), (0, 4), (0, 5), (4, 5)]
    cases.append(record("k4_triangle", from_edges(k4t, 6), brute=True))
    cases.append(record("triangle_plus_isolated", from_edges([(0, 1), (1, 2), (0, 2)], 5),
                        brute=True))
    cases.append(record("edgeless4", from_edges([], 4), brute=True))
    cases.append(record("single_edge", from_edges([(0, 1)], 2), brute=True))
    for parts in (2, 3, 4, 5):
        cases.append(record(f"moon_moser_{parts}", moon_moser(parts), brute=parts <= 4))
    i = 0
    for n in (8, 12, 16, 20, 24):
        for p in (0.2, 0.5, 0.8):
            cases.append(record(f"gnp_{n}_{p}_s{i}", gnp(n, p, seed=i), brute=True))
            i += 1
    cases.append(record("gnp_64_0.3_s5", gnp(64, 0.3, seed=5)))
    cases.append(record("gnp_96_0.25_s11", gnp(96, 0.25, seed=11)))
    cases.append(record("gnp_300_0.08_s42", gnp(300, 0.08, seed=42)))
    cases.append(record("gnp_200_0.5_s3", gnp(200, 0.5, seed=3)))
    cases.append(record("skew_2000_40", planted_skew(n=2_000, community=40, p_in=0.95,
                                                     background_degree=2.0, seed=1)))
    cases.append(record("skew_1000_30", planted_skew(n=1_000, community=30, p_in=0.9,
                                                     background_degree=2.0, seed=3)))
    # configs[0] of BASELINE.json: Erdos-Renyi G(n=2000, p=0.01) with the reference generator
    cases.append(record("er_2000_0.01_s0", gnp(2000, 0.01, seed=0)))
    out = os.path.join(HERE, "reference_vectors.json")
    with open(out, "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "/root/reference/pkg (mce 0.1.0)", "cases": cases}, fh)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
