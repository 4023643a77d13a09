"""Category cycles of single planted1m roots, enumerated alone (diagnostics).
usage: python tools/one_root_timing.py [k]   (the k widest roots of the last 60k)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2212_01473_b200 import RunConfig, from_edges, generate, preprocess, run

k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
e, n = generate.workload_edges("planted1m")
g2, _, st = preprocess(from_edges(e, n))
ro, ci = g2.row_offsets, g2.col_indices
base = n - 60000
later = np.array([int(np.sum(ci[ro[x]:ro[x + 1]] > x)) for x in range(base, n)])
for v in (np.argsort(-later)[:k] + base).tolist():
    for wl in (True, False):
        r = run(g2, st, RunConfig(timing=True, worker_list=wl), root_begin=v, root_end=v + 1)
        tot = {}
        for m in r.worker_metrics:
            for kk, t in m.times.items():
                tot[kk] = tot.get(kk, 0.0) + t * 1e6
        print(f"root {v} |P|={later[v - base]} |X|={ro[v + 1] - ro[v] - later[v - base]} wl={wl}: "
              f"kernel {r.kernel_ms * 1e3:.0f} us cliques {r.clique_count} nodes {r.nodes_total} "
              + " ".join(f"{kk}={t:.0f}us" for kk, t in tot.items()))
