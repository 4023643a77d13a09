"""Per-category worker cycles for the planted1m W = 2 roots (diagnostics).
usage: python tools/w2_timing.py [begin end]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2212_01473_b200 import RunConfig, from_edges, generate, preprocess, run

e, n = generate.workload_edges("planted1m")
g2, _, st = preprocess(from_edges(e, n))
ro, ci = g2.row_offsets, g2.col_indices
later = np.array([int(np.sum(ci[ro[x]:ro[x + 1]] > x)) for x in range(n - 60000, n)])
big = np.nonzero(later > 32)[0] + (n - 60000)
print("W>=2 roots in the last 60k:", len(big), "first", big[:5])
for cfg in (RunConfig(timing=True), RunConfig(timing=True, worker_list=False)):
    for b, e2 in ((int(big[0]), n),):
        r = run(g2, st, cfg, root_begin=b, root_end=e2)
        tot = {}
        for m in r.worker_metrics:
            for k, v in m.times.items():
                tot[k] = tot.get(k, 0.0) + v
        print(f"wl={cfg.worker_list} roots {b}..{e2}: kernel {r.kernel_ms:.3f} ms cliques {r.clique_count} "
              f"nodes {r.nodes_total} p1 {r.phase1_time*1e3:.3f} p2 {r.phase2_time*1e3:.3f} ms", tot)
