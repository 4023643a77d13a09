"""Single-root probe of R-MAT's densest first-level roots (diagnostics).
usage: python tools/w32_probe.py <scale> <induced ip|ipx|auto> <root offsets from n, e.g. 1408,1000,1>
Prints |P|, |X| and the enumeration of each root alone (count, nodes, kernel ms)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess, run, _lib

scale, induced = int(sys.argv[1]), sys.argv[2]
offs = [int(x) for x in sys.argv[3].split(",")]
m, n = 16 << scale, 1 << scale
dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
_lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
g = from_device_edges(dev, m, n)
del dev
g2, order, st = preprocess(g, method="parallel")
ro, col = g2.row_offsets, g2.col_indices
print(f"rmat{scale}: n={n} d={st.degeneracy} maxdeg={st.max_degree}", flush=True)
for o in offs:
    v = n - o
    row = col[ro[v]:ro[v + 1]]
    cut = int(np.searchsorted(row, v))
    t = time.perf_counter()
    r = run(g2, st, RunConfig(induced=induced), root_begin=v, root_end=v + 1)
    print(f"root n-{o} (v={v}): |P|={len(row) - cut} |X|={cut} count={r.clique_count} nodes={r.nodes_total} "
          f"max={r.max_clique_size} kernel {r.kernel_ms:.1f} ms wall {time.perf_counter() - t:.1f}s "
          f"don={r.donation_count} mode={r.induced_mode} -> {r.clique_count / max(r.kernel_ms, 1e-3) / 1e3:.1f} M/s",
          flush=True)
