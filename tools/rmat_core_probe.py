"""Time-bounded probe of the R-MAT dense core on one GPU (diagnostics):
enumerate strided samples of the last first-level roots (the core, where the
maximal cliques concentrate) and extrapolate the full-graph cost.
usage: python tools/rmat_core_probe.py <scale> <core_roots> <stride> <budget_s>"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess, run, _lib

scale, core, stride, budget = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
m, n = 16 << scale, 1 << scale
dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
_lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
g = from_device_edges(dev, m, n)
del dev
g2, order, st = preprocess(g)
print(f"rmat{scale}: n={n} m={st.m} d={st.degeneracy}", flush=True)
t_start = time.perf_counter()
tot_c = tot_ms = 0
for b in range(n - core, n, 1024):
    e = min(b + 1024, n)
    res = run(g2, st, RunConfig(), root_begin=b, root_end=e, root_stride=stride)
    tot_c += res.clique_count
    tot_ms += res.kernel_ms
    print(f"  roots[{b}:{e}:{stride}] count={res.clique_count} nodes={res.nodes_total} max={res.max_clique_size} "
          f"kernel {res.kernel_ms:.1f}ms  (x{stride} est {res.kernel_ms*stride/1e3:.1f}s, {res.clique_count*stride:.3g} cliques)",
          flush=True)
    if time.perf_counter() - t_start > budget:
        print("  budget reached", flush=True)
        break
print(f"sampled total count={tot_c} kernel {tot_ms:.1f}ms -> est full core x{stride}: {tot_ms*stride/1e3:.1f}s, {tot_c*stride:.3g} cliques")
