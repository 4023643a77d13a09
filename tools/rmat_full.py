"""Full R-MAT enumeration on one GPU in root chunks (first-level subtrees are
independent, so chunk results add up exactly: counts, node totals, size
histograms, and the clique-set hash mod 2^64).  Prints every chunk as it
finishes, so a run cut short still leaves its partial sums.
usage: python tools/rmat_full.py <scale> [core_roots] [chunk] [budget_s]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess, run, _lib

scale = int(sys.argv[1])
core = int(sys.argv[2]) if len(sys.argv) > 2 else 8576
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 512
budget = float(sys.argv[4]) if len(sys.argv) > 4 else 1e9
m, n = 16 << scale, 1 << scale
t0 = time.perf_counter()
dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
_lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
g = from_device_edges(dev, m, n)
del dev
g2, order, st = preprocess(g)
print(f"rmat{scale}: n={n} m={st.m} d={st.degeneracy} maxdeg={st.max_degree} "
      f"setup {time.perf_counter() - t0:.1f}s", flush=True)
bounds = [0, n - core] + list(range(n - core + chunk, n, chunk)) + [n]
tot_c = tot_n = tot_h = 0
tot_ms = 0.0
hist = {}
t_run = time.perf_counter()
for b, e in zip(bounds[:-1], bounds[1:]):
    res = run(g2, st, RunConfig(), root_begin=b, root_end=e)
    tot_c += res.clique_count
    tot_n += res.nodes_total
    tot_h = (tot_h + res.clique_hash) % (1 << 64)
    tot_ms += res.kernel_ms
    for s, c in res.size_histogram.items():
        hist[s] = hist.get(s, 0) + c
    print(f"  roots[{b}:{e}] count={res.clique_count} nodes={res.nodes_total} max={res.max_clique_size} "
          f"kernel {res.kernel_ms:.1f} ms don={res.donation_count} | total count={tot_c} "
          f"kernel {tot_ms / 1e3:.1f} s wall {time.perf_counter() - t_run:.1f} s", flush=True)
    if time.perf_counter() - t_run > budget:
        print("  budget reached: partial", flush=True)
        break
else:
    print(f"FULL rmat{scale}: count={tot_c} nodes={tot_n} hash={tot_h:016x} max={max(hist)} "
          f"kernel {tot_ms / 1e3:.2f} s -> {tot_c / (tot_ms / 1e3) / 1e6:.1f} M cliques/s", flush=True)
    print("hist", dict(sorted(hist.items())), flush=True)
