"""One strided chunk of R-MAT first-level roots (diagnostics / ncu target).
usage: python tools/core_chunk.py <scale> <begin> <end> <stride> [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess, run, _lib

scale, b, e, stride = (int(x) for x in sys.argv[1:5])
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 1
m, n = 16 << scale, 1 << scale
dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
_lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
g = from_device_edges(dev, m, n)
del dev
g2, order, st = preprocess(g, method="parallel")  # deterministic order: comparable chunks
for _ in range(reps):
    res = run(g2, st, RunConfig(), root_begin=b, root_end=e, root_stride=stride)
    print(f"rmat{scale} roots[{b}:{e}:{stride}] count={res.clique_count} nodes={res.nodes_total} "
          f"max={res.max_clique_size} kernel {res.kernel_ms:.1f} ms don={res.donation_count} "
          f"hash={res.clique_hash_hex} -> {res.clique_count / (res.kernel_ms / 1e3) / 1e6:.1f} M cliques/s",
          flush=True)
