"""Cliques per first-level root at offsets from the end of R-MAT's order
(where the oracle can still follow: picks the parity-test samples).
usage: python tools/core_offsets.py <scale> <offset>,<offset>,... [stride] [count]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess, run, _lib

scale = int(sys.argv[1])
offs = [int(x) for x in sys.argv[2].split(",")]
stride = int(sys.argv[3]) if len(sys.argv) > 3 else 1
cnt = int(sys.argv[4]) if len(sys.argv) > 4 else 64
m, n = 16 << scale, 1 << scale
dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
_lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
g = from_device_edges(dev, m, n)
del dev
torch.cuda.empty_cache()
g2, order, st = preprocess(g)
ro = g2.row_offsets
print(f"rmat{scale}: n={n} d={st.degeneracy}", flush=True)
for o in offs:
    b = n - o
    e = b + cnt * stride
    t = time.perf_counter()
    r = run(g2, st, RunConfig(), root_begin=b, root_end=e, root_stride=stride)
    print(f"roots[n-{o} : +{cnt}x{stride}] count={r.clique_count} ({r.clique_count / cnt:.0f}/root) "
          f"max={r.max_clique_size} kernel {r.kernel_ms:.1f} ms", flush=True)
