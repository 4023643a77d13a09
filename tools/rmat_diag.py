"""R-MAT pipeline at scale on one GPU (diagnostics): device generation,
canonicalisation, ordering, a sampled enumeration.
usage: python tools/rmat_diag.py <scale> [root_stride] [root_end_frac]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess, run, _lib

scale = int(sys.argv[1])
stride = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
frac = float(sys.argv[3]) if len(sys.argv) > 3 else 0.5
m = 16 << scale
n = 1 << scale
t0 = time.perf_counter()
dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
_lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
torch.cuda.synchronize(); t1 = time.perf_counter()
g = from_device_edges(dev, m, n)
torch.cuda.synchronize(); t2 = time.perf_counter()
del dev
g2, order, st = preprocess(g)
t3 = time.perf_counter()
info = g2.device_info()
print(f"rmat{scale}: n={n} m={st.m} maxdeg={st.max_degree} d={st.degeneracy} max|X|={info['max_earlier']} "
      f"gen {1e3*(t1-t0):.1f}ms canon {1e3*(t2-t1):.1f}ms preprocess {1e3*(t3-t2):.1f}ms", flush=True)
end = int(n * frac)
for rep in range(2):
    t4 = time.perf_counter()
    res = run(g2, st, RunConfig(), root_end=end, root_stride=stride)
    t5 = time.perf_counter()
    print(f"  roots[0:{end}:{stride}] count={res.clique_count} nodes={res.nodes_total} "
          f"maxsize={res.max_clique_size} kernel {res.kernel_ms:.2f}ms run {1e3*(t5-t4):.1f}ms "
          f"launches={res.kernel_launches} hash={res.clique_hash_hex}", flush=True)
