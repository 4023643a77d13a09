"""Enumerate ONE rmat first-level root (an ncu target for the wide classes).
usage: python tools/one_root.py <scale> <offset from n>"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess, run, _lib

scale, off = int(sys.argv[1]), int(sys.argv[2])
m, n = 16 << scale, 1 << scale
dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
_lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
g = from_device_edges(dev, m, n)
del dev
g2, _, st = preprocess(g, method="parallel")
v = n - off
r = run(g2, st, RunConfig(), root_begin=v, root_end=v + 1)
print(f"rmat{scale} root n-{off}: count={r.clique_count} nodes={r.nodes_total} kernel {r.kernel_ms:.1f} ms "
      f"don={r.donation_count} launches={r.kernel_launches}", flush=True)
