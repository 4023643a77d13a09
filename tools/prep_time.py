"""Device time of preprocess() alone (order + reorder), per method (diagnostics).
usage: python tools/prep_time.py <workload> [method] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_01473_b200 import from_edges, from_device_edges, generate, preprocess, _lib

name = sys.argv[1]
method = sys.argv[2] if len(sys.argv) > 2 else "async"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
if name.startswith("rmat"):
    scale = int(name[4:]); m, n = 16 << scale, 1 << scale
    dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
    g = from_device_edges(dev, m, n); del dev
else:
    edges, n = generate.workload_edges(name)
    g = from_edges(edges, n)
ts = []
for i in range(reps + 3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    g2, _, st = preprocess(g, method=method)
    e1.record(); torch.cuda.synchronize()
    if i >= 3: ts.append(e0.elapsed_time(e1))
print(f"{name} {method} preprocess p50 {np.median(ts):.3f} ms (min {min(ts):.3f}) d={st.degeneracy}", flush=True)
