"""Device time of preprocess() per ordering method (diagnostics).
usage: python tools/order_bench.py [workload ...]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_01473_b200 import RunConfig, from_edges, generate, preprocess, run

for name in (sys.argv[1:] or ["ba200k", "planted1m"]):
    edges, n = generate.workload_edges(name)
    g = from_edges(edges, n)
    for method in ("parallel", "async"):
        for _ in range(5):
            preprocess(g, method=method)
        ts, tr = [], []
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        for _ in range(20):
            torch.cuda.synchronize()
            e0.record(); g2, _, st = preprocess(g, method=method); e1.record()
            r = run(g2, st, RunConfig()); e2.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1)); tr.append(e1.elapsed_time(e2))
        print(f"{name} {method:8s} preprocess p50 {np.median(ts):.3f} ms (min {min(ts):.3f})  run p50 {np.median(tr):.3f} ms "
              f"kernel {r.kernel_ms:.3f}  d={st.degeneracy} count={r.clique_count} nodes={r.nodes_total}", flush=True)
