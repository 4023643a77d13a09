"""Split of the e2e step (diagnostics): raw pinned H2D of the edge array,
from_edges (H2D + canonicalisation) and the rest of the step."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_01473_b200 import RunConfig, from_edges, generate, preprocess, run

name = sys.argv[1] if len(sys.argv) > 1 else "ba200k"
edges, n = generate.workload_edges(name)
host = torch.from_numpy(np.ascontiguousarray(edges, dtype=np.int32)).pin_memory()  # as bench.py
hn = host.numpy()
dev = torch.empty_like(host, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for _ in range(5):
    g = from_edges(hn, n); g2, _, st = preprocess(g); run(g2, st, RunConfig())
t_copy, t_fe, t_rest = [], [], []
for _ in range(20):
    torch.cuda.synchronize()
    ev[0].record(); dev.copy_(host, non_blocking=True); ev[1].record()
    torch.cuda.synchronize()
    ev[2].record(); g = from_edges(hn, n); ev[3].record()
    torch.cuda.synchronize()
    t_copy.append(ev[0].elapsed_time(ev[1])); t_fe.append(ev[2].elapsed_time(ev[3]))
    ev[0].record(); g2, _, st = preprocess(g); r = run(g2, st, RunConfig()); ev[1].record()
    torch.cuda.synchronize(); t_rest.append(ev[0].elapsed_time(ev[1]))
print(f"{name}: H2D {host.numel()*4/1e6:.1f} MB {np.median(t_copy):.3f} ms ({host.numel()*4/np.median(t_copy)/1e6:.1f} GB/s); "
      f"from_edges {np.median(t_fe):.3f} ms; preprocess+run {np.median(t_rest):.3f} ms")
