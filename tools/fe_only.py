"""from_edges() alone from pinned int32 host edges (ncu launch-list target).
usage: python tools/fe_only.py <workload> [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_01473_b200 import from_edges, generate

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
edges, n = generate.workload_edges(name)
host = torch.from_numpy(np.ascontiguousarray(edges, dtype=np.int32)).pin_memory().numpy()
ts = []
for i in range(reps + 2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    g = from_edges(host, n)
    e1.record(); torch.cuda.synchronize()
    if i >= 2: ts.append(e0.elapsed_time(e1))
print(f"{name} from_edges p50 {np.median(ts):.3f} ms", flush=True)
