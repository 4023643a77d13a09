"""Device time of from_edges() from pinned int32 host edges, the way bench.py's
e2e arm calls it (L2 flushed before; the previous graph alive meanwhile).
usage: python tools/fe_time.py <workload> [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_01473_b200 import from_edges, generate

name = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
edges, n = generate.workload_edges(name)
host = torch.from_numpy(np.ascontiguousarray(edges, dtype=np.int32)).pin_memory()
hn = host.numpy()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts, prev = [], None
for i in range(reps + 3):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    g = from_edges(hn, n)
    e1.record(); torch.cuda.synchronize()
    prev = g
    if i >= 3: ts.append(e0.elapsed_time(e1))
print(f"{name} from_edges p50 {np.median(ts):.3f} ms (min {min(ts):.3f}, max {max(ts):.3f})", flush=True)
