"""from_edges only, a few times (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2212_01473_b200 import from_edges, generate
edges, n = generate.workload_edges(sys.argv[1] if len(sys.argv) > 1 else "ba200k")
hn = torch.from_numpy(np.ascontiguousarray(edges)).pin_memory().numpy()
for _ in range(3):
    g = from_edges(hn, n); torch.cuda.synchronize()
