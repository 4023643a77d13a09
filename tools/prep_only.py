"""preprocess() only, a few times (ncu launch-list target).
usage: python tools/prep_only.py <workload> [method] [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_01473_b200 import from_edges, generate, preprocess
name = sys.argv[1]; method = sys.argv[2] if len(sys.argv) > 2 else "async"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
edges, n = generate.workload_edges(name)
g = from_edges(edges, n)
for _ in range(reps):
    g2, _, st = preprocess(g, method=method)
    torch.cuda.synchronize()
print("d", st.degeneracy)
