"""cProfile of the host side of preprocess() + run() (diagnostics)."""
import cProfile, os, pstats, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_01473_b200 import RunConfig, from_edges, generate, preprocess, run
edges, n = generate.workload_edges("ba200k")
g = from_edges(edges, n)
cfg = RunConfig()
for _ in range(20):
    g2, _, st = preprocess(g); run(g2, st, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    g2, _, st = preprocess(g); r = run(g2, st, cfg)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
