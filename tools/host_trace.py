"""Host-side cost of one bench step (diagnostics): wall time of preprocess()
and run() per step with a synchronize around each, next to the device time,
plus the cost of individual driver calls the step makes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_01473_b200 import RunConfig, from_edges, generate, preprocess, run

name = sys.argv[1] if len(sys.argv) > 1 else "ba200k"
edges, n = generate.workload_edges(name)
g = from_edges(edges, n)
cfg = RunConfig()
for _ in range(20):
    g2, _, st = preprocess(g); run(g2, st, cfg)
torch.cuda.synchronize()
pre, rn, tot, dev, km = [], [], [], [], []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for i in range(40):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); e0.record()
    g2, _, st = preprocess(g)
    t1 = time.perf_counter()
    r = run(g2, st, cfg)
    e1.record(); t2 = time.perf_counter()
    torch.cuda.synchronize()
    print(f'[step {i}] run wall {1e3*(t2-t1):.3f} ms', file=sys.stderr, flush=True)
    km.append(r.kernel_ms); pre.append(1e3 * (t1 - t0)); rn.append(1e3 * (t2 - t1)); tot.append(1e3 * (t2 - t0)); dev.append(e0.elapsed_time(e1))
def s(x): x = np.array(x); return f"p10 {np.percentile(x,10):.3f} p50 {np.median(x):.3f} p90 {np.percentile(x,90):.3f} max {x.max():.3f}"
print("preprocess wall ms:", s(pre)); print("run wall ms:", s(rn)); print("step wall ms:", s(tot)); print("step device ms:", s(dev))
print("kernel_ms (enumerate):", s(km))
print("per-step (run wall, kernel):", [(round(a,2), round(b,2)) for a, b in zip(rn, km)])
t = []
for i in range(50):
    t0 = time.perf_counter(); torch.cuda.mem_get_info(); t.append(1e3 * (time.perf_counter() - t0))
print("cudaMemGetInfo ms:", s(t))
print("nproc", os.cpu_count(), "loadavg", os.getloadavg())
