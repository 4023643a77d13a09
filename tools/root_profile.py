"""Per-root cycle profile of one run (diagnostics).
usage: python tools/root_profile.py <workload> [stride]"""
import os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2212_01473_b200 import RunConfig, from_edges, generate, preprocess, run

name = sys.argv[1]
stride = int(sys.argv[2]) if len(sys.argv) > 2 else 1
e, n = generate.workload_edges(name)
g2, _, st = preprocess(from_edges(e, n))
run(g2, st, RunConfig(), root_stride=stride)  # warm
path = os.path.join(tempfile.mkdtemp(), "roots.bin")
os.environ["MCE_PROFILE_ROOTS"] = path
res = run(g2, st, RunConfig(), root_stride=stride)
del os.environ["MCE_PROFILE_ROOTS"]
rec = np.fromfile(path, dtype=np.int64).reshape(-1, 3)
ro, ci = g2.row_offsets, g2.col_indices
v = rec[:, 0]
deg = ro[v + 1] - ro[v]
later = np.array([int(np.sum(ci[ro[x]:ro[x + 1]] > x)) for x in v]) if len(v) < 3_000_000 else deg
cyc = rec[:, 2].astype(np.float64)
print(f"{name}: roots {len(v)} kernel_ms {res.kernel_ms:.3f} cycles total {cyc.sum():.3e} "
      f"mean {cyc.mean():.0f} p50 {np.median(cyc):.0f} p99 {np.percentile(cyc, 99):.0f} max {cyc.max():.0f}")
for W in sorted(set(rec[:, 1].tolist())):
    m = rec[:, 1] == W
    print(f"  W={W}: roots {m.sum()} cycles {cyc[m].sum():.3e} ({100 * cyc[m].sum() / cyc.sum():.1f}%) max {cyc[m].max():.0f}")
top = np.argsort(-cyc)[:15]
print("  top roots: (root, W, cycles, |P|, |X|)")
for i in top:
    print(f"   {v[i]:9d} {rec[i, 1]:4d} {cyc[i]:12.0f} {later[i]:6d} {deg[i] - later[i]:7d}")
