"""Per-class cycle profile on an R-MAT root sample (diagnostics).
usage: python tools/root_profile_rmat.py <scale> <stride> <end_frac>"""
import os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_01473_b200 import RunConfig, from_device_edges, preprocess, run, _lib

scale, stride, frac = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
induced = sys.argv[4] if len(sys.argv) > 4 else "auto"
m, n = 16 << scale, 1 << scale
dev = torch.empty((m, 2), dtype=torch.int64, device="cuda")
_lib.check(_lib.lib().mce_gen_rmat(scale, 0, m, 0, _lib.ptr(dev), None), "gen")
g2, _, st = preprocess(from_device_edges(dev, m, n))
del dev
end = int(n * frac)
run(g2, st, RunConfig(induced=induced), root_end=end, root_stride=stride)
path = os.path.join(tempfile.mkdtemp(), "roots.bin")
os.environ["MCE_PROFILE_ROOTS"] = path
res = run(g2, st, RunConfig(induced=induced), root_end=end, root_stride=stride)
del os.environ["MCE_PROFILE_ROOTS"]
rec = np.fromfile(path, dtype=np.int64).reshape(-1, 3)
cyc = rec[:, 2].astype(np.float64)
print(f"rmat{scale} [{res.induced_mode}] roots[0:{end}:{stride}] count={res.clique_count} kernel_ms={res.kernel_ms:.2f} "
      f"donations={res.donation_count} roots={len(rec)} cycles total {cyc.sum():.3e}")
for W in sorted(set(rec[:, 1].tolist())):
    msk = rec[:, 1] == W
    c = cyc[msk]
    print(f"  W={W:3d}: roots {msk.sum():8d} cycles {c.sum():.3e} ({100 * c.sum() / cyc.sum():5.1f}%) "
          f"mean {c.mean():10.0f} max {c.max():12.0f}")
